import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib
lib = _lib.load()
M = 786432; sp = _lib.stream_ptr()
buf = (C.c_ulonglong * 64)()
lib.fv_g3_prof(buf)  # allocate + enable
names = ["prod wait empty", "mma wait conv", "conv wait full", "conv loop total"]
for K, N in [(128, 128), (128, 3)]:
    x = torch.randn(M, K, device="cuda"); dz = torch.randn(M, N, device="cuda")
    dw = torch.zeros(K, N, device="cuda"); db = torch.zeros(N, device="cuda")
    f = lambda: lib.fv_linear_bwd_tc(x.data_ptr(), K, x.data_ptr(), dz.data_ptr(), N, None, 0, None, dw.data_ptr(), db.data_ptr(), M, K, N, sp)
    f(); lib.fv_g3_prof(buf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1); lib.fv_g3_prof(buf)
    cyc = ms * 1e-3 * 1.9e9
    div = [148, 148, 148 * 128, 148 * 128]
    print(f"K={K} N={N}: {ms*1e3:.1f} us = {cyc:.0f} cyc")
    for i, n in enumerate(names):
        print(f"  {n:18s} {buf[i] / div[i]:10.0f} cyc/CTA ({buf[i] / div[i] / cyc:5.1%})")
