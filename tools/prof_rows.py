import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib
lib = _lib.load()
M = 786432; sp = _lib.stream_ptr()
names = ["prod wait empty", "mma wait tempty", "mma wait aready", "conv wait full", "conv wait afree", "epi wait tfull"]
for K, N in [(128, 128)]:
    x = torch.randn(M, K, device="cuda"); w = torch.randn(K, N, device="cuda"); b = torch.randn(N, device="cuda")
    y = torch.empty(M, N, device="cuda")
    buf = (C.c_ulonglong * 64)()
    lib.fv_linear_fwd_tc(x.data_ptr(), K, w.data_ptr(), b.data_ptr(), y.data_ptr(), N, M, K, N, 1, sp)
    lib.fv_g3_prof(buf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.fv_linear_fwd_tc(x.data_ptr(), K, w.data_ptr(), b.data_ptr(), y.data_ptr(), N, M, K, N, 1, sp)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    lib.fv_g3_prof(buf)
    cyc = ms * 1e-3 * 1.9e9
    # per-CTA average: producer/mma counted by 1 thread per CTA; converter/epilogue by 128 threads
    div = [148, 148, 148, 148 * 128, 148 * 128, 148 * 128]
    print(f"K={K} N={N}: {ms*1e3:.1f} us = {cyc:.0f} cyc")
    for i, n in enumerate(names):
        print(f"  {n:18s} {buf[i] / div[i]:10.0f} cyc/CTA ({buf[i] / div[i] / cyc:5.1%})")
