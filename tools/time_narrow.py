"""Time the n_out <= 4 layer kernels (fwd / dX / dW) at config-3 scale (tuning helper)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib  # noqa: E402

lib = _lib.load()
sp = _lib.stream_ptr()
M = 786432


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for K, N in [(128, 3), (64, 4)]:
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(K, N, device="cuda")
    b = torch.randn(N, device="cuda")
    y = torch.empty(M, N, device="cuda")
    dz = torch.randn(M, N, device="cuda")
    dw = torch.zeros(K, N, device="cuda")
    db = torch.zeros(N, device="cuda")
    tf = timeit(lambda: lib.fv_linear_fwd_tc_bits(x.data_ptr(), K, w.data_ptr(), b.data_ptr(), y.data_ptr(), N, M, K, N, 0,
                                                  None, sp))
    tw = timeit(lambda: lib.fv_linear_bwd_tc_bits(x.data_ptr(), K, w.data_ptr(), dz.data_ptr(), N, None, 0, None,
                                                  dw.data_ptr(), db.data_ptr(), M, K, N, sp))
    print(f"narrow K={K} N={N}: fwd {tf:.1f} us  dW {tw:.1f} us", flush=True)
