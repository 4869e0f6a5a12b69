"""Time the training layer GEMM entry points at config-3 scale (tuning helper)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib  # noqa: E402

lib = _lib.load()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 786432
sp = _lib.stream_ptr()


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


for K, N in [(128, 128), (40, 128), (32, 64), (64, 64), (128, 3)]:
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(K, N, device="cuda") / K ** 0.5
    b = torch.randn(N, device="cuda")
    y = torch.empty(M, N, device="cuda")
    bits = torch.empty(M, (N + 31) // 32, device="cuda", dtype=torch.int32)
    dz = torch.randn(M, N, device="cuda")
    dx = torch.empty(M, K, device="cuda")
    dw = torch.zeros(K, N, device="cuda")
    db = torch.zeros(N, device="cuda")
    xb = torch.empty(M, (K + 31) // 32, device="cuda", dtype=torch.int32).fill_(-1)
    t_fwd = timeit(lambda: lib.fv_linear_fwd_tc(x.data_ptr(), K, w.data_ptr(), b.data_ptr(), y.data_ptr(), N, M, K, N, 1, sp))
    t_fwdb = timeit(lambda: lib.fv_linear_fwd_tc_bits(x.data_ptr(), K, w.data_ptr(), b.data_ptr(), y.data_ptr(), N, M, K,
                                                      N, 1, bits.data_ptr(), sp))
    t_dx = timeit(lambda: lib.fv_linear_bwd_tc(x.data_ptr(), K, w.data_ptr(), dz.data_ptr(), N, dx.data_ptr(), K,
                                               x.data_ptr(), None, None, M, K, N, sp))
    t_dxb = timeit(lambda: lib.fv_linear_bwd_tc_bits(x.data_ptr(), K, w.data_ptr(), dz.data_ptr(), N, dx.data_ptr(), K,
                                                     xb.data_ptr(), None, None, M, K, N, sp))
    t_dw = timeit(lambda: lib.fv_linear_bwd_tc(x.data_ptr(), K, w.data_ptr(), dz.data_ptr(), N, None, 0, None,
                                               dw.data_ptr(), db.data_ptr(), M, K, N, sp))
    mb = M * 4 / 1e6
    print(f"K={K:3d} N={N:3d}: fwd {t_fwd:7.1f} us ({mb * (K + N) / t_fwd:5.0f} GB/s)  fwd+bits {t_fwdb:7.1f}  "
          f"dx(float mask) {t_dx:7.1f} ({mb * (N + 2 * K) / t_dx:5.0f} GB/s)  dx(bits) {t_dxb:7.1f} "
          f"({mb * (N + K) / t_dxb:5.0f} GB/s)  dw {t_dw:7.1f} ({mb * (N + K) / t_dw:5.0f} GB/s)", flush=True)
