"""Debug: k_dw on tiny inputs vs numpy (prints the mismatch pattern)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib
lib = _lib.load()
np.set_printoptions(linewidth=200, precision=3, suppress=True)
for (m, k, n, kind) in [(32, 8, 8, "ones"), (32, 32, 32, "ramp"), (64, 39, 128, "rand"), (3000, 39, 128, "rand")]:
    if kind == "ones":
        x = np.ones((m, k), np.float32); dz = np.ones((m, n), np.float32)
    elif kind == "ramp":
        x = np.tile(np.arange(k, dtype=np.float32), (m, 1)); dz = np.tile(np.arange(n, dtype=np.float32) * 0 + 1, (m, 1))
        dz[:, 0] = np.arange(m)
    else:
        rng = np.random.default_rng(0); x = rng.normal(size=(m, k)).astype(np.float32); dz = rng.normal(size=(m, n)).astype(np.float32)
    xt = torch.from_numpy(x).cuda(); zt = torch.from_numpy(dz).cuda()
    dw = torch.zeros((k, n), device="cuda"); db = torch.zeros(n, device="cuda")
    _lib.check(lib.fv_linear_bwd_tc(xt.data_ptr(), k, xt.data_ptr(), zt.data_ptr(), n, None, 0, None,
                                    dw.data_ptr(), db.data_ptr(), m, k, n, _lib.stream_ptr()))
    torch.cuda.synchronize()
    got, ref = dw.cpu().numpy(), x.T.astype(np.float64) @ dz
    print(kind, m, k, n, "dw err", np.abs(got - ref).max(), "max ref", np.abs(ref).max(), "db err",
          np.abs(db.cpu().numpy() - dz.sum(0)).max())
    if kind != "rand":
        print("got\n", got[:8, :8]); print("ref\n", ref[:8, :8]); print("db", db.cpu().numpy()[:8])
