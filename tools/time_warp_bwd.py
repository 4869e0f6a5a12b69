"""Time fv_warp_bwd at config-3 scale on the trainer's own inputs (tuning helper)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib  # noqa: E402
from paper_2306_16541_b200 import scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings  # noqa: E402
from paper_2306_16541_b200.train import Trainer  # noqa: E402

sc = psc.make_scene(psc.config("c3"))
nets = FreeviewModel(sc)
target, mask = psc.target_image(sc)
tr = Trainer(nets, sc.camera, target, mask, RenderSettings.from_config(sc.cfg, seed=1), n_patches=6, patch=32)
for i in range(3):
    tr.step(i)
torch.cuda.synchronize()
w = nets.warp_struct()
sp = _lib.stream_ptr()
dxs = torch.randn_like(tr.dxs) * 1e-3
dvol = torch.zeros_like(tr.dvol)


def run():
    _lib.check(nets.lib.fv_warp_bwd(C.byref(w), tr.st.eps_w, tr.x.data_ptr(), tr.S, dxs.data_ptr(), dvol.data_ptr(), sp))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
print(f"warp bwd: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
