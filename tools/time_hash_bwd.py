"""Time fv_hash_bwd at config-3 scale on the trainer's own inputs (tuning helper)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib  # noqa: E402
from paper_2306_16541_b200 import scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings  # noqa: E402
from paper_2306_16541_b200.train import Trainer  # noqa: E402
import ctypes as C  # noqa: E402

sc = psc.make_scene(psc.config("c3"))
nets = FreeviewModel(sc)
target, mask = psc.target_image(sc)
tr = Trainer(nets, sc.camera, target, mask, RenderSettings.from_config(sc.cfg, seed=1), n_patches=6, patch=32)
for i in range(3):
    tr.step(i)
torch.cuda.synchronize()
h = nets.hash_struct()
lib = nets.lib
sp = _lib.stream_ptr()
dfeat = torch.randn_like(tr.feat) * 1e-3
dt = torch.zeros_like(tr.gviews["table"])
dx = torch.empty_like(tr.xf)


def run():
    _lib.check(lib.fv_hash_bwd(C.byref(h), tr.xf.data_ptr(), tr.S, dfeat.data_ptr(), dt.data_ptr(), dx.data_ptr(), sp))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
print(f"hash bwd: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")


def run_fwd():
    _lib.check(lib.fv_hash_fwd(C.byref(h), tr.xf.data_ptr(), tr.S, tr.feat.data_ptr(), None, sp))


for _ in range(3):
    run_fwd()
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    run_fwd()
e1.record()
torch.cuda.synchronize()
print(f"hash fwd: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
