"""A few config-3 training iterations (for ncu launch lists / profiling)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings  # noqa: E402
from paper_2306_16541_b200.train import Trainer  # noqa: E402

sc = psc.make_scene(psc.config("c3"))
nets = FreeviewModel(sc)
target, mask = psc.target_image(sc)
tr = Trainer(nets, sc.camera, target, mask, RenderSettings.from_config(sc.cfg, seed=1), n_patches=6, patch=32)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    tr.step(i)
torch.cuda.synchronize()
print("loss", tr.loss[0].item())
