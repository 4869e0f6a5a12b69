"""Small end-to-end run of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): tiny config-1/2 renders, config-5 merge, one training step with every optional
stage (patch loss, generator, pose refiner), tensor-core and narrow layer ops."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.pose import PoseRefinerNet  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings, Renderer, render_scene  # noqa: E402
from paper_2306_16541_b200.train import Trainer  # noqa: E402
from paper_2306_16541_b200.weightnet import WeightVolumeNet  # noqa: E402

torch.cuda.set_device(0)
for name in ("c1", "c2"):
    sc = psc.make_scene(psc.config(name, width=32, height=32, n_samples=16))
    nets = FreeviewModel(sc)
    st = RenderSettings.from_config(sc.cfg, seed=1, occupancy=name == "c2", eps_t=1e-3)
    Renderer().render_image(nets, sc.camera, sc.poses[0], st)
ms = psc.make_multi_scene(psc.config("c5", width=32, height=32, n_samples=16, hash=psc.HashGridConfig(log2_T=14, max_res=128)),
                          n_subjects=2)
render_scene([FreeviewModel(s) for s in ms.subjects], ms)
sc = psc.make_scene(psc.config("c3", width=64, height=64, n_samples=16))
nets = FreeviewModel(sc)
target, mask = psc.target_image(sc)
st = RenderSettings.from_config(sc.cfg, seed=1)
tr = Trainer(nets, sc.camera, target, mask, st, n_patches=2, patch=16, lam_mse=0.2, lam_perc=1.0,
             weight_net=WeightVolumeNet(sc.cfg.n_bones + 1), pose_refiner=PoseRefinerNet(sc.cfg.n_bones),
             pose=sc.poses[0])
for i in range(2):
    tr.step(i)
torch.cuda.synchronize()
print("sanitize smoke ok", float(tr.loss[0]))
