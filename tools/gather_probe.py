"""fv_gather_probe on the config-2 frame's real foreground x_final stream and on as many random
box points (one launch each), for ncu captures.  Usage: python tools/gather_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2306_16541_b200 import scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings, Renderer  # noqa: E402

sc = psc.make_scene(psc.config("c2"))
nets = FreeviewModel(sc)
st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
print(bench.gather_rates(nets, Renderer(), sc.camera, st, torch.device("cuda"), reps=0))  # 1 launch per mode
