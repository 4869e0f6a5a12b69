"""Occupancy-grid rebuild of the config-2 model, timed (CUDA events) and launched a few
times for ncu launch lists.  Usage: python tools/time_occ.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings, Renderer  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sc = psc.make_scene(psc.config("c2"))
nets = FreeviewModel(sc)
st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
rnd = Renderer()
for _ in range(3):
    rnd.build_occupancy(nets, st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    rnd.build_occupancy(nets, st)
b.record()
torch.cuda.synchronize()
print(f"occupancy build {a.elapsed_time(b) / reps:.4f} ms")
