"""Config-3 training it/s as bench.py measures it (device time of N steps after 3 warm-up)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings  # noqa: E402
from paper_2306_16541_b200.train import Trainer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sc = psc.make_scene(psc.config("c3"))
nets = FreeviewModel(sc)
target, mask = psc.target_image(sc)
tr = Trainer(nets, sc.camera, target, mask, RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed), n_patches=6,
             patch=32, seed=1000)
for i in range(3):
    tr.step(i)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(2_000_000)
a.record()
for i in range(n):
    tr.step(3 + i)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / n
print(f"train {ms:.3f} ms/it  {1000 / ms:.1f} it/s  loss {tr.loss[0].item():.5f}")
