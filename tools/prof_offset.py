"""Timeline of k_offset_tc from an FV_OFF_PROF=1 build (tools/build_alt.sh prof -DFV_OFF_PROF=1,
copied over libfvcuda.so): clock64 at 10 points per tile for CTA 0's two teams.
Usage: python tools/prof_offset.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib, scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings, Renderer  # noqa: E402

sc = psc.make_scene(psc.config("c2"))
nets = FreeviewModel(sc)
st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
rnd = Renderer()
for _ in range(2):
    rnd.render_image(nets, sc.camera, None, st)
torch.cuda.synchronize()
buf = (C.c_longlong * (2 * 32 * 10))()
lib = _lib.load()
assert lib.fv_debug_offset_prof(buf) == 0
a = np.frombuffer(buf, dtype=np.int64).reshape(2, 32, 10).astype(np.float64)
names = ["B0 issue+wait (L4 prev + L0)", "emit", "epi0", "L1 issue+wait (+posenc next)", "epi1", "L2 issue+wait",
         "epi2", "L3 issue+wait", "epi3", "-> next tile"]
t0 = a[:, :, 0].min()
for team in range(2):
    d = np.diff(a[team, 4:28], axis=1)             # steady-state tiles
    nxt = a[team, 5:29, 0] - a[team, 4:28, 9]
    print(f"team {team}: tile period {np.mean(np.diff(a[team, 4:28, 0])):.0f} cycles")
    for k in range(9):
        print(f"   {names[k]:32s} {d[:, k].mean():7.0f}")
    print(f"   {names[9]:32s} {nxt.mean():7.0f}")
print("team 1 start offset vs team 0 (cycles):", a[1, 4:10, 0] - a[0, 4:10, 0])
