"""Stage times of the C2 render path (tuning helper), optionally with the fp32 copy of the
(fp16-valued) hash table instead of the fp16 one.
Usage: python tools/time_stages.py [--fp32-table] [--reps 7]"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib, scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings, Renderer, camera_struct, march_struct  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--fp32-table", action="store_true")
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--config", default="c2")
ap.add_argument("--no-occ", action="store_true")
ap.add_argument("--opaque", action="store_true", help="scene.opaque_subject body density")
ap.add_argument("--eps-t", type=float, default=0.0)
ap.add_argument("--round", type=int, default=32)
a = ap.parse_args()

sc = psc.make_scene(psc.config(a.config))
if a.opaque:
    sc = psc.opaque_subject(sc)
nets = FreeviewModel(sc)
st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed, eps_t=a.eps_t, round_samples=a.round)
rnd = Renderer()
cam = sc.camera
pix = rnd.pixel_order(cam)
n = pix.numel()
occ = None if a.no_occ else rnd.build_occupancy(nets, st)
m, cs, w = march_struct(st, pix, occ, True), camera_struct(cam), nets.warp_struct()
h = nets.hash_struct(nets.views["table"] if a.fp32_table else None)
f = nets.field_struct()
rgb = torch.empty((n, 3), device="cuda")
alpha = torch.empty(n, device="cuda")
wb = nets.lib.fv_render_workspace_bytes(n, st.n_samples, f.precision)
work = torch.empty(wb, dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
rows, nfg = [], C.c_int64(0)
for _ in range(a.reps):
    t = (C.c_float * 5)()
    _lib.check(nets.lib.fv_render_fwd_timed(C.byref(cs), C.byref(m), C.byref(w), C.byref(h), C.byref(f), n,
                                            work.data_ptr(), wb, rgb.data_ptr(), alpha.data_ptr(), t,
                                            C.byref(nfg), sp))
    rows.append(list(t))
med = np.median(np.array(rows)[1:], axis=0)
print(f"table {'fp32' if a.fp32_table else 'fp16'}: march {med[0]:.3f}  offset {med[1]:.3f}  radiance {med[2]:.3f}  "
      f"composite {med[3]:.3f}  total {med[4]:.3f} ms  ({1e3 / med[4]:.1f} fps)  fg {nfg.value}  "
      f"checksum {rgb.double().sum().item():.6e}")
