"""Time one fv_field_fwd launch on a config-2 frame worth of samples (tuning helper).
Usage: FV_TC_VARIANT=2s python tools/time_field.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib, scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings, Renderer, camera_struct, march_struct  # noqa: E402

sc = psc.make_scene(psc.config("c2"))
nets = FreeviewModel(sc)
st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed, occupancy=False)
rnd = Renderer()
pix = rnd.pixel_order(sc.camera)
n = pix.numel()
S = n * st.n_samples
xs = torch.empty((S, 4), device="cuda")
delta = torch.empty(S, device="cuda")
rgbs = torch.empty((S, 4), device="cuda")
m, cs, w = march_struct(st, pix, None), camera_struct(sc.camera), nets.warp_struct()
h, f = nets.hash_struct(), nets.field_struct()
sp = torch.cuda.current_stream().cuda_stream
_lib.check(nets.lib.fv_march_warp(C.byref(cs), C.byref(m), C.byref(w), n, xs.data_ptr(), delta.data_ptr(), None, None, sp))
ts = []
for i in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(nets.lib.fv_field_fwd(C.byref(f), C.byref(h), xs.data_ptr(), S, 1e-4, rgbs.data_ptr(), None, None, 0, sp))
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"variant {os.environ.get('FV_TC_VARIANT', 'default')}: field {np.median(ts[1:]):.3f} ms  "
      f"({S * 121856 / (np.median(ts[1:]) * 1e-3) / 1e12:.1f} TFLOP/s)  checksum {rgbs.double().sum().item():.6e}")
