"""How much would re-ordering the compacted foreground stream help the radiance kernel?
Times fv_gather_probe (the gather stage alone) and fv_field_fwd with the residual stage off
(k_radiance_tc alone) on the config-2 frame's real x_final stream in four orders:
  march     -- the march's own order (tile = 8x4 pixels x 4 depths, what the renderer ships)
  morton    -- globally sorted by a 30-bit Morton key of the hash-normalised x_final
  tile1024  -- Morton-sorted inside each run of 1024 samples (a per-tile sort the march
               could do in shared memory)
  shuffled  -- a random permutation (no coherence at all)
The sort itself is not timed (this bounds the gain; a real sort would have to pay for itself).
Usage: python tools/order_probe.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16541_b200 import _lib, scene as psc  # noqa: E402
from paper_2306_16541_b200.model import FreeviewModel  # noqa: E402
from paper_2306_16541_b200.render import RenderSettings, Renderer, camera_struct, march_struct  # noqa: E402


def spread10(v):
    v = v & 0x3FF
    v = (v | (v << 16)) & 0x030000FF
    v = (v | (v << 8)) & 0x0300F00F
    v = (v | (v << 4)) & 0x030C30C3
    v = (v | (v << 2)) & 0x09249249
    return v


def rigid_weights(sc, width=0.15):
    """Near one-hot W^c: each canonical grid cell belongs to its nearest rest joint (a
    sharp softmax of -d^2 / width^2), the shape a trained / prior-initialised volume has;
    the seeded uniform logits instead blend all 24 bone transforms everywhere, which
    contracts the canonical point cloud."""
    sk = sc.skeleton
    k = len(sk.parent)
    joints = np.zeros((k, 3))
    for i in range(k):
        joints[i] = sk.rest_offset[i] + (joints[sk.parent[i]] if i > 0 else 0.0)
    g = sc.cfg.vol_res
    c = (np.arange(g) + 0.5) / g * 2.0 - 1.0
    gx, gy, gz = np.meshgrid(c, c, c, indexing="ij")
    pts = np.stack([gx, gy, gz], -1).reshape(-1, 3)
    d2 = ((pts[:, None, :] - joints[None]) ** 2).sum(-1)             # (G^3, k)
    lg = np.concatenate([-d2 / width ** 2, np.full((pts.shape[0], 1), -50.0)], 1)
    sc.vol_logits = np.ascontiguousarray(lg.T.reshape(k + 1, g, g, g).astype(np.float32))
    return sc


def main():
    dev = torch.device("cuda")
    sc = psc.make_scene(psc.config("c2"))
    if "--rigid" in sys.argv:
        sc = rigid_weights(sc)
    if "--small-offset" in sys.argv:    # trained-size residual offsets (SPEC:300 zero-inits the last layer)
        sc.off_w[-1] = sc.off_w[-1] * 0.01
    nets = FreeviewModel(sc)
    st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
    rnd = Renderer()
    lib, sp = nets.lib, torch.cuda.current_stream().cuda_stream
    pix = rnd.pixel_order(sc.camera)
    r = pix.numel()
    S = (r + 31) // 32 * 32 * st.n_samples
    occ = rnd.build_occupancy(nets, st) if st.occupancy else None
    lik, delta = torch.empty(S, device=dev), torch.empty(S, device=dev)
    xsc, idx = torch.empty((S, 4), device=dev), torch.empty(S, dtype=torch.int32, device=dev)
    nfg = torch.zeros(1, dtype=torch.int32, device=dev)
    m, cs, w = march_struct(st, pix, occ), camera_struct(sc.camera), nets.warp_struct()
    _lib.check(lib.fv_march_compact(C.byref(cs), C.byref(m), C.byref(w), r, lik.data_ptr(), delta.data_ptr(),
                                    xsc.data_ptr(), idx.data_ptr(), nfg.data_ptr(), None, None, sp))
    n = int(nfg.item())
    xf = torch.empty((n, 4), device=dev)
    f, h = nets.field_struct(), nets.hash_struct()
    _lib.check(lib.fv_residual_offset(C.byref(f), xsc.data_ptr(), n, st.eps_w, xf.data_ptr(), sp))
    del lik, delta, idx
    cmin = torch.tensor(list(h.cmin), device=dev)
    cinv = torch.tensor(list(h.cinv), device=dev)

    def q_norm(p):
        return ((p[:, :3] - cmin) * cinv).clamp(0, 1)

    def morton(p):
        q = (q_norm(p) * 1023).long()
        return spread10(q[:, 0]) | (spread10(q[:, 1]) << 1) | (spread10(q[:, 2]) << 2)
    key = morton(xf)
    kskel = morton(xsc[:n])
    xsc_n = xsc[:n]
    for b in (30, 24, 18):
        print(f"distinct cells at {1 << (b // 3)}^3: {torch.unique(key >> (30 - b)).numel() / n:.4f} per sample", flush=True)
    lo, hi = torch.quantile(q_norm(xf)[::97], torch.tensor([0.01, 0.99], device=dev), dim=0)
    raw = (xf[:, :3] - cmin) * cinv
    outside = ((raw < 0) | (raw > 1)).any(dim=1).float().mean().item()
    print(f"x_final outside the hash box (clamped to a face): {outside:.4f} of samples", flush=True)
    print("x_final normalised 1-99% range per axis:", lo.tolist(), hi.tolist(), flush=True)
    k32 = key.int()
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.sort(k32)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"torch.sort of {n} int32 Morton keys (+ int64 indices): {np.median(ts[1:]):.3f} ms", flush=True)
    orders = {"march": None, "morton": torch.argsort(key)}
    for bits in (21,):    # stable counting-sort-like buckets of 2^(bits/3) per axis on x_skel
        orders[f"bucket{1 << (bits // 3)}_xskel"] = torch.sort(kskel >> (30 - bits), stable=True).indices
    for bits in (15, 18, 21, 24):    # the same on x_final
        orders[f"bucket{1 << (bits // 3)}_xfinal"] = torch.sort(key >> (30 - bits), stable=True).indices
    res_off = (xf[:, :3] - xsc_n[:, :3]).norm(dim=1)
    print("residual offset |x_final - x_skel| quantiles 50/90/99%:",
          torch.quantile(res_off[::97], torch.tensor([0.5, 0.9, 0.99], device=dev)).tolist(), flush=True)
    inside = ~((raw < 0) | (raw > 1)).any(dim=1)
    kin = key.clone()
    kin[~inside] = (1 << 30) + torch.arange(int((~inside).sum().item()), device=dev)   # clamped ones last, march order
    orders["morton_inside_only"] = torch.argsort(kin)
    for c in (1024,):
        nt = n // c * c
        kt = key[:nt].view(-1, c)
        loc = torch.argsort(kt, dim=1) + torch.arange(0, nt, c, device=dev).view(-1, 1)
        orders[f"chunk{c}"] = torch.cat([loc.view(-1), torch.arange(nt, n, device=dev)])
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    orders["shuffled"] = torch.randperm(n, device=dev, generator=g)
    sink = torch.empty(256 * 148 * 8, device=dev)
    f0 = nets.field_struct()
    f0.offset_enabled = 0
    rgbs = torch.empty((n, 4), device=dev)
    out = {"samples": n}
    for name, o in orders.items():
        x = xf if o is None else xf[o].contiguous()
        res = {}
        for what in ("gather_probe", "radiance"):
            ts = []
            for _ in range(6):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                if what == "gather_probe":
                    _lib.check(lib.fv_gather_probe(C.byref(h), x.data_ptr(), n, 0, sink.data_ptr(), sink.numel(), sp))
                else:
                    _lib.check(lib.fv_field_fwd(C.byref(f0), C.byref(h), x.data_ptr(), n, st.eps_w,
                                                rgbs.data_ptr(), None, None, 0, sp))
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[what + "_ms"] = round(float(np.median(ts[1:])), 4)
        out[name] = res
        print(name, res, flush=True)
    print(out)


if __name__ == "__main__":
    main()
