"""Inverse-LBS skeleton warp (oracle).

* ``softmax0`` / ``softmax0_bwd``: channel softmax of the weight-volume logits (``ad:711-721``).
* ``sample_bone_channels`` / ``sample_bone_channels_bwd``: channel ``i`` of the volume
  sampled trilinearly at ``pts[i]`` (``ad:728-808``): box-corner-aligned grid with
  ``scale = (G-1)/(bmax-bmin)`` (``ad:746``); ``u = (p-bmin)*scale + 1`` into a one-voxel
  zero-padded grid (``ad:748-756``); inside iff every ``u`` in ``[0, G+1]`` (``ad:750``);
  ``i0 = clip(floor u, 0, G)`` (``ad:751-752``); 8-corner blend accumulated in (a,b,c)
  loop order (``ad:767-773``); index order ``vol[ch, x, y, z]`` (``ad:770``).
* ``skeleton_warp``: ``S:327-336`` / Eqs 7-9 -- ``p_i = G_i(x)``, ``w_i`` sampled,
  ``L = sum_i w_i`` over bones only, foreground iff ``L > eps_w`` (1e-4, ``S:373``),
  ``x_skel = sum_i (w_i/L) p_i`` (``weighted_sum0``, ``ad:456-467``), evaluated as
  ``(sum_i w_i p_i) / L`` (same value, the kernel's rounding order).

Every function takes a ``dtype``.  float64 follows the reference's formulas and op order
(``ad:748-773``, ``sk:171-172``).  float32 is the sm_100a kernel's specification: every
op is one rounded float32 op in the kernel's order, and the kernel uses fused
multiply-adds (one rounding) for ``p = R x + t``, ``u = (p - bmin) scale + 1``, the
trilinear blend (written as seven lerps ``v0 + f (v1 - v0)``, the same polynomial as
``ad:767-773``) and the ``sum_i w_i p_i`` accumulation.  ``fma32`` restates a
single-rounded float32 FMA: the float32 product is exact in x87 extended precision (48 of
64 mantissa bits), so only the final rounding to float32 is visible (a double-rounding
tie needs 40 trailing bits to line up, ~2^-40 per op).  Per-bone weights, the likelihood
and the foreground mask therefore compare bit-exactly with the kernel.
"""

from __future__ import annotations

import numpy as np

EPS_W = 1e-4


_XP = np.longdouble
assert np.finfo(_XP).nmant >= 63, "fma32 needs x87 extended precision (x86-64 long double)"


# True (parity): fma32 rounds once, bit-exact with the kernel.  bench.py's CPU-baseline
# workers set it False: plain float32 numpy (a*b, then + c) -- the speed a straightforward
# float32 port of the reference algorithm runs at, without the x87 emulation cost.
EXACT_FMA = True


def fma32(a, b, c):
    """float32 a*b + c with a single rounding (CUDA ``__fmaf_rn``)."""
    if not EXACT_FMA:
        return np.asarray(a, np.float32) * np.asarray(b, np.float32) + np.asarray(c, np.float32)
    return (np.asarray(a, np.float32).astype(_XP) * np.asarray(b, np.float32).astype(_XP)
            + np.asarray(c, np.float32).astype(_XP)).astype(np.float32)


def _lerp32(v0, v1, f):
    """v0 + f*(v1 - v0) as the kernel evaluates it: fma(f, v1 - v0, v0)."""
    return fma32(f, (v1 - v0).astype(np.float32), v0)


def softmax0(a):
    z = a - a.max(axis=0, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=0, keepdims=True)


def softmax0_bwd(out, g):
    dot = (g * out).sum(axis=0, keepdims=True)
    return out * (g - dot)


def _grid_coords(p, gsz, bmin, scale, dt):
    if dt is np.float32:
        u = fma32((p - bmin).astype(dt), np.broadcast_to(scale, p.shape), np.float32(1.0))
    else:
        u = (((p - bmin).astype(dt) * scale).astype(dt) + dt(1.0)).astype(dt)
    inside = np.all((u >= 0.0) & (u <= dt(gsz + 1)), axis=-1)
    i0 = np.clip(np.floor(u), 0, gsz).astype(np.int64)
    f = (u - i0.astype(dt)).astype(dt)
    return u, inside, i0, f


def sample_bone_channels(vol, pts, box_min, box_max, dtype=None):
    """vol (C,G,G,G), pts (K,N,3) -> (K,N) (ad:728-773)."""
    dt = np.dtype(dtype or vol.dtype).type
    v = np.asarray(vol, dtype=dt)
    p = np.asarray(pts, dtype=dt)
    kb = p.shape[0]
    gsz = v.shape[1]
    bmin = np.asarray(box_min, dtype=dt)
    scale = ((dt(gsz) - dt(1.0)) / (np.asarray(box_max, dtype=dt) - bmin)).astype(dt)
    _, inside, i0, f = _grid_coords(p, gsz, bmin, scale, dt)
    vp = np.zeros((v.shape[0],) + tuple(g + 2 for g in v.shape[1:]), dtype=dt)
    vp[:, 1:-1, 1:-1, 1:-1] = v
    ch = np.arange(kb).reshape(kb, 1)
    wx = ((dt(1.0) - f[..., 0]).astype(dt), f[..., 0])
    wy = ((dt(1.0) - f[..., 1]).astype(dt), f[..., 1])
    wz = ((dt(1.0) - f[..., 2]).astype(dt), f[..., 2])
    ix, iy, iz = i0[..., 0], i0[..., 1], i0[..., 2]
    if dt is np.float32:
        cv = [vp[ch, ix + a, iy + b, iz + c] for a in (0, 1) for b in (0, 1) for c in (0, 1)]
        fx, fy, fz = f[..., 0], f[..., 1], f[..., 2]
        c00, c01 = _lerp32(cv[0], cv[1], fz), _lerp32(cv[2], cv[3], fz)
        c10, c11 = _lerp32(cv[4], cv[5], fz), _lerp32(cv[6], cv[7], fz)
        out = _lerp32(_lerp32(c00, c01, fy), _lerp32(c10, c11, fy), fx)
        return np.where(inside, out, dt(0.0)).astype(dt)
    out = np.zeros(p.shape[:2], dtype=dt)
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                cv = vp[ch, ix + a, iy + b, iz + c]
                wgt = ((wx[a] * wy[b]).astype(dt) * wz[c]).astype(dt)
                out = (out + (wgt * cv).astype(dt)).astype(dt)
    return np.where(inside, out, dt(0.0)).astype(dt)


def sample_bone_channels_bwd(vol_shape, pts, box_min, box_max, g, dtype=np.float64,
                             vol=None):
    """Gradients (dvol (C,G,G,G), dpts (K,N,3) or None) of ``sum(g * out)`` (ad:775-806)."""
    dt = np.dtype(dtype).type
    p = np.asarray(pts, dtype=dt)
    kb, n, _ = p.shape
    gsz = vol_shape[1]
    bmin = np.asarray(box_min, dtype=dt)
    scale = ((dt(gsz) - dt(1.0)) / (np.asarray(box_max, dtype=dt) - bmin)).astype(dt)
    _, inside, i0, f = _grid_coords(p, gsz, bmin, scale, dt)
    gm = np.asarray(g, dtype=dt) * inside
    gp = gsz + 2
    flat = np.zeros(vol_shape[0] * gp ** 3, dtype=np.float64)
    ch = np.arange(kb).reshape(kb, 1)
    wx = (1.0 - f[..., 0], f[..., 0])
    wy = (1.0 - f[..., 1], f[..., 1])
    wz = (1.0 - f[..., 2], f[..., 2])
    ix, iy, iz = i0[..., 0], i0[..., 1], i0[..., 2]
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                idx = ((ch * gp + ix + a) * gp + iy + b) * gp + iz + c
                flat += np.bincount(idx.ravel(), weights=(wx[a] * wy[b] * wz[c] * gm).ravel(),
                                    minlength=flat.size)
    dvol = flat.reshape(vol_shape[0], gp, gp, gp)[:, 1:-1, 1:-1, 1:-1].astype(dt)
    dpts = None
    if vol is not None:
        vp = np.zeros((vol_shape[0], gp, gp, gp), dtype=dt)
        vp[:, 1:-1, 1:-1, 1:-1] = vol
        gx = np.zeros((kb, n), dtype=dt)
        gy = np.zeros((kb, n), dtype=dt)
        gz = np.zeros((kb, n), dtype=dt)
        for a in (0, 1):
            for b in (0, 1):
                for c in (0, 1):
                    cv = vp[ch, ix + a, iy + b, iz + c]
                    sx, sy, sz = (1.0 if a else -1.0), (1.0 if b else -1.0), (1.0 if c else -1.0)
                    gx += sx * wy[b] * wz[c] * cv
                    gy += wx[a] * sy * wz[c] * cv
                    gz += wx[a] * wy[b] * sz * cv
        dpts = np.stack([gx * gm * scale[0], gy * gm * scale[1], gz * gm * scale[2]], axis=-1)
    return dvol, dpts


def bone_points(x, g_r, g_t, dtype=np.float32):
    """p_i = x @ R_i^T + t_i for every bone, (K,N,3), kernel op order.

    float32: ``fma(R2, x2, fma(R1, x1, R0*x0)) + t`` per row (the kernel's FMA chain).
    """
    dt = np.dtype(dtype).type
    x = np.asarray(x, dtype=dt)
    r = np.asarray(g_r, dtype=dt)
    t = np.asarray(g_t, dtype=dt)
    out = np.empty((r.shape[0], x.shape[0], 3), dtype=dt)
    if dt is np.float32:
        for j in range(3):
            acc = (r[:, j, 0][:, None] * x[None, :, 0]).astype(dt)
            acc = fma32(r[:, j, 1][:, None], x[None, :, 1], acc)
            acc = fma32(r[:, j, 2][:, None], x[None, :, 2], acc)
            out[:, :, j] = (acc + t[:, j][:, None]).astype(dt)
        return out
    for j in range(3):
        acc = (r[:, j, 0][:, None] * x[None, :, 0]).astype(dt)
        acc = (acc + (r[:, j, 1][:, None] * x[None, :, 1]).astype(dt)).astype(dt)
        acc = (acc + (r[:, j, 2][:, None] * x[None, :, 2]).astype(dt)).astype(dt)
        out[:, :, j] = (acc + t[:, j][:, None]).astype(dt)
    return out


def skeleton_warp(x, g_r, g_t, vol, box_min, box_max, eps_w=EPS_W, dtype=np.float32):
    """Returns dict(x_skel (N,3), L (N), fg (N) bool, w (K,N), p (K,N,3)).

    ``vol`` has C >= K channels; only channels ``0..K-1`` are sampled (``ad:757``).
    Background samples (``L <= eps_w``) get ``x_skel = 0`` (unused downstream).
    """
    dt = np.dtype(dtype).type
    k = g_r.shape[0]
    p = bone_points(x, g_r, g_t, dtype)
    w = sample_bone_channels(np.asarray(vol, dtype=dt)[:k], p, box_min, box_max, dtype)
    lik = np.zeros(x.shape[0], dtype=dt)
    for i in range(k):
        lik = (lik + w[i]).astype(dt)
    fg = lik > dt(eps_w)
    safe = np.where(fg, lik, dt(1.0)).astype(dt)
    # sum_i (w_i/L) p_i evaluated as (sum_i w_i p_i) / L -- the kernel's order
    acc = np.zeros((x.shape[0], 3), dtype=dt)
    for i in range(k):
        if dt is np.float32:
            acc = fma32(w[i][:, None], p[i], acc)
        else:
            acc = (acc + (w[i][:, None] * p[i]).astype(dt)).astype(dt)
    xs = (acc / safe[:, None]).astype(dt)
    xs = np.where(fg[:, None], xs, dt(0.0)).astype(dt)
    return {"x_skel": xs, "L": lik, "fg": fg, "w": w, "p": p}


def skeleton_warp_bwd(warp, d_xskel, vol_shape, box_min, box_max, dtype=np.float64):
    """d x_skel (N,3) -> d vol (C,G,G,G) through Eq 9 and the trilinear sampler.

    ``dw_i = <d x_skel, p_i - x_skel> / L`` on foreground samples; the likelihood gate
    of the compositor is flat there (``clamp(L/eps_w,0,1) = 1``) so L receives none.
    """
    fg = warp["fg"]
    lik = np.where(fg, warp["L"], 1.0).astype(np.float64)
    p = warp["p"].astype(np.float64)
    xs = warp["x_skel"].astype(np.float64)
    g = np.asarray(d_xskel, np.float64) * fg[:, None]
    dw = np.einsum("nd,knd->kn", g, p - xs[None]) / lik[None]
    k = p.shape[0]
    dvol_k, _ = sample_bone_channels_bwd((k,) + tuple(vol_shape[1:]), p, box_min, box_max, dw,
                                         dtype=dtype)
    dvol = np.zeros(vol_shape, dtype=dtype)
    dvol[:k] = dvol_k
    return dvol


def skeleton_warp_bwd_g(warp, x, d_xskel, vol, box_min, box_max):
    """d x_skel (N,3) -> (d G_r (K,3,3), d G_t (K,3)): the gradient into the motion bases
    (SURVEY §8a A4).  With p_i = G_i(x) = R_i x + t_i, x_skel = sum_i (w_i / L) p_i and
    w_i = trilinear(W^c_i, p_i) (``ad:728-808``):
    ``dL/dp_i = (w_i / L) g + dw_i * dw_i/dp_i`` with ``dw_i = <g, p_i - x_skel> / L``, then
    ``dR_i = sum_n dp_i x^T`` and ``dt_i = sum_n dp_i`` (float64; pinned to the reference's
    Tape through ``bmm`` / ``sample_bone_channels`` / ``weighted_sum0``, golden ``wg_*``)."""
    fg = warp["fg"]
    lik = np.where(fg, warp["L"], 1.0).astype(np.float64)
    p = warp["p"].astype(np.float64)
    xs = warp["x_skel"].astype(np.float64)
    w = warp["w"].astype(np.float64)
    g = np.asarray(d_xskel, np.float64) * fg[:, None]
    dw = np.einsum("nd,knd->kn", g, p - xs[None]) / lik[None]
    k = p.shape[0]
    vol = np.asarray(vol, np.float64)
    _, dpts = sample_bone_channels_bwd((k,) + vol.shape[1:], p, box_min, box_max, dw, dtype=np.float64,
                                       vol=vol[:k])
    dp = (w / lik[None])[:, :, None] * g[None] + dpts
    xx = np.asarray(x, np.float64)
    return np.einsum("kna,nb->kab", dp, xx), dp.sum(axis=1)
