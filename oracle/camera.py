"""Camera rays, ray/box slab test and stratified sampling (oracle).

``orbit_camera`` / ``look_at`` / ``rays_f64`` restate the reference camera model
(``cap:40-142``): pinhole intrinsics, world-to-camera ``[R|t]``, pixel centres at
``+0.5``, row-major pixel order, ``d = normalize((K^-1 [u,v,1]) @ R)``, ``o = -R^T t``.

The ``*_f32`` functions are the bit-exact float32 restatement of what the sm_100a
ray-march kernel computes: every product and sum is one IEEE-rounded float32 operation
in the order written here (the kernel uses ``__fmul_rn``/``__fadd_rn`` in the same
order), so per-ray sample counts and occupancy skip masks compare bit-exactly.

Sampling definition (SPEC ``S:410-418``, gaps filled by the builder -- PARITY UNPINNED):
* slab test against the observation-space box, near plane 0; miss => zero samples;
* ``N`` equal bins over ``[t_enter, t_exit]``; sample ``i`` at ``t_enter + (i+u_i)*step``
  with ``u_i = 0.5`` (uniform, config 1) or ``u_i = jitter_u(seed, pixel, i)``;
* spacing ``delta_i = t_{i+1} - t_i`` (``S:401``) for ``i < N-1``; the last sample gets
  ``(t_exit - t_{N-1}) + (t_0 - t_enter)`` so the spacings sum to ``t_exit - t_enter``.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32
U32 = np.uint32


# ---------------------------------------------------------------------------
# float64 reference camera (cap:113-142, cap:73-82)

def look_at(eye, target, up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """World-to-camera 4x4; camera +x right, +y down, +z forward (cap:113-129)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    x = np.cross(fwd, np.asarray(up, dtype=np.float64))
    x = x / np.linalg.norm(x)
    y = np.cross(fwd, x)
    y = y / np.linalg.norm(y)
    r = np.stack([x, y, fwd])
    m = np.eye(4)
    m[:3, :3] = r
    m[:3, 3] = -r @ eye
    return m


def orbit_camera(target, yaw_deg, pitch_deg, radius, fov_deg, width, height):
    """``(K, world_to_camera)`` of a camera orbiting ``target`` (cap:132-142)."""
    yaw, pitch = np.deg2rad(yaw_deg), np.deg2rad(pitch_deg)
    target = np.asarray(target, dtype=np.float64)
    eye = target + radius * np.array([np.sin(yaw) * np.cos(pitch), np.sin(pitch),
                                      np.cos(yaw) * np.cos(pitch)])
    f = 0.5 * height / np.tan(0.5 * np.deg2rad(fov_deg))
    k = np.array([[f, 0, width / 2.0], [0, f, height / 2.0], [0, 0, 1.0]])
    return k, look_at(eye, target)


def rays_f64(k, w2c, width, height):
    """Per-pixel rays through pixel centres, row-major (cap:73-82)."""
    xs, ys = np.meshgrid(np.arange(width) + 0.5, np.arange(height) + 0.5)
    pix = np.stack([xs.ravel(), ys.ravel(), np.ones(width * height)], axis=1)
    rot = w2c[:3, :3]
    dirs = (pix @ np.linalg.inv(k).T) @ rot
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    center = -rot.T @ w2c[:3, 3]
    return np.broadcast_to(center, dirs.shape).copy(), dirs


# ---------------------------------------------------------------------------
# float32 kernel-order restatement

def camera_consts(k, w2c):
    """float32 constants the kernel receives: K^-1, R, camera centre (all from float64)."""
    rot = np.asarray(w2c, dtype=np.float64)[:3, :3]
    return {
        "kinv": np.linalg.inv(np.asarray(k, dtype=np.float64)).astype(F32),
        "rot": rot.astype(F32),
        "center": (-rot.T @ np.asarray(w2c, dtype=np.float64)[:3, 3]).astype(F32),
    }


def rays_f32(cc, pix, width):
    """Rays for linear pixel indices ``pix`` (row-major), float32 kernel order."""
    pix = np.asarray(pix, dtype=np.int64)
    px = ((pix % width).astype(F32) + F32(0.5)).astype(F32)
    py = ((pix // width).astype(F32) + F32(0.5)).astype(F32)
    ki, r = cc["kinv"], cc["rot"]
    dc = [((ki[i, 0] * px + ki[i, 1] * py) + ki[i, 2]).astype(F32) for i in range(3)]
    d = [((dc[0] * r[0, j] + dc[1] * r[1, j]) + dc[2] * r[2, j]).astype(F32) for j in range(3)]
    n = np.sqrt(((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]).astype(F32)).astype(F32)
    d = np.stack([(dj / n).astype(F32) for dj in d], axis=1)
    o = np.broadcast_to(cc["center"].astype(F32), d.shape).copy()
    return o, d


def slab_f32(o, d, bmin, bmax, near=0.0):
    """Ray/box slab test, float32 (fminf/fmaxf semantics: NaN operands are ignored)."""
    bmin = np.asarray(bmin, dtype=F32)
    bmax = np.asarray(bmax, dtype=F32)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = (F32(1.0) / d).astype(F32)
        t0 = ((bmin[None, :] - o) * inv).astype(F32)
        t1 = ((bmax[None, :] - o) * inv).astype(F32)
    tn = np.fmin(t0, t1)
    tf = np.fmax(t0, t1)
    t_enter = np.fmax(np.fmax(np.fmax(tn[:, 0], tn[:, 1]), tn[:, 2]), F32(near)).astype(F32)
    t_exit = np.fmin(np.fmin(tf[:, 0], tf[:, 1]), tf[:, 2]).astype(F32)
    hit = t_exit > t_enter
    return t_enter, t_exit, hit


def hash_u32(seed, pix, i):
    """Counter hash (seed, pixel, sample) -> uint32 (a 32-bit integer finaliser)."""
    pix = np.asarray(pix, dtype=np.uint64).astype(U32)
    i = np.asarray(i, dtype=np.uint64).astype(U32)
    with np.errstate(over="ignore"):
        h = U32(seed) ^ (pix * U32(0x9E3779B1)) ^ ((i + U32(1)) * U32(0x85EBCA77))
        h = h ^ (h >> U32(16))
        h = h * U32(0x7FEB352D)
        h = h ^ (h >> U32(15))
        h = h * U32(0x846CA68B)
        h = h ^ (h >> U32(16))
    return h.astype(U32)


def jitter_u(seed, pix, i):
    """Uniform in [0,1) with 24 random bits (exact in float32)."""
    return ((hash_u32(seed, pix, i) >> U32(8)).astype(F32) * F32(2.0 ** -24)).astype(F32)


def stratified_f32(t_enter, t_exit, hit, pix, n_samples, jitter, seed):
    """Sample depths (R,N), spacings (R,N) and per-ray sample counts (R,) in float32."""
    r = t_enter.shape[0]
    nf = F32(n_samples)
    step = ((t_exit - t_enter) / nf).astype(F32)
    ii = np.arange(n_samples, dtype=np.int64)
    if jitter:
        u = jitter_u(seed, np.asarray(pix)[:, None], ii[None, :])
    else:
        u = np.full((r, n_samples), F32(0.5), dtype=F32)
    s = (ii[None, :].astype(F32) + u).astype(F32)
    t = (t_enter[:, None] + (s * step[:, None]).astype(F32)).astype(F32)
    delta = np.empty_like(t)
    delta[:, :-1] = (t[:, 1:] - t[:, :-1]).astype(F32)
    delta[:, -1] = ((t_exit - t[:, -1]).astype(F32) + (t[:, 0] - t_enter).astype(F32)).astype(F32)
    count = np.where(hit, n_samples, 0).astype(np.int32)
    return t, delta, count


def positions_f32(o, d, t):
    """x = o + t d per component (two rounded float32 ops)."""
    return (o[:, None, :] + (t[:, :, None] * d[:, None, :]).astype(F32)).astype(F32)


# ---------------------------------------------------------------------------
# Occupancy grid lookup (32^3 bitfield over the observation box) -- PARITY UNPINNED

OCC_RES = 32


def occ_scale(bmin, bmax):
    return (OCC_RES / (np.asarray(bmax, np.float64) - np.asarray(bmin, np.float64))).astype(F32)


def occ_cell(x, bmin, scale):
    """Linear x-major cell index of float32 points (..., 3)."""
    bmin = np.asarray(bmin, dtype=F32)
    q = np.floor(((x - bmin).astype(F32) * scale).astype(F32))
    c = np.clip(q, 0, OCC_RES - 1).astype(np.int64)
    return (c[..., 0] * OCC_RES + c[..., 1]) * OCC_RES + c[..., 2]


def occ_test(bits, cell):
    """bits: uint32[1024] bitfield; returns bool occupancy of ``cell``."""
    w = np.asarray(bits, dtype=U32)[cell >> 5]
    return ((w >> (cell & 31).astype(U32)) & U32(1)).astype(bool)
