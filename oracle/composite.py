"""Front-to-back alpha compositing with likelihood gating (oracle).

Forward (``S:428-437``, Eq 3 ``P:64-69``, augmentation ``P:199``):
  ``a_i = 1 - exp(-sigma_i delta_i)``; ``abar_i = a_i * clamp(L_i/eps_w, 0, 1)``;
  ``T_0 = 1``, ``T_{i+1} = T_i (1 - abar_i)`` (exclusive scan, ``ad:815-826``);
  ``rgb = sum_i T_i abar_i c_i + T_stop * bg``; ``alpha = 1 - T_stop``.
Early termination (builder-defined, PARITY UNPINNED): sample ``i`` is composited only
while ``T_i >= eps_t``; ``T_stop`` is the transmittance at the first skipped sample (or
``T_N``).  ``eps_t = 0`` disables it.

Backward: division-free reverse scan in the spirit of ``ad:828-835``: with
``Q_N = bg``, ``Q_i = abar_i c_i + (1 - abar_i) Q_{i+1}`` and ``P_N = 1``,
``P_i = (1 - abar_i) P_{i+1}``:
``d rgb / d abar_i = T_i (c_i - Q_{i+1})`` and ``d alpha / d abar_i = T_i P_{i+1}``.
"""

from __future__ import annotations

import numpy as np

EPS_W = 1e-4


def composite(sigma, color, delta, lik, bg, eps_w=EPS_W, eps_t=0.0, dtype=np.float32):
    """sigma/delta/lik (R,N), color (R,N,3), bg (3,) -> dict(rgb, alpha, T, abar, active)."""
    dt = np.dtype(dtype).type
    sigma = np.asarray(sigma, dt)
    delta = np.asarray(delta, dt)
    a = (dt(1.0) - np.exp((-(sigma * delta)).astype(dt)).astype(dt)).astype(dt)
    gate = np.clip((np.asarray(lik, dt) / dt(eps_w)).astype(dt), dt(0.0), dt(1.0))
    abar = (a * gate).astype(dt)
    r, n = sigma.shape
    t = np.empty((r, n + 1), dtype=dt)
    t[:, 0] = 1.0
    for i in range(n):
        t[:, i + 1] = (t[:, i] * (dt(1.0) - abar[:, i]).astype(dt)).astype(dt)
    active = t[:, :n] >= dt(eps_t) if eps_t > 0 else np.ones((r, n), dtype=bool)
    n_act = active.sum(axis=1)
    t_stop = t[np.arange(r), n_act]
    wgt = np.where(active, (t[:, :n] * abar).astype(dt), dt(0.0)).astype(dt)
    rgb = np.zeros((r, 3), dtype=dt)
    for i in range(n):
        rgb = (rgb + (wgt[:, i:i + 1] * np.asarray(color[:, i], dt)).astype(dt)).astype(dt)
    rgb = (rgb + (t_stop[:, None] * np.asarray(bg, dt)[None, :]).astype(dt)).astype(dt)
    alpha = (dt(1.0) - t_stop).astype(dt)
    return {"rgb": rgb, "alpha": alpha, "T": t, "abar": abar, "a": a, "active": active,
            "gate": gate}


def composite_bwd(out, sigma, color, delta, lik, bg, d_rgb, d_alpha, eps_w=EPS_W):
    """Gradients (d sigma (R,N), d color (R,N,3)) in float64; eps_t must have been 0."""
    t = out["T"].astype(np.float64)
    abar = out["abar"].astype(np.float64)
    a = out["a"].astype(np.float64)
    gate = out["gate"].astype(np.float64)
    color = np.asarray(color, np.float64)
    r, n = abar.shape
    d_rgb = np.asarray(d_rgb, np.float64)
    d_alpha = np.asarray(d_alpha, np.float64)
    q = np.broadcast_to(np.asarray(bg, np.float64), (r, 3)).copy()
    p = np.ones(r)
    d_abar = np.zeros((r, n))
    d_color = np.zeros((r, n, 3))
    for i in range(n - 1, -1, -1):
        d_abar[:, i] = t[:, i] * (np.sum(d_rgb * (color[:, i] - q), axis=1) + d_alpha * p)
        d_color[:, i] = (t[:, i] * abar[:, i])[:, None] * d_rgb
        q = abar[:, i:i + 1] * color[:, i] + (1.0 - abar[:, i:i + 1]) * q
        p = (1.0 - abar[:, i]) * p
    d_a = d_abar * gate
    d_sigma = d_a * np.asarray(delta, np.float64) * (1.0 - a)
    return d_sigma, d_color
