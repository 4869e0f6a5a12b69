"""Patch loss of the training step -- TEST INFRASTRUCTURE (oracle).

SPEC ``compute_loss`` (``S:496-504``, Eq 14 ``P:225``): ``lam_mse * MSE + lam_perc * GD``
where the perceptual term is the SPEC's proxy (DESIGN DECISIONS, ``S:540``): the
multi-scale gradient difference ``GD = sum over scales {1, 2} of mean|d_x r - d_x t| +
mean|d_y r - d_y t|``, first differences as ``diff_axis`` (``ad:844-859``), scale 2 by
``avgpool2`` (``ad:862-873``), ``|.|`` with ``sign(0) = 0`` in the backward (``absval``
``ad:243-244``).  Pinned to the reference by ``tests/golden`` (``pl_*``).
"""

from __future__ import annotations

import numpy as np


def _pool2(a):
    b, h, w, c = a.shape
    return a.reshape(b, h // 2, 2, w // 2, 2, c).mean(axis=(2, 4))


def _unpool2(g):
    return np.repeat(np.repeat(g, 2, axis=1), 2, axis=2) / 4.0


def patch_loss(r, t, lam_mse=0.2, lam_perc=1.0):
    """r, t (G, S, S, 3) -> (loss, mse, perc, d loss / d r), float64."""
    r = np.asarray(r, np.float64)
    t = np.asarray(t, np.float64)
    e = r - t
    mse = float(np.mean(e * e))
    grad = lam_mse * 2.0 * e / e.size
    perc = 0.0
    rs, ts = r, t
    for lvl in range(2):
        if lvl:
            rs, ts = _pool2(rs), _pool2(ts)
        g_lvl = np.zeros_like(rs)
        for ax in (2, 1):                    # horizontal, then vertical first differences
            d = np.diff(rs, axis=ax) - np.diff(ts, axis=ax)
            perc += float(np.mean(np.abs(d)))
            sg = np.sign(d) / d.size
            hi = [slice(None)] * 4
            lo = [slice(None)] * 4
            hi[ax], lo[ax] = slice(1, None), slice(None, -1)
            g_lvl[tuple(hi)] += sg
            g_lvl[tuple(lo)] -= sg
        grad += lam_perc * (g_lvl if lvl == 0 else _unpool2(g_lvl))
    return lam_mse * mse + lam_perc * perc, mse, perc, grad
