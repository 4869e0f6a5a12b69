"""Forward kinematics and motion bases G_i (oracle; float64).

Restates ``rodrigues`` (``sk:186-209``), ``forward_kinematics`` (``sk:240-273``) and
``motion_basis`` (``sk:288-303``): ``T_i = T_parent(i) o translate(rest_offset_i) o
rotate(omega_i)``; ``G_i = T_i(canonical) o T_i(observed)^-1`` so ``G_r = Rc Ro^T`` and
``G_t = tc - G_r to``.  Vectors are rows: a transform applies as ``x @ R.T + t``.
"""

from __future__ import annotations

import numpy as np


def rodrigues(omega):
    """(K,3) axis-angle -> (K,3,3) rotations, series branch for |w|^2 < 1e-8 (sk:186-209)."""
    w = np.atleast_2d(np.asarray(omega, dtype=np.float64))
    k = w.shape[0]
    s = np.zeros((k, 3, 3))
    s[:, 0, 1], s[:, 0, 2] = -w[:, 2], w[:, 1]
    s[:, 1, 0], s[:, 1, 2] = w[:, 2], -w[:, 0]
    s[:, 2, 0], s[:, 2, 1] = -w[:, 1], w[:, 0]
    ss = s @ s
    sumsq = np.sum(w * w, axis=1)
    near = sumsq < 1e-8
    n = np.sqrt(np.maximum(sumsq, 1e-120))
    a = np.where(near, 1.0 - sumsq / 6.0, np.sin(n) / n)
    b = np.where(near, 0.5 - sumsq / 24.0, (1.0 - np.cos(n)) / np.maximum(sumsq, 1e-120))
    return np.eye(3)[None] + a[:, None, None] * s + b[:, None, None] * ss


def topo_order(parent):
    order, placed, pending = [], set(), list(range(len(parent)))
    while pending:
        rest = []
        for i in pending:
            p = int(parent[i])
            if p < 0 or p in placed:
                order.append(i)
                placed.add(i)
            else:
                rest.append(i)
        pending = rest
    return order


def forward_kinematics(parent, rest_offset, angles, root_translation):
    """Per-bone world (R, t) (sk:240-273)."""
    rots = rodrigues(angles)
    k = len(parent)
    r_w = [None] * k
    t_w = [None] * k
    root = np.asarray(root_translation, dtype=np.float64)
    for i in topo_order(parent):
        off = np.asarray(rest_offset[i], dtype=np.float64)
        p = int(parent[i])
        if p < 0:
            r_w[i] = rots[i]
            t_w[i] = root + off
        else:
            r_w[i] = r_w[p] @ rots[i]
            t_w[i] = t_w[p] + off @ r_w[p].T
    return np.stack(r_w), np.stack(t_w)


def motion_basis(parent, rest_offset, canon_angles, canon_root, angles, root_translation):
    """G_r (K,3,3), G_t (K,3) mapping observation -> canonical (sk:288-303)."""
    rc, tc = forward_kinematics(parent, rest_offset, canon_angles, canon_root)
    ro, to = forward_kinematics(parent, rest_offset, angles, root_translation)
    g_r = rc @ np.swapaxes(ro, -1, -2)
    g_t = tc - np.einsum("kij,kj->ki", g_r, to)
    return g_r, g_t
