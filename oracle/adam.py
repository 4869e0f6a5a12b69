"""Bias-corrected Adam, in place (oracle; restates ``ad:880-912``).

``m = b1 m + (1-b1) g``; ``v = b2 v + (1-b2) g^2``;
``p -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)``; a non-finite gradient
raises before any update, naming the parameter block (``ad:901-902``).
"""

from __future__ import annotations

import numpy as np


class AdamState:
    def __init__(self, params, beta1=0.9, beta2=0.99, eps=1e-8):
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.t = 0
        self.m = [np.zeros_like(p) for p in params]
        self.v = [np.zeros_like(p) for p in params]


def adam_step(params, grads, state, lrs, names=None):
    """``lrs``: one learning rate per block (or a scalar)."""
    if np.isscalar(lrs):
        lrs = [lrs] * len(params)
    for i, g in enumerate(grads):
        if not np.all(np.isfinite(g)):
            name = names[i] if names else "unnamed"
            raise FloatingPointError(f"non-finite gradient in parameter block '{name}'")
    state.t += 1
    b1, b2 = state.beta1, state.beta2
    bc1 = 1.0 - b1 ** state.t
    bc2 = 1.0 - b2 ** state.t
    for p, g, m, v, lr in zip(params, grads, state.m, state.v, lrs):
        m *= b1
        m += (1.0 - b1) * g
        v *= b2
        v += (1.0 - b2) * (g * g)
        p -= lr * (m / bc1) / (np.sqrt(v / bc2) + state.eps)
