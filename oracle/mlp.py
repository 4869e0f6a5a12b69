"""MLP layers and radiance heads (oracle).

``mlp_forward`` is the reference's naive evaluation (``fu:132-142``; each layer is
``linear`` = ``act(x @ W + b)`` with ``W`` stored (in, out), ``ad:403-425``): ReLU after
every layer except the last.  ``mlp_backward`` restates the ``linear`` backward
(``ad:417-422``).  Heads: ``c = sigmoid(h[:3])``, ``sigma = softplus(h[3] - 1)``
(``S:422``; stable forms ``ad:200-222``).
"""

from __future__ import annotations

import numpy as np


def mlp_forward(x, weights, biases, dtype=np.float32, keep=False):
    dt = np.dtype(dtype).type
    h = np.asarray(x, dtype=dt)
    acts = [h]
    last = len(weights) - 1
    for i, (w, b) in enumerate(zip(weights, biases)):
        h = (h @ np.asarray(w, dtype=dt) + np.asarray(b, dtype=dt)).astype(dt)
        if i != last:
            h = np.maximum(h, dt(0.0))
        acts.append(h)
    return (h, acts) if keep else h


def mlp_backward(acts, weights, g_out):
    """Returns (g_input, [gW], [gb]) in float64 for the activations ``acts`` of a forward."""
    g = np.asarray(g_out, dtype=np.float64)
    last = len(weights) - 1
    gws, gbs = [None] * len(weights), [None] * len(weights)
    for i in range(last, -1, -1):
        if i != last:
            g = g * (acts[i + 1] > 0)
        gws[i] = acts[i].astype(np.float64).T @ g
        gbs[i] = g.sum(axis=0)
        g = g @ np.asarray(weights[i], dtype=np.float64).T
    return g, gws, gbs


def sigmoid(x):
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def softplus(x):
    return np.log1p(np.exp(-np.abs(x))) + np.maximum(x, 0)


def radiance_heads(h):
    """h (N,4) -> (c (N,3), sigma (N,))."""
    dt = h.dtype.type
    return sigmoid(h[:, :3]), softplus((h[:, 3] - dt(1.0)).astype(dt))


def radiance_heads_bwd(h, dc, dsigma):
    """d head pre-activations (N,4) given dL/dc (N,3), dL/dsigma (N,)."""
    h = h.astype(np.float64)
    c = sigmoid(h[:, :3])
    out = np.empty_like(h)
    out[:, :3] = dc * c * (1.0 - c)
    out[:, 3] = dsigma * sigmoid(h[:, 3] - 1.0)
    return out


def xavier_uniform(rng, fan_in, fan_out):
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-lim, lim, (fan_in, fan_out))
