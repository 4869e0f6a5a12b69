"""CUDA-backed equivalent of the reference's ``freeview.fused`` (``fu:39-227``):
``FusedMlp`` (ReLU hidden layers, linear output, weights stored (in, out) as in ``linear``,
``ad:403-425``) and ``fused_forward(mlp, batch)``.

The reference evaluates the MLP in 128-sample chunks with 16x16 tiles loaded once per chunk
(``fu:145-179``); here ``fused_forward`` is one persistent kernel (``fv_fused_mlp_fwd``) that
stages every layer's weights in shared memory once per CTA and walks 128-row chunks with the
activations on chip, fp32 FMAs in fixed k order: a row's result does not depend on its chunk
(the reference's bitwise chunk invariance, ``t_fused:69-76``) and matches ``naive_forward``
to fp32 rounding.
"""

from __future__ import annotations

from typing import Optional, Sequence

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import DimensionError


WIDTH = 64          # fu:29: fixed hidden width of the reference's fused evaluator


class FusedMlp:
    """Fixed-width MLP (``fu:64-129``): ``weights`` ``[in x 64, 64 x 64, ..., 64 x out]`` (in, out
    storage as ``linear``, ``ad:403-425``), ReLU after every layer but the last; biases default
    to zeros.  The reference's shape rules raise ``DimensionError``: at least input and output
    layers, input/output width <= 64, hidden width 64, bias per layer width."""

    def __init__(self, weights: Sequence[torch.Tensor], biases: Optional[Sequence[torch.Tensor]] = None,
                 activation: str = "relu"):
        if activation != "relu":
            raise ValueError(f"unsupported activation '{activation}'")
        if len(weights) < 2:
            raise DimensionError("FusedMlp needs at least input and output layers")
        self.in_dim = int(weights[0].shape[0])
        self.out_dim = int(weights[-1].shape[1])
        if self.in_dim > WIDTH or self.out_dim > WIDTH:
            raise DimensionError(f"input/output width must be <= {WIDTH}, got {self.in_dim}/{self.out_dim}")
        for i, w in enumerate(weights):
            want_in = self.in_dim if i == 0 else WIDTH
            want_out = self.out_dim if i == len(weights) - 1 else WIDTH
            if tuple(w.shape) != (want_in, want_out):
                raise DimensionError(f"layer {i}: expected {(want_in, want_out)}, got {tuple(w.shape)}")
        self.activation = activation
        self.weights = [w.float().contiguous() for w in weights]
        if biases is None:
            biases = [torch.zeros(w.shape[1], dtype=torch.float32, device=w.device) for w in weights]
        self.biases = [b.float().contiguous() for b in biases]
        for w, b in zip(self.weights, self.biases):
            if tuple(b.shape) != (w.shape[1],):
                raise DimensionError(f"bias shape {tuple(b.shape)} vs layer width {w.shape[1]}")

    @property
    def n_in(self) -> int:
        return self.in_dim

    @property
    def n_out(self) -> int:
        return self.out_dim

    @property
    def depth(self) -> int:
        """Number of hidden (ReLU) layers."""
        return len(self.weights) - 1

    @classmethod
    def random(cls, in_dim: int, out_dim: int, depth: int, seed: int = 0, with_bias: bool = True,
               device: str = "cuda") -> "FusedMlp":
        """``fu:120-130``: per layer (in draw order) He-normal weights N(0, 2/in), then biases
        N(0, 0.01^2) (zeros without ``with_bias``), float32 -- the reference's exact draws."""
        rng = np.random.default_rng(seed)
        dims = [in_dim] + [WIDTH] * depth + [out_dim]
        ws, bs = [], []
        for a, b in zip(dims[:-1], dims[1:]):
            w = (rng.standard_normal((a, b)) * np.sqrt(2.0 / a)).astype(np.float32)
            bb = (rng.standard_normal(b) * 0.01 if with_bias else np.zeros(b)).astype(np.float32)
            ws.append(torch.from_numpy(w).to(device))
            bs.append(torch.from_numpy(bb).to(device))
        return cls(ws, bs)


def fused_forward(mlp: FusedMlp, batch: torch.Tensor) -> torch.Tensor:
    """(B, in) -> (B, out) float32 (``fu:182-193``): ONE ``fv_fused_mlp_fwd`` launch evaluates
    the whole network chunk by chunk with all weights resident in shared memory (the
    reference's ``_fused_kernel`` scheme, ``fu:145-179``).  The batch must be 2-D, of the MLP's
    input width, with B >= 1 (DimensionError otherwise, as the reference)."""
    if not isinstance(batch, torch.Tensor) or not batch.is_cuda:
        raise DimensionError("fused_forward: expected a CUDA tensor (no CPU fallback)")
    if batch.dim() != 2:
        raise DimensionError(f"fused_forward: batch must be 2-D, got shape {tuple(batch.shape)}")
    if batch.shape[1] != mlp.in_dim:
        raise DimensionError(f"fused_forward: batch width {batch.shape[1]} != MLP input width {mlp.in_dim}")
    if batch.shape[0] < 1:
        raise DimensionError("fused_forward: empty batch")
    for w in mlp.weights:
        if not w.is_cuda:
            raise DimensionError("fused_forward: MLP weights must live on the GPU (no CPU fallback)")
    lib = _lib.load()
    x = batch.float().contiguous()
    m = x.shape[0]
    n = len(mlp.weights)
    wp = (C.c_void_p * n)(*[w.data_ptr() for w in mlp.weights])
    bp = (C.c_void_p * n)(*[b.data_ptr() for b in mlp.biases])
    y = torch.empty((m, mlp.out_dim), dtype=torch.float32, device=x.device)
    _lib.check(lib.fv_fused_mlp_fwd(x.data_ptr(), m, mlp.in_dim, mlp.out_dim, n, wp, bp, y.data_ptr(),
                                    _lib.stream_ptr()), "fv_fused_mlp_fwd")
    return y


def naive_forward(mlp: FusedMlp, batch: torch.Tensor) -> torch.Tensor:
    """``fu:132-142`` on the device: alternating dense layer and ReLU, one ``fv_linear_fwd_tc``
    launch per layer (split-precision 3xTF32, fp32-accurate) -- the unfused reference path
    ``fused_forward`` is checked against."""
    if batch.dim() != 2 or batch.shape[1] != mlp.in_dim:
        raise DimensionError(f"batch width {tuple(batch.shape)} vs mlp input {mlp.in_dim}")
    from .autodiff import linear
    h = batch
    last = len(mlp.weights) - 1
    for i, (w, b) in enumerate(zip(mlp.weights, mlp.biases)):
        h = linear(h, w, b, "none" if i == last else "relu")
    return h
