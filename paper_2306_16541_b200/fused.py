"""CUDA-backed equivalent of the reference's ``freeview.fused`` (``fu:39-227``):
``FusedMlp`` (ReLU hidden layers, linear output, weights stored (in, out) as in ``linear``,
``ad:403-425``) and ``fused_forward(mlp, batch)``.

The reference evaluates the MLP in 128-sample chunks with 16x16 tiles (``fu:145-179``); here
every layer is one persistent tcgen05 kernel over the whole batch (``fv_linear_fwd_tc``:
split-precision 3xTF32 on fp32 data, fp32 accumulation, i.e. fp32-accurate), so the result
does not depend on chunking at all (the reference's bitwise chunk-invariance property,
``t_fused:48-86``, holds trivially) and matches ``naive_forward`` to fp32 rounding.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np
import torch

from . import _lib
from .errors import DimensionError


@dataclass
class FusedMlp:
    """weights[i] (in_i, out_i), biases[i] (out_i), CUDA float32; ReLU on all but the last."""
    weights: List[torch.Tensor]
    biases: List[torch.Tensor]

    @property
    def n_in(self) -> int:
        return int(self.weights[0].shape[0])

    @property
    def n_out(self) -> int:
        return int(self.weights[-1].shape[1])

    @staticmethod
    def random(n_in: int, n_out: int, depth: int = 2, width: int = 64, seed: int = 0,
               device: str = "cuda") -> "FusedMlp":
        """depth hidden layers of `width` (fu:120-130: He-normal weights, zero biases)."""
        rng = np.random.default_rng(seed)
        dims = [n_in] + [width] * depth + [n_out]
        ws, bs = [], []
        for a, b in zip(dims[:-1], dims[1:]):
            ws.append(torch.from_numpy((rng.standard_normal((a, b)) * np.sqrt(2.0 / a)).astype(np.float32)).to(device))
            bs.append(torch.zeros(b, dtype=torch.float32, device=device))
        return FusedMlp(ws, bs)


def fused_forward(mlp: FusedMlp, batch: torch.Tensor) -> torch.Tensor:
    """(B, n_in) -> (B, n_out) float32 (fu:182-193): batch must be 2-D, of the MLP's input
    width, with B >= 1 (DimensionError otherwise, as the reference)."""
    if not isinstance(batch, torch.Tensor) or not batch.is_cuda:
        raise DimensionError("fused_forward: expected a CUDA tensor (no CPU fallback)")
    if batch.dim() != 2:
        raise DimensionError(f"fused_forward: batch must be 2-D, got shape {tuple(batch.shape)}")
    if batch.shape[1] != mlp.n_in:
        raise DimensionError(f"fused_forward: batch width {batch.shape[1]} != MLP input width {mlp.n_in}")
    if batch.shape[0] < 1:
        raise DimensionError("fused_forward: empty batch")
    lib = _lib.load()
    sp = _lib.stream_ptr()
    x = batch.float().contiguous()
    m = x.shape[0]
    last = len(mlp.weights) - 1
    for i, (w, b) in enumerate(zip(mlp.weights, mlp.biases)):
        k, n = int(w.shape[0]), int(w.shape[1])
        if k != x.shape[1] or b.shape[0] != n:
            raise DimensionError(f"fused_forward: layer {i} is ({k}, {n}) with bias {tuple(b.shape)}, input {x.shape[1]}")
        wc, bc = w.float().contiguous(), b.float().contiguous()
        y = torch.empty((m, n), dtype=torch.float32, device=x.device)
        _lib.check(lib.fv_linear_fwd_tc(x.data_ptr(), k, wc.data_ptr(), bc.data_ptr(), y.data_ptr(), n, m, k, n,
                                        0 if i == last else 1, sp), "fv_linear_fwd_tc")
        x = y
    return x
