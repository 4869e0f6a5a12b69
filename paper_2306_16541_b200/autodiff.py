"""CUDA-backed equivalents of the reference's ``freeview.autodiff`` primitives on the hot path
(keep ``sample_bone_channels``, ``posenc`` and ``transmittance`` by name), plus
``softmax0`` (the W^c normalisation they consume).  Each takes and returns CUDA tensors and
runs one kernel of ``libfvcuda.so``; there is no CPU fallback (a CPU tensor is refused, a
missing library raises).  Errors follow the reference: shape problems raise
``DimensionError`` (``ad:26-27``).

  * ``sample_bone_channels(nets, pts)``  -- ad:728-773 on the model's packed W^c
  * ``posenc(p, num_bands, alpha)``       -- ad:581-611 (raw xyz, then per band sin/cos)
  * ``transmittance(alpha)``              -- ad:815-837 (exclusive running product, N+1 entries)
  * ``softmax0(logits)``                  -- ad:711-721 (softmax over channel axis 0)

The backward passes of these ops live in the fused training kernels (``train.Trainer``);
these entry points are the forward operators the reference's tests and callers use.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from .errors import DimensionError
from .model import FreeviewModel, hann_band_weights


def _cuda_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise DimensionError(f"{name}: expected a CUDA tensor (no CPU fallback)")
    return t.float().contiguous()


def sample_bone_channels(nets: FreeviewModel, pts: torch.Tensor) -> torch.Tensor:
    """pts (K, N, 3) bone-space points -> (K, N): channel i of the model's W^c sampled
    trilinearly at pts[i] (ad:728-773; zero outside the one-voxel-padded grid)."""
    p = _cuda_f32(pts, "sample_bone_channels")
    k = nets.n_bones
    if p.dim() != 3 or p.shape[0] != k or p.shape[2] != 3:
        raise DimensionError(f"sample_bone_channels: pts must be ({k}, N, 3), got {tuple(p.shape)}")
    out = torch.empty((k, p.shape[1]), dtype=torch.float32, device=p.device)
    w = nets.warp_struct()
    _lib.check(nets.lib.fv_sample_bone_channels(C.byref(w), p.data_ptr(), p.shape[1], out.data_ptr(),
                                                _lib.stream_ptr()), "fv_sample_bone_channels")
    return out


def posenc(p: torch.Tensor, num_bands: int, alpha: Optional[float] = None) -> torch.Tensor:
    """(N, 3) -> (N, 3 + 6 num_bands): [x, y, z, then per band k: w_k sin(2^k pi x), w_k cos(..)]
    with the Hann window w_k(alpha) (ad:574-600); alpha defaults to num_bands (all on)."""
    x = _cuda_f32(p, "posenc")
    if x.dim() != 2 or x.shape[1] != 3:
        raise DimensionError(f"posenc: expected (N, 3), got {tuple(x.shape)}")
    if not 1 <= num_bands <= 8:
        raise DimensionError(f"posenc: 1..8 bands, got {num_bands}")
    n = x.shape[0]
    d = 3 + 6 * num_bands
    xs4 = torch.cat([x, torch.ones((n, 1), device=x.device)], 1).contiguous()
    out = torch.empty((n, d), dtype=torch.float32, device=x.device)
    if n == 0:
        return out
    w = hann_band_weights(num_bands, float(num_bands if alpha is None else alpha))
    wc = (C.c_float * 8)(*[float(v) for v in w])
    lib = _lib.load()
    _lib.check(lib.fv_posenc_fwd(xs4.data_ptr(), n, 0.0, num_bands, wc, out.data_ptr(), d, _lib.stream_ptr()),
               "fv_posenc_fwd")
    return out


def transmittance(alpha: torch.Tensor) -> torch.Tensor:
    """alpha (R, N) -> T (R, N + 1): T[:, 0] = 1, T[:, i + 1] = T[:, i] (1 - alpha[:, i])
    (ad:815-837, exclusive; T[:, N] is the background weight)."""
    a = _cuda_f32(alpha, "transmittance")
    if a.dim() != 2:
        raise DimensionError(f"transmittance: expected (R, N), got {tuple(a.shape)}")
    r, n = a.shape
    out = torch.empty((r, n + 1), dtype=torch.float32, device=a.device)
    lib = _lib.load()
    _lib.check(lib.fv_transmittance(a.data_ptr(), r, n, out.data_ptr(), _lib.stream_ptr()), "fv_transmittance")
    return out


def softmax0(logits: torch.Tensor) -> torch.Tensor:
    """Softmax over axis 0 of (C, ...) logits (ad:711-721), e.g. the (K+1, G, G, G) W^c."""
    a = _cuda_f32(logits, "softmax0")
    if a.dim() < 1 or a.shape[0] < 1:
        raise DimensionError(f"softmax0: expected (C, ...), got {tuple(a.shape)}")
    out = torch.empty_like(a)
    vox = a[0].numel()
    lib = _lib.load()
    _lib.check(lib.fv_softmax0_fwd(a.data_ptr(), a.shape[0], vox, out.data_ptr(), _lib.stream_ptr()),
               "fv_softmax0_fwd")
    return out
