"""CUDA-backed drop-ins for the reference's ``freeview.autodiff`` operators on the hot path
(same names, same argument meaning, same errors), as ``torch.autograd``
functions whose forward AND backward are libfvcuda.so kernels.

The reference op is ``op(*Tensor, **consts) -> Tensor`` that records ``backward(g)`` on a
``Tape`` when a parent requires grad (``_emit``, ``ad:144-150``).  Here the tape is torch
autograd: every op below is a ``torch.autograd.Function`` (recorded only when an input
requires grad, as ``_emit``), operands are CUDA float32 tensors, and each direction is one
C-ABI call on the current stream:

  * ``sample_bone_channels(vol, pts, box_min, box_max)``  ad:728-808   fv_warp_pack +
    fv_sample_bone_channels / fv_sample_bone_channels_bwd (d vol and d pts)
  * ``posenc(p, num_bands, alpha, include_raw=True)``     ad:581-611   fv_posenc_fwd / _bwd
  * ``transmittance(atten)``                              ad:815-837   fv_transmittance /
    fv_transmittance_bwd (the division-free reverse scan, exact zeros safe)
  * ``softmax0(a)``                                       ad:711-721   fv_softmax0_fwd / _bwd
  * ``linear(x, w, b, activation)``                       ad:403-425   fv_linear_fwd_tc
    (split-precision 3xTF32, fp32-accurate) / fv_linear_bwd
  * ``AdamState`` / ``adam_step(params, grads, state, lr)`` ad:880-912  fv_adam_step (in
    place; non-finite gradients raise TrainingError naming the block before any update)

No CPU fallback: CPU tensors are refused (``DimensionError``), a missing library raises.
Shape errors raise ``DimensionError`` (``ad:26-27``) with the offending shapes.
"""

from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import DimensionError, TrainingError
from .model import hann_band_weights

__all__ = ["sample_bone_channels", "posenc", "posenc_dim", "transmittance", "softmax0", "linear", "AdamState",
           "adam_step", "hann_band_weights"]


def _cuda_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise DimensionError(f"{name}: expected a CUDA tensor (no CPU fallback)")
    return t.float().contiguous()


def _sp() -> int:
    return _lib.stream_ptr()


# ------------------------------------------------------------------- sample_bone_channels

def _bone_warp(vol: torch.Tensor, k: int, box_min, box_max):
    """fv_warp view of an arbitrary (C, G, G, G) grid: first k channels corner-packed (fp32)."""
    g = int(vol.shape[1])
    w = _lib.FvWarp()
    w.n_bones, w.vol_res, w.vol_half = k, g, 0
    bmin = np.asarray(box_min, np.float32).reshape(3)
    bmax = np.asarray(box_max, np.float32).reshape(3)
    if np.any(bmax <= bmin):
        raise DimensionError(f"sample_bone_channels: empty box {bmin} .. {bmax}")
    _lib.farr(w.wbox_min, bmin)
    _lib.farr(w.wscale, (np.float32(g - 1) / (bmax - bmin)).astype(np.float32))
    packed = torch.empty(k * (g + 1) ** 3 * 8, dtype=torch.float32, device=vol.device)
    w.d_vol_packed = packed.data_ptr()
    w.d_g = None
    lib = _lib.load()
    _lib.check(lib.fv_warp_pack(vol.data_ptr(), int(vol.shape[0]), C.byref(w), packed.data_ptr(), _sp()),
               "fv_warp_pack")
    return w, packed


class _SampleBoneChannels(torch.autograd.Function):
    @staticmethod
    def forward(ctx, vol, pts, box_min, box_max):
        vol, pts = vol.contiguous(), pts.contiguous()
        k, n = int(pts.shape[0]), int(pts.shape[1])
        w, packed = _bone_warp(vol, k, box_min, box_max)
        out = torch.empty((k, n), dtype=torch.float32, device=pts.device)
        if n:
            _lib.check(_lib.load().fv_sample_bone_channels(C.byref(w), pts.data_ptr(), n, out.data_ptr(), _sp()),
                       "fv_sample_bone_channels")
        ctx.save_for_backward(pts)
        ctx.w, ctx.packed, ctx.vshape = w, packed, tuple(vol.shape)
        return out

    @staticmethod
    def backward(ctx, g):
        (pts,) = ctx.saved_tensors
        k, n = int(pts.shape[0]), int(pts.shape[1])
        need_vol, need_pts = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        dvol = torch.zeros(ctx.vshape, dtype=torch.float32, device=pts.device) if need_vol else None
        dpts = torch.empty_like(pts) if need_pts else None
        if n and (need_vol or need_pts):
            gc = g.float().contiguous()
            _lib.check(_lib.load().fv_sample_bone_channels_bwd(
                C.byref(ctx.w), pts.data_ptr(), n, gc.data_ptr(), dvol.data_ptr() if need_vol else None,
                dpts.data_ptr() if need_pts else None, _sp()), "fv_sample_bone_channels_bwd")
        return dvol, dpts, None, None


def sample_bone_channels(vol: torch.Tensor, pts: torch.Tensor, box_min, box_max) -> torch.Tensor:
    """Channel ``i`` of ``vol`` (C, G, G, G) sampled trilinearly at ``pts[i]`` (K, N, 3), K <= C
    (``ad:728-808``): box-corner-aligned grid, linear fall-off to the zero padding, exactly 0
    beyond one voxel outside.  Differentiable in both the grid values and the positions."""
    v = _cuda_f32(vol, "sample_bone_channels")
    p = _cuda_f32(pts, "sample_bone_channels")
    if p.dim() != 3 or p.shape[-1] != 3:
        raise DimensionError(f"sample_bone_channels: points {tuple(pts.shape)}")
    if v.dim() != 4:
        raise DimensionError(f"sample_bone_channels: volume {tuple(vol.shape)} is not (C, G0, G1, G2)")
    if p.shape[0] > v.shape[0]:
        raise DimensionError(f"sample_bone_channels: {p.shape[0]} bones > {v.shape[0]} channels")
    if not (v.shape[1] == v.shape[2] == v.shape[3]) or v.shape[1] < 2 or v.shape[1] > _lib.MAX_VOL_RES:
        raise DimensionError(f"sample_bone_channels: cubic grids 2..{_lib.MAX_VOL_RES} supported, got {tuple(v.shape)}")
    if p.shape[0] < 1 or p.shape[0] > _lib.MAX_BONES:
        raise DimensionError(f"sample_bone_channels: 1..{_lib.MAX_BONES} bones, got {p.shape[0]}")
    return _SampleBoneChannels.apply(vol.float(), pts.float(), box_min, box_max)


# ------------------------------------------------------------------------------ posenc

def posenc_dim(num_bands: int, include_raw: bool = True, point_dim: int = 3) -> int:
    """ad:614-615."""
    return (point_dim if include_raw else 0) + 2 * point_dim * num_bands


class _Posenc(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, num_bands, alpha, include_raw):
        x = x.contiguous()
        n = int(x.shape[0])
        d = 3 + 6 * num_bands
        xs4 = torch.cat([x, torch.ones((n, 1), device=x.device)], 1).contiguous()
        out = torch.empty((n, d), dtype=torch.float32, device=x.device)
        w = (C.c_float * 8)(*[float(v) for v in hann_band_weights(num_bands, float(alpha))])
        if n:
            _lib.check(_lib.load().fv_posenc_fwd(xs4.data_ptr(), n, 0.0, num_bands, w, out.data_ptr(), d, _sp()),
                       "fv_posenc_fwd")
        ctx.save_for_backward(xs4)
        ctx.num_bands, ctx.w, ctx.include_raw = num_bands, w, include_raw
        return out if include_raw else out[:, 3:].contiguous()

    @staticmethod
    def backward(ctx, g):
        (xs4,) = ctx.saved_tensors
        n = int(xs4.shape[0])
        d = 3 + 6 * ctx.num_bands
        if ctx.include_raw:
            gfull = g.float().contiguous()
        else:                                     # raw columns carry no gradient (ad:603)
            gfull = torch.zeros((n, d), dtype=torch.float32, device=g.device)
            gfull[:, 3:] = g
        dx = torch.zeros((n, 3), dtype=torch.float32, device=g.device)
        if n:
            _lib.check(_lib.load().fv_posenc_bwd(xs4.data_ptr(), n, 0.0, ctx.num_bands, ctx.w, gfull.data_ptr(), d,
                                                 dx.data_ptr(), _sp()), "fv_posenc_bwd")
        return dx, None, None, None


def posenc(p: torch.Tensor, num_bands: int, alpha: Optional[float] = None, include_raw: bool = True) -> torch.Tensor:
    """(N, 3) -> (N, posenc_dim): raw xyz (when ``include_raw``), then per band k the weighted
    ``sin(2^k pi p)`` and ``cos(2^k pi p)`` triples, weights w_k(alpha) = Hann window
    (``ad:574-611``); ``alpha`` defaults to ``num_bands`` (all bands on)."""
    x = _cuda_f32(p, "posenc")
    if x.dim() != 2 or x.shape[1] != 3:
        raise DimensionError(f"posenc expects (N,3)-like input, got {tuple(p.shape)}")
    if not 1 <= num_bands <= 8:
        raise DimensionError(f"posenc: 1..8 bands, got {num_bands}")
    a = float(num_bands if alpha is None else alpha)
    return _Posenc.apply(p.float(), int(num_bands), a, bool(include_raw))


# ----------------------------------------------------------------------- transmittance

class _Transmittance(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a):
        a = a.contiguous()
        r, n = int(a.shape[0]), int(a.shape[1])
        out = torch.empty((r, n + 1), dtype=torch.float32, device=a.device)
        if r:
            _lib.check(_lib.load().fv_transmittance(a.data_ptr(), r, n, out.data_ptr(), _sp()), "fv_transmittance")
        ctx.save_for_backward(a, out)
        return out

    @staticmethod
    def backward(ctx, g):
        a, out = ctx.saved_tensors
        r, n = int(a.shape[0]), int(a.shape[1])
        gx = torch.empty_like(a)
        gc = g.float().contiguous()
        if r and n:
            _lib.check(_lib.load().fv_transmittance_bwd(a.data_ptr(), out.data_ptr(), gc.data_ptr(), r, n,
                                                        gx.data_ptr(), _sp()), "fv_transmittance_bwd")
        return gx


def transmittance(atten: torch.Tensor) -> torch.Tensor:
    """Exclusive running product of per-sample attenuations (``ad:815-837``): ``atten`` (R, N)
    holds ``1 - opacity``; output (R, N+1) with ``T[:, 0] = 1`` and ``T[:, i] = prod_{j<i}
    atten[:, j]``.  The backward is the reference's division-free reverse scan."""
    a = _cuda_f32(atten, "transmittance")
    if a.dim() != 2:
        raise DimensionError(f"transmittance: expected (R, N), got {tuple(atten.shape)}")
    return _Transmittance.apply(atten.float())


# ----------------------------------------------------------------------------- softmax0

class _Softmax0(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a):
        a = a.contiguous()
        out = torch.empty_like(a)
        ch, vox = int(a.shape[0]), int(a[0].numel())
        if a.numel():
            _lib.check(_lib.load().fv_softmax0_fwd(a.data_ptr(), ch, vox, out.data_ptr(), _sp()), "fv_softmax0_fwd")
        ctx.save_for_backward(out)
        return out

    @staticmethod
    def backward(ctx, g):
        (out,) = ctx.saved_tensors
        da = torch.zeros_like(out)
        gc = g.float().contiguous()
        if out.numel():
            _lib.check(_lib.load().fv_softmax0_bwd(out.data_ptr(), gc.data_ptr(), int(out.shape[0]),
                                                   int(out[0].numel()), da.data_ptr(), _sp()), "fv_softmax0_bwd")
        return da


def softmax0(a: torch.Tensor) -> torch.Tensor:
    """Softmax over the leading (channel) axis (``ad:711-721``), e.g. the (K+1, G, G, G) W^c;
    backward ``out * (g - sum(g * out))``."""
    x = _cuda_f32(a, "softmax0")
    if x.dim() < 1 or x.shape[0] < 1:
        raise DimensionError(f"softmax0: expected (C, ...), got {tuple(a.shape)}")
    return _Softmax0.apply(a.float())


# -------------------------------------------------------------------------------- linear

class _Linear(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b, act):
        x, w = x.contiguous(), w.contiguous()
        b = b.contiguous() if b is not None else None
        m, k = int(x.shape[0]), int(x.shape[1])
        n = int(w.shape[1])
        y = torch.empty((m, n), dtype=torch.float32, device=x.device)
        bias = b if b is not None else torch.zeros(n, dtype=torch.float32, device=x.device)
        if m:
            _lib.check(_lib.load().fv_linear_fwd_tc(x.data_ptr(), k, w.data_ptr(), bias.data_ptr(), y.data_ptr(), n,
                                                    m, k, n, act, _sp()), "fv_linear_fwd_tc")
        ctx.save_for_backward(x, w, y)
        ctx.act, ctx.has_b = act, b is not None
        return y

    @staticmethod
    def backward(ctx, g):
        x, w, y = ctx.saved_tensors
        m, k, n = int(x.shape[0]), int(x.shape[1]), int(w.shape[1])
        gc = g.float().contiguous()
        dx = torch.empty_like(x) if ctx.needs_input_grad[0] else None
        dw = torch.zeros_like(w)
        db = torch.zeros(n, dtype=torch.float32, device=x.device)
        if m:
            _lib.check(_lib.load().fv_linear_bwd(x.data_ptr(), w.data_ptr(), y.data_ptr(), gc.data_ptr(),
                                                 dx.data_ptr() if dx is not None else None, dw.data_ptr(),
                                                 db.data_ptr(), m, k, n, ctx.act, _sp()), "fv_linear_bwd")
        elif dx is not None:
            dx.zero_()
        return dx, (dw if ctx.needs_input_grad[1] else None), (db if ctx.has_b and ctx.needs_input_grad[2] else None), None


def linear(x: torch.Tensor, w: torch.Tensor, b: Optional[torch.Tensor], activation: str = "none") -> torch.Tensor:
    """``act(x @ w + b)`` with w stored (in, out) (``ad:403-425``); activation "none" or "relu"."""
    if activation not in ("none", "relu"):
        raise ValueError(f"unknown activation '{activation}'")
    xs, ws = _cuda_f32(x, "linear"), _cuda_f32(w, "linear")
    if xs.dim() != 2 or ws.dim() != 2 or xs.shape[1] != ws.shape[0]:
        raise DimensionError(f"linear: input {tuple(x.shape)} vs weight {tuple(w.shape)}")
    bs = None
    if b is not None:
        bs = _cuda_f32(b, "linear")
        if bs.dim() != 1 or bs.shape[0] != ws.shape[1]:
            raise DimensionError(f"linear: bias {tuple(b.shape)} vs weight {tuple(w.shape)}")
    return _Linear.apply(x.float(), w.float(), b.float() if b is not None else None, 1 if activation == "relu" else 0)


# --------------------------------------------------------------------------------- Adam

class AdamState:
    """First/second moment buffers (device, zero) and step counter for one parameter group
    (``ad:880-890``)."""

    def __init__(self, params: Sequence[torch.Tensor], beta1: float = 0.9, beta2: float = 0.99, eps: float = 1e-8):
        self.beta1, self.beta2, self.eps = float(beta1), float(beta2), float(eps)
        self.t = 0
        self.m = [torch.zeros_like(p, dtype=torch.float32) for p in params]
        self.v = [torch.zeros_like(p, dtype=torch.float32) for p in params]
        self._flag = None


def adam_step(params: Sequence[torch.Tensor], grads: Sequence[torch.Tensor], state: AdamState, lr: float,
              names: Optional[List[str]] = None) -> None:
    """Bias-corrected Adam applied in place (``ad:893-912``): m <- b1 m + (1-b1) g,
    v <- b2 v + (1-b2) g^2, p <- p - lr (m/bc1) / (sqrt(v/bc2) + eps).  Every gradient is
    checked first (one device pass per block, one host read): a non-finite one raises
    ``TrainingError`` naming the block and no parameter, moment or step count changes
    (``ad:898-902``)."""
    if len(params) != len(state.m) or len(grads) != len(params):
        raise DimensionError("adam_step: parameter/gradient/state count mismatch")
    lib = _lib.load()
    for p, g in zip(params, grads):
        if not (isinstance(p, torch.Tensor) and p.is_cuda and p.dtype == torch.float32 and p.is_contiguous()):
            raise DimensionError("adam_step: parameters must be contiguous float32 CUDA tensors (updated in place)")
        if tuple(g.shape) != tuple(p.shape):
            raise DimensionError(f"adam_step: grad shape {tuple(g.shape)} vs param {tuple(p.shape)}")
    dev = params[0].device if params else torch.device("cuda")
    if state._flag is None:
        state._flag = torch.zeros(1, dtype=torch.int32, device=dev)
    flag = state._flag
    flag.zero_()
    gs = [_cuda_f32(g, "adam_step") for g in grads]
    for i, g in enumerate(gs):
        _lib.check(lib.fv_check_finite(g.data_ptr(), g.numel(), i + 1, flag.data_ptr(), _sp()), "fv_check_finite")
    bad = int(flag.item())
    if bad:
        name = names[bad - 1] if names else getattr(params[bad - 1], "name", None) or f"#{bad - 1}"
        raise TrainingError(f"non-finite gradient in parameter block '{name}'")
    state.t += 1
    ends = (C.c_int64 * 1)()
    lrs = (C.c_float * 1)(float(lr))
    for p, g, m, v in zip(params, gs, state.m, state.v):
        ends[0] = p.numel()
        _lib.check(lib.fv_adam_step(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel(), ends, lrs, 1,
                                    state.t, state.beta1, state.beta2, state.eps, None, 0, 0, flag.data_ptr(), _sp()),
                   "fv_adam_step")
