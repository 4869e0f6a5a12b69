"""Patch-based training step on the sm_100a path (SPEC ``S:468-551``; BASELINE config 3).

One iteration (``S:505-513``): sample G patches of S x S pixels whose window meets the
mask's dilated bounding box (``S:487-490``), render their rays through the full per-sample
pipeline keeping every activation, L2 loss against the target (``S:496-504``; the
perceptual term is off in config 3), backward through compositing, radiance heads and MLP,
hash-grid scatter, residual MLP, posenc and the skinning-weight volume, then one fused
Adam step over all parameter blocks (lr 5e-4 for table + radiance MLP, 5e-5 for the
residual MLP and W^c logits; beta = (0.9, 0.99), ``P:227``).

The reference replays a numpy Tape of per-op closures (``ad:87-150``); here every op of
that tape is one libfvcuda entry point on the current CUDA stream.  Gradients are fp32;
the hash table is kept as an fp32 master with the fp16 copy the forward reads rewritten
by the Adam kernel.  With ``torch.distributed`` initialised (NCCL), the flat gradient
buffer is all-reduced (mean) between backward and Adam -- the only exchange of the path.
"""

from __future__ import annotations

import copy
import csv
import ctypes as C
import json
import os
import time
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from .camera import CameraModel
from .errors import TrainingError
from .model import FreeviewModel, hann_band_weights
from .render import RenderSettings, camera_struct, march_struct
from .scene import PE_BANDS
from .skeleton import Pose
from .shard import GradBuckets


def sample_patches(mask: np.ndarray, n_patches: int, size: int, seed: int, step: int) -> np.ndarray:
    """Top-left origins (G,2) = (y0, x0) of S x S windows meeting the mask's bounding box
    dilated by S/2; uniform, deterministic per (seed, step); an empty mask falls
    back to image-uniform origins."""
    h, w = mask.shape
    rng = np.random.default_rng([seed, step])
    ys, xs = np.nonzero(mask)
    if len(ys) == 0:
        y_lo, y_hi, x_lo, x_hi = 0, h - size, 0, w - size
    else:
        d = size // 2
        by0, by1 = max(ys.min() - d, 0), min(ys.max() + d, h - 1)
        bx0, bx1 = max(xs.min() - d, 0), min(xs.max() + d, w - 1)
        y_lo, y_hi = max(0, by0 - size + 1), min(h - size, by1)
        x_lo, x_hi = max(0, bx0 - size + 1), min(w - size, bx1)
    return np.stack([rng.integers(y_lo, y_hi + 1, n_patches), rng.integers(x_lo, x_hi + 1, n_patches)], axis=1)


def patch_pixels(origins: np.ndarray, size: int, width: int) -> np.ndarray:
    """Linear pixel ids of the patches, each patch row-major (32 rays per row = one ray block)."""
    yy, xx = np.meshgrid(np.arange(size), np.arange(size), indexing="ij")
    return np.concatenate([((o[0] + yy) * width + o[1] + xx).reshape(-1) for o in origins]).astype(np.int32)


class Trainer:
    """Owns every activation / gradient buffer of one training step (no allocation per step)."""

    def __init__(self, nets: FreeviewModel, camera: CameraModel, target: np.ndarray, mask: np.ndarray,
                 settings: RenderSettings, n_patches: int = 6, patch: int = 32, seed: int = 0,
                 process_group=None, precision: str = "tf32", lam_mse: float = 1.0, lam_perc: float = 0.0,
                 weight_net=None, pose_refiner=None, pose=None):
        if precision not in ("tf32", "fp32"):
            raise ValueError("precision must be 'tf32' (tcgen05 kind::tf32 layers) or 'fp32' (SIMT, strict parity)")
        self.tc = precision == "tf32"
        self.nets, self.cam, self.st = nets, camera, settings
        self.lib = nets.lib
        self.dev = nets.device
        self.mask = mask
        self.n_patches, self.patch, self.seed = n_patches, patch, seed
        self.pg = process_group
        self.R = n_patches * patch * patch
        self.N = settings.n_samples
        self.S = (self.R + 31) // 32 * 32 * self.N
        S, dev = self.S, self.dev
        f32 = dict(device=dev, dtype=torch.float32)
        self.target = torch.from_numpy(np.ascontiguousarray(target.reshape(-1, 3), np.float32)).to(dev)
        self.pix = torch.empty(self.R, device=dev, dtype=torch.int32)
        # pinned ring for the per-step patch pixel ids: the host may run ahead of the GPU, so a
        # slot is rewritten only after the H2D copy that last read it has completed
        self.pix_ring = [torch.empty(self.R, dtype=torch.int32, pin_memory=True) for _ in range(4)]
        self.pix_events = [None] * 4
        self.pix_slot = 0
        d_pe = 3 + 6 * PE_BANDS
        self.d_pe = d_pe
        self.pe_ld = (d_pe + 3) // 4 * 4 if self.tc else d_pe   # 16-byte rows for the TF32 GEMMs
        self.xs = torch.empty((S, 4), **f32)
        self.delta = torch.empty(S, **f32)
        self.x = torch.empty((S, 3), **f32)
        self.pe = torch.empty((S, self.pe_ld), **f32)
        self.h = [torch.empty((S, 128), **f32) for _ in range(4)]
        # ReLU masks of the hidden activations as bits (tensor-core path): 1 uint32 per 32 units
        i32 = dict(device=dev, dtype=torch.int32)
        self.hbits = [torch.empty((S, 4), **i32) for _ in range(4)] if self.tc else [None] * 4
        self.rbits = [torch.empty((S, 2), **i32) for _ in range(2)] if self.tc else [None] * 2
        self.xres = torch.empty((S, 3), **f32)
        self.xf = torch.empty((S, 3), **f32)
        self.feat = torch.empty((S, 32), **f32)
        self.r = [torch.empty((S, 64), **f32) for _ in range(2)]
        self.hd = torch.empty((S, 4), **f32)
        self.rgbs = torch.empty((S, 4), **f32)
        self.rgb = torch.empty((self.R, 3), **f32)
        self.alpha = torch.empty(self.R, **f32)
        self.trans = torch.empty((self.R, self.N + 1), **f32)
        self.loss = torch.zeros(3, **f32)      # (total, mse term, perceptual-proxy term)
        self.lam_mse, self.lam_perc = float(lam_mse), float(lam_perc)
        if self.lam_perc != 0.0 and patch % 2:
            raise ValueError("the perceptual proxy needs an even patch size (2x2 pooling, ad:862-866)")
        self.drgb = torch.empty((self.R, 3), **f32)
        self.d_rgbs = torch.empty((S, 4), **f32)
        self.dh = torch.empty((S, 4), **f32)
        self.g128 = [torch.empty((S, 128), **f32) for _ in range(2)]
        self.g64 = [torch.empty((S, 64), **f32) for _ in range(2)]
        self.dfeat = torch.empty((S, 32), **f32)
        self.dxf = torch.empty((S, 3), **f32)
        self.dxs = torch.empty((S, 3), **f32)
        self.dpe = torch.empty((S, self.pe_ld), **f32)
        self.dvol = torch.empty_like(nets.vol)
        # optimizer state over the flat master buffer
        self.grad = torch.zeros_like(nets.flat)
        self.m = torch.zeros_like(nets.flat)
        self.v = torch.zeros_like(nets.flat)
        self.flag = torch.zeros(1, device=dev, dtype=torch.int32)
        self.buckets = GradBuckets(self.grad, process_group)
        self.t = 0
        self.gviews = {}
        for name, (a, b) in nets.block_ranges.items():
            self.gviews[name] = self.grad[a:b].view(nets.views[name].shape)
        self.seg_end = (C.c_int64 * 2)(*[int(e) for e, _ in nets.segments])
        self.seg_lr = (C.c_float * 2)(*[float(lr) for _, lr in nets.segments])
        self.pe_w = (C.c_float * 8)(*hann_band_weights(PE_BANDS, nets.pe_alpha).tolist())
        self.residual = bool(nets.offset_enabled)
        self.bg = (C.c_float * 3)(*settings.background)
        self.table_elems = nets.views["table"].numel()
        # optional pose refiner (pose.py): per step the frame's pose is refined, its motion bases
        # uploaded, and dL/dG_i (fv_warp_bwd_g) plus the residual MLP's pose-input gradient are
        # chained to the refiner on the host
        self.pose_refiner = pose_refiner
        if pose_refiner is not None:
            if pose is None:
                raise ValueError("a pose refiner needs the frame's pose")
            from .model import LR_OTHER
            self.base_pose = pose
            self.dg = torch.zeros((nets.n_bones, 12), device=dev, dtype=torch.float32)
            self.popt = torch.optim.Adam(pose_refiner.parameters(), lr=LR_OTHER, betas=(0.9, 0.99), eps=1e-8)
            self._refined = None
        # optional canonical weight-volume generator (weightnet.py): W^c logits come from it
        self.weight_net = weight_net
        self._wlogits = None
        if weight_net is not None:
            weight_net.to(dev)
            if tuple(weight_net().shape) != tuple(nets.views["vol_logits"].shape):
                raise ValueError("weight-volume generator output does not match the model's W^c logits")
            from .model import LR_OTHER
            self.wopt = torch.optim.Adam(weight_net.parameters(), lr=LR_OTHER, betas=(0.9, 0.99), eps=1e-8)

    def set_frame(self, camera: CameraModel, target: np.ndarray, mask: np.ndarray) -> None:
        """Switch the training frame ("pick a training frame"): its camera, target image
        and foreground mask (same resolution, so every step buffer is reused)."""
        t = np.ascontiguousarray(np.asarray(target, np.float32).reshape(-1, 3))
        if t.shape != tuple(self.target.shape) or camera.width * camera.height != t.shape[0]:
            raise ValueError("set_frame: every frame must have the trainer's resolution")
        self.cam, self.mask = camera, mask
        self.target.copy_(torch.from_numpy(t).to(self.dev), non_blocking=False)

    def set_schedule(self, alpha: float, residual: bool) -> None:
        """Coarse-to-fine state of one iteration: Hann window alpha of the
        positional encoding and whether the residual stage runs (off => x_res exactly 0 and
        no residual-MLP gradient)."""
        self.nets.set_schedule(alpha=alpha, residual=residual)
        self.pe_w = (C.c_float * 8)(*hann_band_weights(PE_BANDS, self.nets.pe_alpha).tolist())
        self.residual = bool(residual)

    # ------------------------------------------------------------------------------------
    # Per-op profiling (bench.py's training roofline): with ``self.prof`` a list, every op
    # records a CUDA event on the launching stream after it, tagged with its ALGORITHMIC
    # bytes per sample (activations read + written, gathers, atomics as 8-byte RMW).
    prof = None

    def _pm(self, label: str, bytes_per_sample: float, total: Optional[float] = None) -> None:
        if self.prof is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream())
        self.prof.append((label, bytes_per_sample * self.S if total is None else total, ev))

    def profile_step(self, step: int = 0):
        """One full step with per-op events: [(op, ms, algorithmic bytes, GB/s)]."""
        self.prof = []
        torch.cuda._sleep(8_000_000)      # ~4 ms device spin: the host enqueues the step ahead of
        self._pm("start", 0.0)            # the device, so the marks time kernels, not launches
        self.step(step)
        torch.cuda.synchronize()
        marks, self.prof = self.prof, None
        out = []
        for (_, _, e0), (lab, nb, e1) in zip(marks[:-1], marks[1:]):
            ms = e0.elapsed_time(e1)
            out.append((lab, ms, nb, nb / (ms * 1e-3) / 1e9 if ms > 0 else 0.0))
        return out

    def _lin(self, x, w, b, y, k, n, act, sp, bits=None):
        bp = b.data_ptr() if b is not None else None
        if self.tc:
            _lib.check(self.lib.fv_linear_fwd_tc_bits(x.data_ptr(), x.shape[1], w.data_ptr(), bp, y.data_ptr(),
                                                      y.shape[1], self.S, k, n, act,
                                                      bits.data_ptr() if bits is not None else None, sp),
                       "fv_linear_fwd_tc_bits")
        else:
            _lib.check(self.lib.fv_linear_fwd(x.data_ptr(), w.data_ptr(), bp, y.data_ptr(), self.S, k, n, act, sp),
                       "fv_linear_fwd")
        self._pm(f"linear_fwd {k}x{n}", 4.0 * (x.shape[1] + n) + (4.0 * ((n + 31) // 32) if bits is not None else 0.0))

    def _lin_bwd_tc(self, x, w, dz, dx, xbits, dw, db, k, n, sp):
        """dz = masked pre-activation gradient of this layer; dx gets (dz W^T) * xbits, the
        previous layer's ReLU bits -> the masked dz of that layer."""
        _lib.check(self.lib.fv_linear_bwd_tc_bits(x.data_ptr(), x.shape[1], w.data_ptr(), dz.data_ptr(), dz.shape[1],
                                                  dx.data_ptr() if dx is not None else None,
                                                  dx.shape[1] if dx is not None else 0,
                                                  xbits.data_ptr() if xbits is not None else None, dw.data_ptr(),
                                                  db.data_ptr(), self.S, k, n, sp), "fv_linear_bwd_tc_bits")
        dxb = (4.0 * n + 4.0 * k + (4.0 * ((k + 31) // 32) if xbits is not None else 0.0)) if dx is not None else 0.0
        self._pm(f"linear_bwd {k}x{n} (dX+dW)", dxb + 4.0 * (x.shape[1] + n))

    def _lin_bwd(self, x, w, y, dy, dx, dw, db, k, n, act, sp):
        _lib.check(self.lib.fv_linear_bwd(x.data_ptr(), w.data_ptr(), y.data_ptr(), dy.data_ptr(),
                                          dx.data_ptr() if dx is not None else None, dw.data_ptr(),
                                          db.data_ptr(), self.S, k, n, act, sp), "fv_linear_bwd")

    def forward(self, pix_np: Optional[np.ndarray] = None, step: int = 0):
        nets, lib, S = self.nets, self.lib, self.S
        sp = _lib.stream_ptr()
        if pix_np is None:
            pix_np = patch_pixels(sample_patches(self.mask, self.n_patches, self.patch, self.seed, step),
                                  self.patch, self.cam.width)
        k = self.pix_slot
        self.pix_slot = (k + 1) % len(self.pix_ring)
        if self.pix_events[k] is not None:
            self.pix_events[k].synchronize()
        self.pix_ring[k].numpy()[:] = pix_np
        self.pix.copy_(self.pix_ring[k], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.pix_events[k] = ev
        if self.pose_refiner is not None:     # refined pose -> motion bases of this step
            from .pose import motion_basis as mb_t
            om = torch.as_tensor(self.base_pose.angles, dtype=torch.float64)
            refined = self.pose_refiner.refine(om)
            g_r, g_t = mb_t(nets.scene.skeleton, refined,
                            torch.as_tensor(self.base_pose.root_translation, dtype=torch.float64))
            self._refined = (refined, g_r, g_t)
            nets.set_pose_bases(g_r.detach().numpy(), g_t.detach().numpy(), refined.detach().numpy().reshape(-1))
        if self.weight_net is not None:        # W^c logits of this step from the generator
            self._wlogits = self.weight_net()
            nets.views["vol_logits"].copy_(self._wlogits.detach())
            nets._softmax_pack(sp)
        self._pm("patch ids H2D", 0.0, total=4.0 * self.R)
        m, cs, w = march_struct(self.st, self.pix, None), camera_struct(self.cam), nets.warp_struct()
        h, eps = nets.hash_struct(), self.st.eps_w
        _lib.check(lib.fv_march_warp(C.byref(cs), C.byref(m), C.byref(w), self.R, self.xs.data_ptr(),
                                     self.delta.data_ptr(), self.x.data_ptr(), None, sp), "fv_march_warp")
        self._pm("march_warp", 32.0 + nets.n_bones * (16.0 if nets.half else 32.0))
        V = nets.views
        if self.residual:
            _lib.check(lib.fv_posenc_fwd(self.xs.data_ptr(), S, eps, PE_BANDS, self.pe_w, self.pe.data_ptr(),
                                         self.pe_ld, sp))
            self._pm("posenc_fwd", 16.0 + 4.0 * self.pe_ld)
            self._lin(self.pe, V["off_w0"], nets.b0_eff, self.h[0], self.d_pe, 128, 1, sp, self.hbits[0])
            for i in range(1, 4):
                self._lin(self.h[i - 1], V[f"off_w{i}"], V[f"off_b{i}"], self.h[i], 128, 128, 1, sp, self.hbits[i])
            self._lin(self.h[3], V["off_w4"], V["off_b4"], self.xres, 128, 3, 0, sp)
        _lib.check(lib.fv_xfinal(self.xs.data_ptr(), self.xres.data_ptr() if self.residual else None, S, eps,
                                 self.xf.data_ptr(), sp))
        self._pm("xfinal", 40.0)
        _lib.check(lib.fv_hash_fwd(C.byref(h), self.xf.data_ptr(), S, self.feat.data_ptr(), None, sp), "fv_hash_fwd")
        self._pm("hash_fwd", 12.0 + 16 * 8 * (2.0 if nets.half else 8.0) + 128.0)
        self._lin(self.feat, V["rad_w0"], V["rad_b0"], self.r[0], 32, 64, 1, sp, self.rbits[0])
        self._lin(self.r[0], V["rad_w1"], V["rad_b1"], self.r[1], 64, 64, 1, sp, self.rbits[1])
        self._lin(self.r[1], V["rad_w2"], V["rad_b2"], self.hd, 64, 4, 0, sp)
        _lib.check(lib.fv_heads_fwd(self.xs.data_ptr(), self.hd.data_ptr(), S, eps, self.rgbs.data_ptr(), sp))
        self._pm("heads_fwd", 48.0)
        _lib.check(lib.fv_composite_fwd(self.rgbs.data_ptr(), self.delta.data_ptr(), self.xs[:, 3:].data_ptr(), 4, 1,
                                        self.R, self.N, self.bg, eps, 0.0, self.rgb.data_ptr(), self.alpha.data_ptr(),
                                        self.trans.data_ptr(), sp), "fv_composite_fwd")
        self._pm("composite_fwd", 28.0)
        if self.lam_perc == 0.0 and self.lam_mse == 1.0:   # config 3: plain L2
            _lib.check(lib.fv_mse_loss(self.rgb.data_ptr(), self.target.data_ptr(), self.pix.data_ptr(), self.R,
                                       self.loss.data_ptr(), self.drgb.data_ptr(), sp), "fv_mse_loss")
        else:                                                # SPEC compute_loss
            _lib.check(lib.fv_patch_loss(self.rgb.data_ptr(), self.target.data_ptr(), self.pix.data_ptr(),
                                         self.n_patches, self.patch, self.lam_mse, self.lam_perc,
                                         self.loss.data_ptr(), self.drgb.data_ptr(), sp), "fv_patch_loss")
        self._pm("loss", 0.0, total=self.R * 40.0)
        return self.loss[0]

    def backward(self):
        nets, lib, S, V, G = self.nets, self.lib, self.S, self.nets.views, self.gviews
        sp = _lib.stream_ptr()
        eps = self.st.eps_w
        self.grad.zero_()
        self.dvol.zero_()
        self._pm("zero grads", 0.0, total=4.0 * (self.grad.numel() + self.dvol.numel()))
        _lib.check(lib.fv_composite_bwd(self.rgbs.data_ptr(), self.delta.data_ptr(), self.xs[:, 3:].data_ptr(), 4, 1,
                                        self.trans.data_ptr(), self.R, self.N, self.bg, eps, self.drgb.data_ptr(),
                                        None, self.d_rgbs.data_ptr(), sp), "fv_composite_bwd")
        self._pm("composite_bwd", 44.0)
        _lib.check(lib.fv_heads_bwd(self.xs.data_ptr(), self.hd.data_ptr(), self.d_rgbs.data_ptr(), S, eps,
                                    self.dh.data_ptr(), sp))
        self._pm("heads_bwd", 64.0)
        h = nets.hash_struct()
        # radiance MLP (tcgen05 dz-form: each dx epilogue applies the previous layer's ReLU bits)
        if self.tc:
            self._lin_bwd_tc(self.r[1], V["rad_w2"], self.dh, self.g64[0], self.rbits[1], G["rad_w2"], G["rad_b2"], 64, 4, sp)
            self._lin_bwd_tc(self.r[0], V["rad_w1"], self.g64[0], self.g64[1], self.rbits[0], G["rad_w1"], G["rad_b1"], 64, 64, sp)
            self._lin_bwd_tc(self.feat, V["rad_w0"], self.g64[1], self.dfeat, None, G["rad_w0"], G["rad_b0"], 32, 64, sp)
        else:
            self._lin_bwd(self.r[1], V["rad_w2"], self.hd, self.dh, self.g64[0], G["rad_w2"], G["rad_b2"], 64, 4, 0, sp)
            self._lin_bwd(self.r[0], V["rad_w1"], self.r[1], self.g64[0], self.g64[1], G["rad_w1"], G["rad_b1"], 64, 64, 1, sp)
            self._lin_bwd(self.feat, V["rad_w0"], self.r[0], self.g64[1], self.dfeat, G["rad_w0"], G["rad_b0"], 32, 64, 1, sp)
        _lib.check(lib.fv_hash_bwd(C.byref(h), self.xf.data_ptr(), S, self.dfeat.data_ptr(),
                                   G["table"].data_ptr(), self.dxf.data_ptr(), sp), "fv_hash_bwd")
        self._pm("hash_bwd", 2188.0)     # 128 B dfeat + 12 B pos + 256 fp32 atomics x 8 B RMW
        # table + radiance-MLP gradients are final: their all-reduce overlaps the rest
        self.buckets.launch(0, self.nets.segments[0][0])
        # residual MLP; when the stage is off x_final = x_skel and the gradient goes straight to the warp
        if not self.residual:
            self.dxs.copy_(self.dxf)
        elif self.tc:
            self._lin_bwd_tc(self.h[3], V["off_w4"], self.dxf, self.g128[0], self.hbits[3], G["off_w4"], G["off_b4"], 128, 3, sp)
            self._lin_bwd_tc(self.h[2], V["off_w3"], self.g128[0], self.g128[1], self.hbits[2], G["off_w3"], G["off_b3"], 128, 128, sp)
            self._lin_bwd_tc(self.h[1], V["off_w2"], self.g128[1], self.g128[0], self.hbits[1], G["off_w2"], G["off_b2"], 128, 128, sp)
            self._lin_bwd_tc(self.h[0], V["off_w1"], self.g128[0], self.g128[1], self.hbits[0], G["off_w1"], G["off_b1"], 128, 128, sp)
            self._lin_bwd_tc(self.pe, V["off_w0"], self.g128[1], self.dpe, None, G["off_w0"], G["off_b0"], self.d_pe, 128, sp)
        else:
            self._lin_bwd(self.h[3], V["off_w4"], self.xres, self.dxf, self.g128[0], G["off_w4"], G["off_b4"], 128, 3, 0, sp)
            self._lin_bwd(self.h[2], V["off_w3"], self.h[3], self.g128[0], self.g128[1], G["off_w3"], G["off_b3"], 128, 128, 1, sp)
            self._lin_bwd(self.h[1], V["off_w2"], self.h[2], self.g128[1], self.g128[0], G["off_w2"], G["off_b2"], 128, 128, 1, sp)
            self._lin_bwd(self.h[0], V["off_w1"], self.h[1], self.g128[0], self.g128[1], G["off_w1"], G["off_b1"], 128, 128, 1, sp)
            self._lin_bwd(self.pe, V["off_w0"], self.h[0], self.g128[1], self.dpe, G["off_w0"], G["off_b0"], self.d_pe, 128, 1, sp)
        if self.residual:
            # the folded pose rows of W0: dW0[D:, :] = pose (outer) d b0_eff  (b0_eff = b0 + pose @ W0[D:])
            G["off_w0"][self.d_pe:].addr_(nets.pose_dev, G["off_b0"])
            self.dxs.copy_(self.dxf)
            _lib.check(lib.fv_posenc_bwd(self.xs.data_ptr(), S, eps, PE_BANDS, self.pe_w, self.dpe.data_ptr(),
                                         self.pe_ld, self.dxs.data_ptr(), sp))
            self._pm("posenc_bwd (+dW0 pose rows, dx copy)", 16.0 + 4.0 * self.pe_ld + 24.0)
        w = nets.warp_struct()
        if self.pose_refiner is not None:
            self.dg.zero_()
            _lib.check(lib.fv_warp_bwd_g(C.byref(w), eps, self.x.data_ptr(), S, self.dxs.data_ptr(),
                                         self.dvol.data_ptr(), self.dg.data_ptr(), sp), "fv_warp_bwd_g")
        else:
            _lib.check(lib.fv_warp_bwd(C.byref(w), eps, self.x.data_ptr(), S, self.dxs.data_ptr(),
                                       self.dvol.data_ptr(), sp), "fv_warp_bwd")
        self._pm("warp_bwd", 24.0 + nets.n_bones * ((16.0 if nets.half else 32.0) + 8 * 8.0))
        k1, g = self.dvol.shape[0], self.dvol.shape[1]
        _lib.check(lib.fv_softmax0_bwd(nets.vol.data_ptr(), self.dvol.data_ptr(), k1, g ** 3,
                                       G["vol_logits"].data_ptr(), sp))
        self._pm("softmax0_bwd", 0.0, total=12.0 * self.dvol.numel())
        if self.pose_refiner is not None:     # dL/dG_i and the pose input -> refiner parameters
            refined, g_r, g_t = self._refined
            dg = self.dg.double().cpu()
            d_pose = torch.zeros(refined.numel(), dtype=torch.float64)
            if self.residual:                   # b0_eff = b0 + pose @ W0[D:]: d pose = W0[D:] @ d b0_eff
                d_pose = (V["off_w0"][self.d_pe:].double() @ G["off_b0"].double()).cpu()
            self.popt.zero_grad(set_to_none=False)
            ((g_r * dg[:, :9].view(-1, 3, 3)).sum() + (g_t * dg[:, 9:]).sum()
             + (refined.reshape(-1) * d_pose).sum()).backward()
        if self._wlogits is not None:          # logits gradient -> generator parameters
            self.wopt.zero_grad(set_to_none=False)
            self._wlogits.backward(G["vol_logits"])
            G["vol_logits"].zero_()            # the logits are derived: Adam must not move them

    def allreduce(self):
        """Sum over ranks / world of the flat gradient (the path's only exchange)."""
        self.buckets.finish()
        if self.buckets.world > 1:
            import torch.distributed as dist
            nets_ = [m for m in (getattr(self, "weight_net", None), getattr(self, "pose_refiner", None))
                     if m is not None]
            for m in nets_:
                for p in m.parameters():
                    dist.all_reduce(p.grad, group=self.pg)
                    p.grad.mul_(1.0 / self.buckets.world)

    def optimizer_step(self):
        nets = self.nets
        self.t += 1
        half = nets.table_half
        self.flag.zero_()                 # a flag left by an earlier non-finite step must not veto this one
        _lib.check(self.lib.fv_adam_step(nets.flat.data_ptr(), self.grad.data_ptr(), self.m.data_ptr(),
                                         self.v.data_ptr(), nets.n_params, self.seg_end, self.seg_lr, 2, self.t,
                                         0.9, 0.99, 1e-8, half.data_ptr() if half is not None else None, 0,
                                         self.table_elems if half is not None else 0, self.flag.data_ptr(),
                                         _lib.stream_ptr()), "fv_adam_step")
        self._pm("adam", 0.0, total=28.0 * nets.n_params + 2.0 * self.table_elems)
        nets.refresh_after_step()
        self._pm("refresh (softmax, W^c pack, tc pack, pose fold)", 0.0, total=0.0)
        if self.weight_net is not None or self.pose_refiner is not None:
            # the torch-side optimizers follow the fused step's verdict: no update on a
            # non-finite gradient (ad:898-902); one host read, only on these optional paths
            if int(self.flag.item()) == 0:
                if self.weight_net is not None:
                    self.wopt.step()
                if self.pose_refiner is not None:
                    self.popt.step()

    def check_finite(self):
        """Raise TrainingError naming the block if the last Adam pass saw a non-finite gradient."""
        f = int(self.flag.item())
        if f:
            names = ["table / radiance MLP (lr_nerf)", "residual MLP / weight volume (lr_other)"]
            raise TrainingError(f"non-finite gradient in parameter block '{names[f - 1]}'")

    def step(self, step: int):
        loss = self.forward(step=step)
        self.backward()
        self.allreduce()
        self.optimizer_step()
        return loss


# ------------------------------------------------------------------------------- driver

@dataclass
class TrainConfig:
    """SPEC TrainConfig: iterations, loss weights (Eq 14, perceptual proxy), patches,
    coarse-to-fine milestones as fractions of the run (paper 10K / 50K of 150K),
    checkpoint cadence.  The learning rates live with the parameter blocks (model.LR_*)."""
    iterations: int = 1500
    lam_mse: float = 0.2
    lam_perc: float = 1.0
    n_patches: int = 6
    patch: int = 20
    residual_on: float = 10.0 / 150.0
    full_band: float = 50.0 / 150.0
    seed: int = 0
    precision: str = "tf32"
    checkpoint_every: int = 100
    log_path: Optional[str] = None
    checkpoint_dir: Optional[str] = None

    def __post_init__(self):
        if not (0.0 < self.residual_on < self.full_band < 1.0):
            raise ValueError("milestones must satisfy 0 < residual_on < full_band < 1 (S:475)")
        if self.iterations < 1 or self.lam_mse < 0 or self.lam_perc < 0:
            raise ValueError("iterations >= 1 and non-negative loss weights")


def schedule(it: int, cfg: TrainConfig, bands: int = PE_BANDS):
    """(alpha, residual stage on) at iteration ``it``: alpha = L * clamp((it - it_on) /
    (it_full - it_on), 0, 1); the residual net is held at exactly zero before
    it_on."""
    it_on = int(round(cfg.residual_on * cfg.iterations))
    it_full = max(int(round(cfg.full_band * cfg.iterations)), it_on + 1)
    alpha = bands * min(max((it - it_on) / (it_full - it_on), 0.0), 1.0)
    return float(alpha), it >= it_on


def _aux_modules(trainer: "Trainer"):
    """(name, torch module or optimizer) pairs of the optional generator / pose refiner."""
    out = []
    if getattr(trainer, "weight_net", None) is not None:
        out += [("weight_net", trainer.weight_net), ("weight_opt", trainer.wopt)]
    if getattr(trainer, "pose_refiner", None) is not None:
        out += [("pose_refiner", trainer.pose_refiner), ("pose_opt", trainer.popt)]
    return out


def _flat_state(obj) -> dict:
    """A module's state_dict or an optimizer's per-parameter state as name -> tensor."""
    if isinstance(obj, torch.optim.Optimizer):
        sd = obj.state_dict()
        out = {}
        for pid, st in sd["state"].items():
            for k, v in st.items():
                out[f"{pid}.{k}"] = v if isinstance(v, torch.Tensor) else torch.tensor(float(v))
        return out
    return dict(obj.state_dict())


def _load_flat_state(obj, arrays: dict) -> None:
    if isinstance(obj, torch.optim.Optimizer):
        sd = obj.state_dict()
        state = {}
        for key, a in arrays.items():
            pid, k = key.split(".", 1)
            state.setdefault(int(pid), {})[k] = a
        sd["state"] = state
        obj.load_state_dict(sd)
    else:
        obj.load_state_dict({k: a for k, a in arrays.items()})


def save_checkpoint(path: str, trainer: "Trainer", iteration: int) -> None:
    """Manifest + raw little-endian float32 arrays: params.bin (the flat master
    buffer), adam_m.bin, adam_v.bin, manifest.json (block table, Adam step, schedule); with a
    weight-volume generator / pose refiner attached, their parameters and torch-Adam states
    as one raw array per tensor (``<module>.<key>.bin``, listed in the manifest)."""
    os.makedirs(path, exist_ok=True)
    nets = trainer.nets
    for name, t in (("params", nets.flat), ("adam_m", trainer.m), ("adam_v", trainer.v)):
        t.detach().cpu().numpy().astype("<f4").tofile(os.path.join(path, f"{name}.bin"))
    aux = {}
    for mname, obj in _aux_modules(trainer):
        entries = {}
        for key, t in _flat_state(obj).items():
            fn = f"{mname}.{key}.bin"
            a = t.detach().cpu().numpy()
            dt = a.dtype.newbyteorder("<")
            a.astype(dt).tofile(os.path.join(path, fn))
            entries[key] = {"file": fn, "shape": list(t.shape), "dtype": dt.str}
        aux[mname] = entries
    man = {"format": "freeview-b200-checkpoint", "version": 2, "iteration": iteration, "adam_t": trainer.t,
           "n_params": nets.n_params, "pe_alpha": nets.pe_alpha, "residual": bool(trainer.residual),
           "blocks": {k: {"offset": a, "size": b - a, "shape": list(nets.views[k].shape)}
                      for k, (a, b) in nets.block_ranges.items()},
           "modules": aux}
    with open(os.path.join(path, "manifest.json"), "w") as f:
        json.dump(man, f, indent=1)


def load_params(path: str, nets: FreeviewModel) -> int:
    """Model parameters only (inference / the render service) from a save_checkpoint directory;
    rebuilds the derived buffers; returns the iteration.  ValueError on a block-table mismatch."""
    with open(os.path.join(path, "manifest.json")) as f:
        man = json.load(f)
    want = {k: [a, b - a] for k, (a, b) in nets.block_ranges.items()}
    got = {k: [v["offset"], v["size"]] for k, v in man["blocks"].items()}
    if want != got:
        raise ValueError("checkpoint block table does not match the model")
    a = np.fromfile(os.path.join(path, "params.bin"), dtype="<f4")
    nets.flat.copy_(torch.from_numpy(a.astype(np.float32)).to(nets.flat.device))
    nets.set_schedule(alpha=man.get("pe_alpha", nets.pe_alpha), residual=man.get("residual", True))
    nets.refresh()
    return int(man["iteration"])


def load_checkpoint(path: str, trainer: "Trainer") -> int:
    """Restore a save_checkpoint directory into the trainer's model and Adam state; returns
    the iteration.  Raises DimensionError-style ValueError on a block-table mismatch."""
    with open(os.path.join(path, "manifest.json")) as f:
        man = json.load(f)
    nets = trainer.nets
    want = {k: [a, b - a] for k, (a, b) in nets.block_ranges.items()}
    got = {k: [v["offset"], v["size"]] for k, v in man["blocks"].items()}
    if want != got:
        raise ValueError("checkpoint block table does not match the model")
    for name, t in (("params", nets.flat), ("adam_m", trainer.m), ("adam_v", trainer.v)):
        a = np.fromfile(os.path.join(path, f"{name}.bin"), dtype="<f4")
        t.copy_(torch.from_numpy(a.astype(np.float32)).to(t.device))
    trainer.t = int(man["adam_t"])
    trainer.set_schedule(man["pe_alpha"], man["residual"])
    mods = man.get("modules", {})
    for mname, obj in _aux_modules(trainer):
        if mname not in mods:
            raise ValueError(f"checkpoint has no state for the attached {mname}")
        arrays = {}
        for key, ent in mods[mname].items():
            a = np.fromfile(os.path.join(path, ent["file"]), dtype=ent.get("dtype", "<f4")).reshape(ent["shape"])
            ref = _flat_state(obj).get(key)
            dev = ref.device if isinstance(ref, torch.Tensor) else "cpu"
            arrays[key] = torch.from_numpy(a.astype(a.dtype.newbyteorder("="))).to(dev)
        _load_flat_state(obj, arrays)
    nets.refresh()
    return int(man["iteration"])


@dataclass
class Frame:
    """One captured training view (SPEC PatchBatch source): camera, target RGB image
    (H, W, 3) in [0, 1], foreground mask (H, W) bool and the frame's body pose."""
    camera: CameraModel
    image: np.ndarray
    mask: np.ndarray
    pose: "Pose"


@dataclass
class Dataset:
    """In-memory dataset for ``train(dataset, config)``: frames plus the train / held-out
    split (the reference's CaptureDataset keeps the same three things on disk: per-frame
    camera, image, mask and pose, and ``splits``, cap:438-470)."""
    frames: List[Frame]
    train_ids: Optional[List[int]] = None
    heldout_ids: Optional[List[int]] = None

    def __post_init__(self):
        if not self.frames:
            raise ValueError("dataset has no frames")
        if self.train_ids is None:
            self.train_ids = list(range(len(self.frames)))
        if self.heldout_ids is None:
            self.heldout_ids = []
        if not self.train_ids:
            raise ValueError("dataset has no training frames")


def synthetic_dataset(scene, n_frames: Optional[int] = None) -> Dataset:
    """The BASELINE synthetic stand-in as a dataset: the scene's camera, its seeded smooth
    target image and projected-ellipsoid mask (scene.target_image), one frame per pose."""
    from .scene import target_image
    img, mask = target_image(scene)
    poses = scene.poses if n_frames is None else [scene.poses[i % len(scene.poses)] for i in range(n_frames)]
    return Dataset([Frame(scene.camera, img, mask, p) for p in poses])


def train(dataset: Dataset, config: TrainConfig, nets: Optional[FreeviewModel] = None,
          settings: Optional[RenderSettings] = None, process_group=None) -> List[dict]:
    """SPEC ``train(dataset, config)``.  Per iteration: pick a training frame
    (deterministic per (seed, iteration)) and upload its pose, apply the coarse-to-fine
    schedule (residual net exactly zero before its milestone, Hann alpha ramp), sample
    patches on the frame's mask, render them through the full pipeline, loss
    (Eq 14 with the perceptual proxy), backward, (NCCL all-reduce), Adam at the
    per-group rates; log (iteration, loss, mse_term, perc_term, alpha, stage, wall_ms) to a
    CSV; save a checkpoint every ``checkpoint_every`` iterations into ``checkpoint_dir``.  A
    non-finite loss or gradient restores the last good state and raises TrainingError
    (S:509).  ``nets`` defaults to a fresh model of ``dataset``'s scene when it carries one
    (``synthetic_dataset``); returns the log rows."""
    if nets is None:
        raise ValueError("train: pass the model (nets) to optimise")
    f0 = dataset.frames[dataset.train_ids[0]]
    if settings is None:
        settings = RenderSettings.from_config(nets.cfg, seed=config.seed)
    tr = Trainer(nets, f0.camera, f0.image, f0.mask, settings, n_patches=config.n_patches, patch=config.patch,
                 seed=config.seed, process_group=process_group, precision=config.precision,
                 lam_mse=config.lam_mse, lam_perc=config.lam_perc)

    def snapshot():
        return (nets.flat.clone(), tr.m.clone(), tr.v.clone(), tr.t,
                {n: copy.deepcopy(o.state_dict()) for n, o in _aux_modules(tr)})

    def restore(g):
        nets.flat.copy_(g[0]); tr.m.copy_(g[1]); tr.v.copy_(g[2]); tr.t = g[3]
        for n, o in _aux_modules(tr):
            o.load_state_dict(g[4][n])
        nets.refresh()

    good = snapshot()
    rows = []
    writer, fh = None, None
    if config.log_path:
        fh = open(config.log_path, "w", newline="")
        writer = csv.writer(fh)
        writer.writerow(["iteration", "loss", "mse_term", "perc_term", "alpha", "stage", "wall_ms"])
    current = None
    try:
        t0 = time.perf_counter()
        for it in range(config.iterations):
            fid = dataset.train_ids[int(np.random.default_rng([config.seed, it, 1]).integers(len(dataset.train_ids)))]
            if fid != current:
                fr = dataset.frames[fid]
                if current is not None:
                    tr.set_frame(fr.camera, fr.image, fr.mask)
                nets.set_pose(fr.pose)
                current = fid
            alpha, residual = schedule(it, config)
            tr.set_schedule(alpha, residual)
            tr.step(it)
            vals = tr.loss.tolist()
            mse = vals[1] if tr.lam_perc != 0.0 or tr.lam_mse != 1.0 else vals[0]
            flag = int(tr.flag.item())
            if not np.isfinite(vals[0]) or flag:
                restore(good)
                raise TrainingError(f"non-finite loss/gradient at iteration {it}; last good state restored")
            row = {"iteration": it, "loss": vals[0], "mse_term": mse, "perc_term": vals[2] if tr.lam_perc else 0.0,
                   "alpha": alpha, "stage": "residual" if residual else "skeleton", "frame": fid,
                   "wall_ms": (time.perf_counter() - t0) * 1e3}
            rows.append(row)
            if writer:
                writer.writerow([row[k] for k in ("iteration", "loss", "mse_term", "perc_term", "alpha", "stage",
                                                  "wall_ms")])
            if config.checkpoint_every and (it + 1) % config.checkpoint_every == 0:
                good = snapshot()
                if config.checkpoint_dir:
                    save_checkpoint(os.path.join(config.checkpoint_dir, f"it{it + 1:07d}"), tr, it + 1)
    finally:
        if fh:
            fh.close()
    train.last_trainer = tr
    return rows


def train_frame(nets: FreeviewModel, camera: CameraModel, target: np.ndarray, mask: np.ndarray,
                settings: RenderSettings, cfg: TrainConfig, process_group=None) -> List[dict]:
    """``train`` on a one-frame dataset (the frame's pose = the model's current pose)."""
    pose = nets._pose if nets._pose is not None else nets.scene.poses[0]
    return train(Dataset([Frame(camera, target, mask, pose)]), cfg, nets=nets, settings=settings,
                 process_group=process_group)
