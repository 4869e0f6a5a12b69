"""GPU-resident network state ("nets" of the SPEC render/train API) and the parameter
blocks handed to libfvcuda.

All trainable parameters live in ONE flat fp32 master buffer (views per block) so the
fused Adam kernel updates everything in a single pass; derived device buffers are
rebuilt by :meth:`FreeviewModel.refresh` after every parameter change:
  * weight volume  W^c = softmax0(logits) -> corner-packed fp32/fp16 volume (fv_warp_pack)
  * fp16 copy of the hash table (config 2/3)
  * fp16 tcgen05 weight pack of both MLPs (fv_field_pack)
Per frame, :meth:`set_pose` uploads the 24 motion bases G_i and folds the 72-d pose
term of the residual MLP's first layer into a per-frame bias (fv_offset_bias).
"""

from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import _lib
from .scene import PE_BANDS, Scene
from .skeleton import Pose, motion_basis, pack_g

LR_NERF = 5e-4   # hash table + radiance MLP
LR_OTHER = 5e-5  # residual MLP + weight-volume logits


def hann_band_weights(num_bands: int, alpha: float) -> np.ndarray:
    """Truncated raised-cosine band weights (ad:574-578), float32."""
    k = np.arange(num_bands, dtype=np.float32)
    x = np.clip(np.float32(alpha) - k, 0.0, 1.0).astype(np.float32)
    return ((np.float32(1.0) - np.cos(np.float32(np.pi) * x)) / np.float32(2.0)).astype(np.float32)


class FreeviewModel:
    """Device-resident parameters of the warp, residual MLP, hash grid and radiance MLP."""

    def __init__(self, scene: Scene, device: str = "cuda", precision: Optional[int] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("FreeviewModel needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.scene = scene
        cfg = scene.cfg
        self.cfg = cfg
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.half = bool(cfg.half)
        self.precision = (1 if self.half else 0) if precision is None else int(precision)
        self.n_bones = cfg.n_bones
        self.vol_res = cfg.vol_res
        # ---- flat fp32 master buffer; segment 0 = lr_nerf blocks, segment 1 = lr_other
        blocks: List[Tuple[str, np.ndarray]] = [("table", scene.table)]
        blocks += [(f"rad_w{i}", w) for i, w in enumerate(scene.rad_w)]
        blocks += [(f"rad_b{i}", b) for i, b in enumerate(scene.rad_b)]
        nerf_end = sum(a.size for _, a in blocks)
        blocks += [(f"off_w{i}", w) for i, w in enumerate(scene.off_w)]
        blocks += [(f"off_b{i}", b) for i, b in enumerate(scene.off_b)]
        blocks += [("vol_logits", scene.vol_logits)]
        total = sum(a.size for _, a in blocks)
        host = np.concatenate([np.asarray(a, np.float32).reshape(-1) for _, a in blocks])
        self.flat = torch.from_numpy(host).to(self.device)
        self.views: Dict[str, torch.Tensor] = {}
        self.block_ranges: Dict[str, Tuple[int, int]] = {}
        off = 0
        for name, a in blocks:
            self.views[name] = self.flat[off:off + a.size].view(*a.shape)
            self.block_ranges[name] = (off, off + a.size)
            off += a.size
        self.segments = [(nerf_end, LR_NERF), (total, LR_OTHER)]
        self.n_params = total
        # ---- derived buffers
        k, g = self.n_bones, self.vol_res
        self.vol = torch.empty((k + 1, g, g, g), device=self.device, dtype=torch.float32)
        self.vol_packed = torch.empty(k * (g + 1) ** 3 * 8, device=self.device,
                                      dtype=torch.float16 if self.half else torch.float32)
        self.table_half = (torch.empty(scene.table.shape, device=self.device, dtype=torch.float16)
                           if self.half else None)
        self.tc_pack = (torch.empty(self.lib.fv_field_pack_bytes(), device=self.device, dtype=torch.uint8)
                        if self.precision == 1 else None)
        self.g = torch.zeros((k, 12), device=self.device, dtype=torch.float32)
        self.pose_dev = torch.zeros(3 * k, device=self.device, dtype=torch.float32)
        self.b0_eff = torch.zeros(128, device=self.device, dtype=torch.float32)
        self._pin, self._pin_ev, self._pin_slot = None, None, 0   # pinned pose-upload ring
        self.pe_alpha = float(PE_BANDS)
        self.offset_enabled = True
        self._pose: Optional[Pose] = None
        self.refresh()
        self.set_pose(scene.poses[0])

    # ------------------------------------------------------------------ parameter blocks
    def _wscale(self) -> np.ndarray:
        s = self.scene
        return (np.float32(self.vol_res - 1) / (s.wbox_max.astype(np.float32) - s.wbox_min.astype(np.float32))).astype(np.float32)

    def warp_struct(self) -> _lib.FvWarp:
        w = _lib.FvWarp()
        w.n_bones, w.vol_res, w.vol_half = self.n_bones, self.vol_res, int(self.half)
        w.d_vol_packed = self.vol_packed.data_ptr()
        w.d_g = self.g.data_ptr()
        _lib.farr(w.wbox_min, self.scene.wbox_min.astype(np.float32))
        _lib.farr(w.wscale, self._wscale())
        return w

    def hash_struct(self, table: Optional[torch.Tensor] = None) -> _lib.FvHash:
        hc = self.cfg.hash
        h = _lib.FvHash()
        h.n_levels, h.n_feat, h.log2_T = hc.n_levels, hc.n_feat, hc.log2_T
        _lib.farr(h.res, hc.resolutions())
        _lib.farr(h.dense, [int(d) for d in hc.dense()])
        _lib.farr(h.offset, hc.offsets())
        if table is None:
            table = self.table_half if self.half else self.views["table"]
        h.table_half = int(table.dtype == torch.float16)
        h.d_table = table.data_ptr()
        s = self.scene
        _lib.farr(h.cmin, s.wbox_min.astype(np.float32))
        _lib.farr(h.cinv, (1.0 / (s.wbox_max - s.wbox_min)).astype(np.float32))
        return h

    def field_struct(self, precision: Optional[int] = None, offset_enabled: Optional[bool] = None) -> _lib.FvField:
        f = _lib.FvField()
        f.precision = self.precision if precision is None else precision
        f.pe_bands = PE_BANDS
        _lib.farr(f.pe_w, hann_band_weights(PE_BANDS, self.pe_alpha))
        f.offset_enabled = int(self.offset_enabled if offset_enabled is None else offset_enabled)
        for i in range(5):
            f.d_off_w[i] = self.views[f"off_w{i}"].data_ptr()
            f.d_off_b[i] = self.views[f"off_b{i}"].data_ptr()
        for i in range(3):
            f.d_rad_w[i] = self.views[f"rad_w{i}"].data_ptr()
            f.d_rad_b[i] = self.views[f"rad_b{i}"].data_ptr()
        f.d_off_b0_eff = self.b0_eff.data_ptr()
        f.d_tc_pack = self.tc_pack.data_ptr() if self.tc_pack is not None else None
        return f

    # ------------------------------------------------------------------ state updates
    def refresh(self, stream=None) -> None:
        """Rebuild every derived device buffer from the fp32 master parameters."""
        st = _lib.stream_ptr(stream)
        self._softmax_pack(st)
        if self.half:
            self.table_half.copy_(self.views["table"])
        if self.tc_pack is not None:
            f = self.field_struct()
            _lib.check(self.lib.fv_field_pack(C.byref(f), self.tc_pack.data_ptr(), st), "fv_field_pack")
        if self._pose is not None:
            self._fold_pose(st)

    def refresh_after_step(self, stream=None) -> None:
        """After an Adam step (which already rewrote the fp16 table copy): W^c, packs, pose fold."""
        st = _lib.stream_ptr(stream)
        self._softmax_pack(st)
        if self.tc_pack is not None:
            f = self.field_struct()
            _lib.check(self.lib.fv_field_pack(C.byref(f), self.tc_pack.data_ptr(), st), "fv_field_pack")
        if self._pose is not None:
            self._fold_pose(st)

    def _softmax_pack(self, st) -> None:
        k1, g = self.vol.shape[0], self.vol.shape[1]
        _lib.check(self.lib.fv_softmax0_fwd(self.views["vol_logits"].data_ptr(), k1, g ** 3, self.vol.data_ptr(), st),
                   "fv_softmax0_fwd")
        w = self.warp_struct()
        _lib.check(self.lib.fv_warp_pack(self.vol.data_ptr(), self.n_bones + 1, C.byref(w),
                                         self.vol_packed.data_ptr(), st), "fv_warp_pack")

    PIN_SLOTS = 4     # frames the host may run ahead of the device before a slot is reused

    def _upload_pose(self, g_packed: np.ndarray, pose_vec: np.ndarray, stream=None) -> None:
        """G_i and the pose vector -> device through a pinned staging ring (PIN_SLOTS slots)
        with asynchronous copies: the host computes the next frames' motion bases while the
        GPU still renders the current one (a pageable copy would wait for it)."""
        if self._pin is None:
            self._pin = [torch.empty(self.g.numel() + self.pose_dev.numel(), dtype=torch.float32,
                                     pin_memory=True) for _ in range(self.PIN_SLOTS)]
            self._pin_ev = [None] * self.PIN_SLOTS
        k = self._pin_slot
        self._pin_slot = (k + 1) % self.PIN_SLOTS
        if self._pin_ev[k] is not None:
            self._pin_ev[k].synchronize()          # the copy that last used this slot is done
        buf = self._pin[k]
        ng = self.g.numel()
        buf[:ng].numpy()[:] = g_packed.reshape(-1)
        buf[ng:].numpy()[:] = pose_vec.reshape(-1)
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        if st.device != self.device:
            raise ValueError(f"pose upload stream is on {st.device}, the model on {self.device}")
        with torch.cuda.device(self.device), torch.cuda.stream(st):
            self.g.view(-1).copy_(buf[:ng], non_blocking=True)
            self.pose_dev.copy_(buf[ng:], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
        self._pin_ev[k] = ev       # the slot is rewritten only after this event (the H2D read)

    def set_pose(self, pose: Pose, stream=None) -> None:
        """Upload the frame's motion bases G_i and fold the pose into the residual bias."""
        g_r, g_t = motion_basis(self.scene.skeleton, pose)
        self._upload_pose(pack_g(g_r, g_t), pose.flat().astype(np.float32), stream)
        self._pose = pose
        self._fold_pose(_lib.stream_ptr(stream))

    def set_pose_bases(self, g_r: np.ndarray, g_t: np.ndarray, pose_vec: np.ndarray, stream=None) -> None:
        """Upload given motion bases and pose vector (e.g. of a refined pose) and fold the
        pose into the residual bias; the refined pose is remembered for refresh()."""
        self._upload_pose(pack_g(np.asarray(g_r), np.asarray(g_t)), np.asarray(pose_vec, np.float32).reshape(-1),
                          stream)
        self._pose = Pose(np.asarray(pose_vec, np.float64).reshape(-1, 3), np.zeros(3))
        self._fold_pose(_lib.stream_ptr(stream))

    def _fold_pose(self, st) -> None:
        f = self.field_struct()
        _lib.check(self.lib.fv_offset_bias(C.byref(f), self.pose_dev.data_ptr(), 3 * self.n_bones,
                                           self.b0_eff.data_ptr(), st), "fv_offset_bias")

    def set_schedule(self, alpha: Optional[float] = None, residual: Optional[bool] = None) -> None:
        """Coarse-to-fine window alpha and residual stage flag."""
        if alpha is not None:
            self.pe_alpha = float(alpha)
        if residual is not None:
            self.offset_enabled = bool(residual)
