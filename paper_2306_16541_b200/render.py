"""Radiance renderer API (SPEC ``S:387-466``) on the sm_100a path.

``render_image(nets, camera, pose, settings, schedule)`` (``S:438-446``) is one
``fv_render_fwd`` call: ray generation, slab test, stratified jittered sampling,
occupancy skip and skeleton warp (``fv_march_warp``, one thread per sample), the fused
tcgen05 field (residual MLP -> hash grid -> radiance MLP) or its fp32 twin, and the
front-to-back compositor with the likelihood gate and early termination.

The primitive operators of the SPEC are exposed on the same kernels:
``skeleton_warp``, ``query_radiance``, ``composite``,
``warp_point``.  No CPU fallback exists: without libfvcuda.so or a CUDA device
every entry point raises.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np
import torch

from . import _lib
from .camera import CameraModel, tiled_pixel_order
from .errors import DimensionError
from .model import FreeviewModel
from .skeleton import Pose

EPS_W = 1e-4


@dataclass
class RenderSettings:
    """samples per ray, subject box, background, jitter seed, eps_w."""
    n_samples: int = 128
    jitter: bool = True
    seed: int = 0
    eps_w: float = EPS_W
    eps_t: float = 0.0                     # early-termination transmittance (0 = off)
    background: Tuple[float, float, float] = (0.5, 0.5, 0.5)
    box_min: Tuple[float, float, float] = (-1.0, -1.0, -1.0)
    box_max: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    occupancy: bool = False                # build + use the 32^3 skip grid per pose
    occ_threshold: float = 0.01
    round_samples: int = 32                # marching-round size when eps_t > 0

    @classmethod
    def from_config(cls, cfg, **kw) -> "RenderSettings":
        base = dict(n_samples=cfg.n_samples, jitter=cfg.jitter, background=tuple(cfg.background),
                    occupancy=cfg.occupancy)
        base.update(kw)
        return cls(**base)


def camera_struct(cam: CameraModel) -> _lib.FvCamera:
    kinv, rot, ctr = cam.kernel_consts()
    c = _lib.FvCamera()
    _lib.farr(c.kinv, kinv.reshape(-1))
    _lib.farr(c.rot, rot.reshape(-1))
    _lib.farr(c.center, ctr)
    c.width, c.height = cam.width, cam.height
    return c


def march_struct(s: RenderSettings, pix: Optional[torch.Tensor], occ: Optional[torch.Tensor],
                 out_by_pixel: bool = False) -> _lib.FvMarch:
    m = _lib.FvMarch()
    bmin = np.asarray(s.box_min, np.float64)
    bmax = np.asarray(s.box_max, np.float64)
    _lib.farr(m.obox_min, bmin.astype(np.float32))
    _lib.farr(m.obox_max, bmax.astype(np.float32))
    m.n_samples, m.jitter, m.seed = s.n_samples, int(s.jitter), s.seed & 0xFFFFFFFF
    m.eps_w, m.eps_t = s.eps_w, s.eps_t
    _lib.farr(m.bg, s.background)
    m.d_occ = occ.data_ptr() if occ is not None else None
    _lib.farr(m.occ_scale, (32.0 / (bmax - bmin)).astype(np.float32))
    m.d_pix = pix.data_ptr() if pix is not None else None
    m.pix_offset = 0
    m.out_by_pixel = int(out_by_pixel)
    m.round_samples = int(s.round_samples)
    return m


class Renderer:
    """Owns the reusable device workspace, pixel orders and the occupancy bitfield."""

    MAX_SAMPLES_PER_LAUNCH = 1 << 28    # 2048^2 rays x 64 samples; 11.8 GB of workspace

    def __init__(self, device: str = "cuda"):
        self.lib = _lib.load()
        self.device = torch.device(device)
        self._work = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._orders = {}
        self.occ = torch.zeros(1024, dtype=torch.int32, device=self.device)

    def workspace(self, nbytes: int) -> torch.Tensor:
        if self._work.numel() < nbytes:
            self._work = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self._work

    def pixel_order(self, cam: CameraModel) -> torch.Tensor:
        key = (cam.width, cam.height)
        if key not in self._orders:
            self._orders[key] = torch.from_numpy(tiled_pixel_order(cam.width, cam.height)).to(self.device)
        return self._orders[key]

    def build_occupancy(self, nets: FreeviewModel, settings: RenderSettings, stream=None) -> torch.Tensor:
        """fv_occupancy_build for the current pose (32^3 bits over the observation box)."""
        m = march_struct(settings, None, None)
        w, h, f = nets.warp_struct(), nets.hash_struct(), nets.field_struct()
        nb = self.lib.fv_occupancy_workspace_bytes(f.precision)
        work = self.workspace(nb)
        _lib.check(self.lib.fv_occupancy_build(C.byref(m), C.byref(w), C.byref(h), C.byref(f),
                                               settings.occ_threshold, work.data_ptr(), nb,
                                               self.occ.data_ptr(), _lib.stream_ptr(stream)),
                   "fv_occupancy_build")
        return self.occ

    def render_pixels(self, nets: FreeviewModel, cam: CameraModel, pix: torch.Tensor, settings: RenderSettings,
                      out_rgb: Optional[torch.Tensor] = None, out_alpha: Optional[torch.Tensor] = None,
                      counts: Optional[torch.Tensor] = None, by_pixel: bool = False, occ: Optional[torch.Tensor] = None,
                      stream=None):
        """Render the rays of linear pixel ids ``pix`` (int32, device).  Outputs are per ray
        (or written at the pixel id into image-sized buffers when ``by_pixel``)."""
        if pix.dtype != torch.int32 or not pix.is_cuda:
            raise DimensionError("pix must be an int32 CUDA tensor")
        n = pix.numel()
        n_out = cam.width * cam.height if by_pixel else n
        if out_rgb is None:
            out_rgb = torch.empty((n_out, 3), dtype=torch.float32, device=self.device)
        if out_alpha is None:
            out_alpha = torch.empty(n_out, dtype=torch.float32, device=self.device)
        cs = camera_struct(cam)
        w, h, f = nets.warp_struct(), nets.hash_struct(), nets.field_struct()
        # one launch holds at most MAX_SAMPLES_PER_LAUNCH sample slots (sample ids are int32 in
        # the C ABI, and the workspace is ~44 B per slot): larger ray sets go in chunks of
        # whole 32-ray blocks -- jitter is keyed by pixel id, so the pixels are bitwise the same
        per = max(32, self.MAX_SAMPLES_PER_LAUNCH // settings.n_samples // 32 * 32)
        for r0 in range(0, max(n, 1), per):
            r1 = min(n, r0 + per)
            p = pix[r0:r1]
            m = march_struct(settings, p, occ, by_pixel)
            nb = self.lib.fv_render_workspace_bytes(r1 - r0, settings.n_samples, f.precision)
            work = self.workspace(nb)
            o_rgb, o_alpha = (out_rgb, out_alpha) if by_pixel else (out_rgb[r0:r1], out_alpha[r0:r1])
            _lib.check(self.lib.fv_render_fwd(C.byref(cs), C.byref(m), C.byref(w), C.byref(h), C.byref(f), r1 - r0,
                                              work.data_ptr(), nb, o_rgb.data_ptr(), o_alpha.data_ptr(),
                                              counts[r0:r1].data_ptr() if counts is not None else None,
                                              _lib.stream_ptr(stream)), "fv_render_fwd")
        return out_rgb, out_alpha

    def render_image(self, nets: FreeviewModel, cam: CameraModel, pose: Optional[Pose], settings: RenderSettings,
                     out_rgb=None, out_alpha=None, stream=None):
        if pose is not None:
            nets.set_pose(pose, stream)
        occ = self.build_occupancy(nets, settings, stream) if settings.occupancy else None
        pix = self.pixel_order(cam)
        rgb, alpha = self.render_pixels(nets, cam, pix, settings, out_rgb, out_alpha, by_pixel=True, occ=occ,
                                        stream=stream)
        return rgb.view(cam.height, cam.width, 3), alpha.view(cam.height, cam.width)


_DEFAULT = {}


def _renderer(device) -> Renderer:
    key = str(device)
    if key not in _DEFAULT:
        _DEFAULT[key] = Renderer(device)
    return _DEFAULT[key]


def render_image(nets: FreeviewModel, camera: CameraModel, pose: Optional[Pose], settings: RenderSettings,
                 schedule=None):
    """(image (H,W,3), alpha (H,W)) CUDA tensors; deterministic given the jitter seed."""
    if schedule is not None:
        nets.set_schedule(**schedule)
    return _renderer(nets.device).render_image(nets, camera, pose, settings)


# ---------------------------------------------------------------------------------- primitives

def skeleton_warp(nets: FreeviewModel, x: torch.Tensor, eps_w: float = EPS_W):
    """x (n,3) world -> (x_skel (n,3), likelihood (n), fg (n) bool) for the current pose."""
    n = x.shape[0]
    xs = torch.empty((n, 3), dtype=torch.float32, device=x.device)
    lik = torch.empty(n, dtype=torch.float32, device=x.device)
    fg = torch.empty(n, dtype=torch.uint8, device=x.device)
    w = nets.warp_struct()
    _lib.check(nets.lib.fv_warp_fwd(C.byref(w), eps_w, x.contiguous().data_ptr(), n, xs.data_ptr(),
                                    lik.data_ptr(), fg.data_ptr(), None, _lib.stream_ptr()), "fv_warp_fwd")
    return xs, lik, fg.bool()


def _field(nets, xs4, eps_w, offset_enabled, want_xfinal=False):
    n = xs4.shape[0]
    out = torch.empty((n, 4), dtype=torch.float32, device=xs4.device)
    xf = torch.empty((n, 3), dtype=torch.float32, device=xs4.device) if want_xfinal else None
    f = nets.field_struct(offset_enabled=offset_enabled)
    h = nets.hash_struct()
    nb = nets.lib.fv_field_workspace_bytes(n, f.precision)
    work = torch.empty(max(nb, 1), dtype=torch.uint8, device=xs4.device)
    _lib.check(nets.lib.fv_field_fwd(C.byref(f), C.byref(h), xs4.contiguous().data_ptr(), n, eps_w, out.data_ptr(),
                                     xf.data_ptr() if xf is not None else None, work.data_ptr(), nb,
                                     _lib.stream_ptr()), "fv_field_fwd")
    return out, xf


def warp_point(nets: FreeviewModel, x: torch.Tensor, eps_w: float = EPS_W):
    """(x_final (n,3), likelihood (n)) = skeleton warp + residual offset."""
    xs, lik, fg = skeleton_warp(nets, x, eps_w)
    _, xf = _field(nets, torch.cat([xs, lik[:, None]], 1), eps_w, nets.offset_enabled, want_xfinal=True)
    return xf, lik


def positional_encode(p: torch.Tensor, num_bands: int = 6, alpha: Optional[float] = None) -> torch.Tensor:
    """SPEC positional_encode: (n,3) -> (n, 3 + 6 num_bands), Hann-windowed bands
    (alpha defaults to all bands on).  One fv_posenc_fwd launch (autodiff.posenc)."""
    from .autodiff import posenc
    return posenc(p, num_bands, alpha)


def residual_offset(nets: FreeviewModel, x_skel: torch.Tensor, pose: Optional[Pose] = None,
                    alpha: Optional[float] = None, stage: bool = True) -> torch.Tensor:
    """SPEC residual_offset: x_res (n,3) = MLP([posenc_alpha(x_skel), Omega]) with the
    pose columns folded into layer 0's bias (fv_offset_bias; ``pose`` sets the model's pose
    first, else the current one is used); exactly zero when the stage is off.  fp32
    path: the training layer kernels (split-precision 3xTF32 tcgen05, fp32-accurate)."""
    x = x_skel.float().contiguous()
    if x.dim() != 2 or x.shape[1] != 3 or not x.is_cuda:
        raise DimensionError(f"residual_offset: expected CUDA (n, 3), got {tuple(x.shape)}")
    n = x.shape[0]
    if not stage or n == 0:
        return torch.zeros((n, 3), dtype=torch.float32, device=x.device)
    if pose is not None:
        nets.set_pose(pose)
    from .autodiff import posenc
    from .scene import PE_BANDS
    pe = posenc(x, PE_BANDS, nets.pe_alpha if alpha is None else alpha)
    d = pe.shape[1]
    ld = (d + 3) // 4 * 4
    a = torch.zeros((n, ld), dtype=torch.float32, device=x.device)
    a[:, :d] = pe
    lib, sp, V = nets.lib, _lib.stream_ptr(), nets.views
    layers = [(V["off_w0"], nets.b0_eff, d, 128, 1)] + [(V[f"off_w{i}"], V[f"off_b{i}"], 128, 128, 1)
                                                         for i in range(1, 4)] + [(V["off_w4"], V["off_b4"], 128, 3, 0)]
    k_ld = ld
    for w, b, k, m_out, act in layers:
        y = torch.empty((n, m_out), dtype=torch.float32, device=x.device)
        _lib.check(lib.fv_linear_fwd_tc(a.data_ptr(), k_ld, w.data_ptr(), b.data_ptr(), y.data_ptr(), m_out, n, k,
                                        m_out, act, sp), "fv_linear_fwd_tc")
        a, k_ld = y, m_out
    return a


def stratified_sample(nets: FreeviewModel, camera: CameraModel, pix: torch.Tensor, settings: RenderSettings):
    """SPEC stratified_sample for the rays of pixel ids ``pix`` (int32, CUDA):
    (x (R,N,3) world sample positions, delta (R,N), count (R) int32 samples per ray -- N if the
    ray hits the box, else 0).  One fv_march_warp launch (slab, jittered bins, delta rule of
    DESIGN §3); the kernel's ray-block-major layout is returned ray-major."""
    if pix.dtype != torch.int32 or not pix.is_cuda:
        raise DimensionError("stratified_sample: pix must be an int32 CUDA tensor")
    r, n = pix.numel(), settings.n_samples
    rp = (r + 31) // 32 * 32
    xs = torch.empty((rp * n, 4), dtype=torch.float32, device=pix.device)
    delta = torch.empty(rp * n, dtype=torch.float32, device=pix.device)
    x = torch.empty((rp * n, 3), dtype=torch.float32, device=pix.device)
    count = torch.empty(r, dtype=torch.int32, device=pix.device)
    if r == 0:
        return x.view(0, n, 3), delta.view(0, n), count
    m, cs, w = march_struct(settings, pix, None), camera_struct(camera), nets.warp_struct()
    _lib.check(nets.lib.fv_march_warp(C.byref(cs), C.byref(m), C.byref(w), r, xs.data_ptr(), delta.data_ptr(),
                                      x.data_ptr(), count.data_ptr(), _lib.stream_ptr()), "fv_march_warp")

    def ray_major(a, tail):
        return a.view((rp // 32, n, 32) + tail).transpose(1, 2).reshape((rp, n) + tail)[:r]

    return ray_major(x, (3,)), ray_major(delta, ()), count


def query_radiance(nets: FreeviewModel, x_final: torch.Tensor):
    """(c (n,3), sigma (n)) of canonical points."""
    n = x_final.shape[0]
    xs4 = torch.cat([x_final.float(), torch.ones((n, 1), device=x_final.device)], 1)
    out, _ = _field(nets, xs4, EPS_W, False)
    return out[:, :3], out[:, 3]


def composite(sigma: torch.Tensor, color: torch.Tensor, delta: torch.Tensor, likelihood: torch.Tensor,
              background, eps_w: float = EPS_W, eps_t: float = 0.0):
    """(rgb (R,3), alpha (R)) from per-sample sigma/delta/likelihood (R,N) and color (R,N,3)."""
    r, n = sigma.shape
    rgbs = torch.cat([color.reshape(r * n, 3), sigma.reshape(r * n, 1)], 1).float().contiguous()
    rgb = torch.empty((r, 3), dtype=torch.float32, device=sigma.device)
    alpha = torch.empty(r, dtype=torch.float32, device=sigma.device)
    bg = (C.c_float * 3)(*background)
    lib = _lib.load()
    _lib.check(lib.fv_composite_fwd(rgbs.data_ptr(), delta.float().contiguous().data_ptr(),
                                    likelihood.float().contiguous().data_ptr(), 1, 0, r, n, bg, eps_w, eps_t,
                                    rgb.data_ptr(), alpha.data_ptr(), None, _lib.stream_ptr()), "fv_composite_fwd")
    return rgb, alpha


# ----------------------------------------------------------------------- config 5: scenes

def subject_pixels(cam: CameraModel, box_min, box_max, rows=None) -> np.ndarray:
    """Pixel ids (8x4-tiled order) of every tile that the projection of the box touches,
    optionally restricted to the image row bands ``rows`` ([(r0, r1), ...]): a superset of the pixels whose ray hits
    the box, so a subject is only marched where it can be seen.  All pixels if a box
    corner is behind the camera."""
    w, h = cam.width, cam.height
    corners = np.array([[x, y, z] for x in (box_min[0], box_max[0]) for y in (box_min[1], box_max[1])
                        for z in (box_min[2], box_max[2])], np.float64)
    pc = corners @ cam.rotation.T + cam.world_to_camera[:3, 3]
    order = tiled_pixel_order(w, h)
    if np.any(pc[:, 2] <= 1e-6):
        sel = order
    else:
        uv = pc @ cam.intrinsics.T
        u, v = uv[:, 0] / uv[:, 2], uv[:, 1] / uv[:, 2]
        x0, x1 = int(np.floor(u.min())) - 1, int(np.ceil(u.max())) + 1
        y0, y1 = int(np.floor(v.min())) - 1, int(np.ceil(v.max())) + 1
        if w % 8 == 0 and h % 4 == 0:     # whole 8x4 tiles (32-ray blocks stay spatially coherent)
            x0, x1 = x0 // 8 * 8, (x1 + 8) // 8 * 8
            y0, y1 = y0 // 4 * 4, (y1 + 4) // 4 * 4
        px, py = order % w, order // w
        sel = order[(px >= x0) & (px < x1) & (py >= y0) & (py < y1)]
    if rows is not None:
        py = sel // w
        keep = np.zeros(len(sel), bool)
        for r0, r1 in rows:
            keep |= (py >= r0) & (py < r1)
        sel = sel[keep]
    return np.ascontiguousarray(sel, dtype=np.int32)


class SceneRenderer:
    """Config 5: every subject through the single-subject path (its own pose, occupancy
    grid and jitter seed, camera shifted into its frame, background 0) over the pixels its
    box can cover, then ``fv_scene_composite`` merges them front to back."""

    def __init__(self, n_subjects: int, device: str = "cuda"):
        if n_subjects < 1 or n_subjects > _lib.MAX_SUBJECTS:
            raise DimensionError(f"1..{_lib.MAX_SUBJECTS} subjects")
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.renderers = [Renderer(device) for _ in range(n_subjects)]
        shared = self.renderers[0]
        for r in self.renderers[1:]:
            r.workspace = shared.workspace          # one workspace, subjects render in turn
        self._pix = {}
        self._bufs = None

    def _buffers(self, n_pix):
        if self._bufs is None or self._bufs[1].shape[1] != n_pix:
            s = len(self.renderers)
            self._bufs = (torch.zeros((s, n_pix, 3), dtype=torch.float32, device=self.device),
                          torch.zeros((s, n_pix), dtype=torch.float32, device=self.device))
        return self._bufs

    def subject_pix(self, s: int, cam: CameraModel, settings: RenderSettings, rows=None) -> torch.Tensor:
        if rows is not None:
            rows = tuple((int(a), int(b)) for a, b in rows)
        key = (s, cam.world_to_camera.tobytes(), cam.width, cam.height, tuple(settings.box_min),
               tuple(settings.box_max), rows)
        if key not in self._pix:
            self._pix[key] = torch.from_numpy(subject_pixels(cam, settings.box_min, settings.box_max, rows)).to(self.device)
        return self._pix[key]

    def render_scene(self, subject_nets, scene, settings: List[RenderSettings], background, poses=None,
                     rows=None, out_rgb=None, out_alpha=None, stream=None):
        """(image (H,W,3), alpha (H,W)); with ``rows`` = [(r0, r1), ...] only those image row
        bands are produced (tile sharding across ranks; other rows are left undefined).
        ``settings[s]`` must carry background 0."""
        if rows is not None:
            rows = tuple((int(a), int(b)) for a, b in rows)
        cam = scene.camera
        n_pix = cam.width * cam.height
        rgb_s, alpha_s = self._buffers(n_pix)
        if out_rgb is None:
            out_rgb = torch.empty((n_pix, 3), dtype=torch.float32, device=self.device)
        if out_alpha is None:
            out_alpha = torch.empty(n_pix, dtype=torch.float32, device=self.device)
        m = _lib.FvSceneMerge()
        m.n_subjects = len(subject_nets)
        for s, (nets, st) in enumerate(zip(subject_nets, settings)):
            if any(b != 0.0 for b in st.background):
                raise DimensionError("subject settings must use background 0 (the scene background is merged once)")
            r = self.renderers[s]
            cam_s = scene.subject_camera(s)
            if poses is not None:
                nets.set_pose(poses[s], stream)
            occ = r.build_occupancy(nets, st, stream) if st.occupancy else None
            pix = self.subject_pix(s, cam_s, st, rows)
            if pix.numel():
                r.render_pixels(nets, cam_s, pix, st, rgb_s[s], alpha_s[s], by_pixel=True, occ=occ, stream=stream)
            m.cam[s] = camera_struct(cam_s)
            m.d_rgb[s] = rgb_s[s].data_ptr()
            m.d_alpha[s] = alpha_s[s].data_ptr()
        _lib.farr(m.box_min, np.asarray(settings[0].box_min, np.float32))
        _lib.farr(m.box_max, np.asarray(settings[0].box_max, np.float32))
        _lib.farr(m.bg, background)
        p0, p1 = (0, n_pix) if rows is None else (min(a for a, _ in rows) * cam.width, max(b for _, b in rows) * cam.width)
        _lib.check(self.lib.fv_scene_composite(C.byref(m), p0, p1 - p0, out_rgb.data_ptr(), out_alpha.data_ptr(),
                                               _lib.stream_ptr(stream)), "fv_scene_composite")
        return out_rgb.view(cam.height, cam.width, 3), out_alpha.view(cam.height, cam.width)


def scene_settings(scene, **kw) -> List[RenderSettings]:
    """Per-subject render settings of a MultiScene: config samples/jitter/occupancy, the
    subject's own jitter seed, background 0."""
    return [RenderSettings.from_config(scene.cfg, seed=sub.jitter_seed, background=(0.0, 0.0, 0.0), **kw)
            for sub in scene.subjects]


def render_scene(subject_nets, scene, poses=None, settings: Optional[List[RenderSettings]] = None):
    """Config 5 public entry: joint image of all subjects over the scene background."""
    key = ("scene", str(subject_nets[0].device), len(subject_nets))
    if key not in _DEFAULT:
        _DEFAULT[key] = SceneRenderer(len(subject_nets), subject_nets[0].device)
    st = settings if settings is not None else scene_settings(scene)
    return _DEFAULT[key].render_scene(subject_nets, scene, st, tuple(scene.cfg.background), poses)
