"""Synthetic, seeded stand-ins for the BASELINE.json configurations (no dataset or
checkpoint is available offline; ZJU-MoCap, SPIN/SMPL and trained weights are absent).

Config 1 ("c1", CPU-runnable PR1): 64x64 fp32 frame, camera at 3 m facing the origin,
64 uniform samples/ray in the body box [-1,1]^3; 24 joints with rest positions
~U([-1,1]^3), axis-angle ~N(0, 0.2); weight-volume logits ~U(0,1) (25 x 32^3, channel
softmax); offset MLP 4x128 on the 72-d pose + 6-band posenc; hash grid 16 x 2,
T = 2^14, resolution 16 -> 512, table ~U(-1e-4, 1e-4); radiance MLP 2x64; Xavier-uniform
weights, zero biases.
Config 2 ("c2"): 512x512, 128 jittered samples, T = 2^19, resolution 16 -> 2048, fp16
table / weight volume / tensor-core MLPs with fp32 accumulation, 32^3 occupancy grid.
Config 3 ("c3"): config-2 model trained on 6 random 32x32 patches of a seeded smooth
512x512 target (foreground = projected body-box ellipsoid), fp16 grid with fp32 master.
Config 4 ("c4"): 8 poses ~N(0, 0.3), otherwise config 2.
Config 5 ("c5"): 4 independently posed subjects (own seeded skeleton, pose, weight volume,
MLPs and T = 2^19 hash table each) at seeded offsets in a shared 4 m scene, 1024x1024,
192 jittered samples per ray inside each subject's box, depth-ordered joint compositing
over a constant background (``make_multi_scene``; builder-defined, SS3).

Every tensor comes from its own child of ``np.random.SeedSequence(seed)``.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

from .camera import CameraModel, orbit_camera
from .skeleton import SMPL24_PARENTS, Pose, Skeleton, motion_basis

PE_BANDS = 6
POSE_DIM = 72
OFF_WIDTH = 128
RAD_WIDTH = 64


@dataclass(frozen=True)
class HashGridConfig:
    """Hash-grid layout (definition: oracle/encoding.py, SS3)."""
    n_levels: int = 16
    n_feat: int = 2
    log2_T: int = 14
    base_res: int = 16
    max_res: int = 512

    @property
    def table_size(self) -> int:
        return 1 << self.log2_T

    def resolutions(self) -> List[int]:
        b = np.exp(np.log(self.max_res / self.base_res) / (self.n_levels - 1))
        return [int(np.floor(self.base_res * b ** l + 1e-9)) for l in range(self.n_levels)]

    def dense(self) -> List[bool]:
        return [(r + 1) ** 3 <= self.table_size for r in self.resolutions()]

    def sizes(self) -> List[int]:
        return [min((r + 1) ** 3, self.table_size) for r in self.resolutions()]

    def offsets(self) -> List[int]:
        """Level start entries, each a multiple of 4 (16-byte aligned fp16 blocks)."""
        out, o = [], 0
        for sz in self.sizes():
            out.append(o)
            o += (sz + 3) // 4 * 4
        return out

    @property
    def n_entries(self) -> int:
        return self.offsets()[-1] + (self.sizes()[-1] + 3) // 4 * 4


@dataclass(frozen=True)
class SceneConfig:
    name: str = "c1"
    width: int = 64
    height: int = 64
    n_samples: int = 64
    jitter: bool = False
    hash: HashGridConfig = HashGridConfig()
    half: bool = False              # fp16 table + weight volume + tensor-core MLPs
    occupancy: bool = False
    pose_sigma: float = 0.2
    n_poses: int = 1
    n_bones: int = 24
    vol_res: int = 32
    table_scale: float = 1e-4       # table ~U(-s, s)
    bias_scale: float = 0.0         # biases ~U(-s, s) (0: Xavier default zero biases)
    fov_deg: float = 45.0
    radius: float = 3.0
    seed: int = 0
    background: tuple = (0.5, 0.5, 0.5)


CONFIGS = {
    "c1": SceneConfig(),
    "c2": SceneConfig(name="c2", width=512, height=512, n_samples=128, jitter=True,
                      hash=HashGridConfig(log2_T=19, max_res=2048), half=True, occupancy=True),
    "c3": SceneConfig(name="c3", width=512, height=512, n_samples=128, jitter=True,
                      hash=HashGridConfig(log2_T=19, max_res=2048), half=True),
    "c4": SceneConfig(name="c4", width=512, height=512, n_samples=128, jitter=True,
                      hash=HashGridConfig(log2_T=19, max_res=2048), half=True, occupancy=True,
                      pose_sigma=0.3, n_poses=8),
    "c5": SceneConfig(name="c5", width=1024, height=1024, n_samples=192, jitter=True,
                      hash=HashGridConfig(log2_T=19, max_res=2048), half=True, occupancy=True,
                      radius=8.0, background=(0.2, 0.2, 0.2)),
}


def config(name: str, **overrides) -> SceneConfig:
    return replace(CONFIGS[name], **overrides)


@dataclass
class Scene:
    cfg: SceneConfig
    skeleton: Skeleton
    poses: List[Pose]
    vol_logits: np.ndarray          # (25, G, G, G) float32
    off_w: List[np.ndarray]         # (in, out) float32
    off_b: List[np.ndarray]
    rad_w: List[np.ndarray]
    rad_b: List[np.ndarray]
    table: np.ndarray               # (entries, 2) float32 (fp16-representable when cfg.half)
    jitter_seed: int
    camera: CameraModel
    obox_min: np.ndarray = field(default_factory=lambda: np.array([-1.0, -1.0, -1.0]))
    obox_max: np.ndarray = field(default_factory=lambda: np.array([1.0, 1.0, 1.0]))
    wbox_min: np.ndarray = field(default_factory=lambda: np.array([-1.0, -1.0, -1.0]))
    wbox_max: np.ndarray = field(default_factory=lambda: np.array([1.0, 1.0, 1.0]))

    def vol(self) -> np.ndarray:
        """Channel softmax of the logits (ad:711-721), float32; fp16-rounded when cfg.half."""
        z = self.vol_logits.astype(np.float64)
        e = np.exp(z - z.max(axis=0, keepdims=True))
        v = (e / e.sum(axis=0, keepdims=True)).astype(np.float32)
        return v.astype(np.float16).astype(np.float32) if self.cfg.half else v


def _xavier(rng, fan_in, fan_out):
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-lim, lim, (fan_in, fan_out)).astype(np.float32)


def make_scene(cfg: SceneConfig) -> Scene:
    ch = np.random.SeedSequence(cfg.seed).spawn(8)
    rng_sk, rng_pose, rng_vol, rng_off, rng_tab, rng_rad, rng_jit = (np.random.default_rng(c) for c in ch[:7])
    k = cfg.n_bones
    parents = np.array(SMPL24_PARENTS[:k]) if k <= 24 else np.concatenate([SMPL24_PARENTS, np.arange(23, k - 1)])
    rest = rng_sk.uniform(-1.0, 1.0, (k, 3))
    offs = rest.copy()
    offs[1:] = rest[1:] - rest[parents[1:]]
    skel = Skeleton(parent=parents, rest_offset=offs, canonical_angles=np.zeros((k, 3)),
                    canonical_root=np.zeros(3))
    poses = [Pose(rng_pose.normal(0.0, cfg.pose_sigma, (k, 3)), np.zeros(3)) for _ in range(cfg.n_poses)]
    g = cfg.vol_res
    logits = rng_vol.uniform(0.0, 1.0, (k + 1, g, g, g)).astype(np.float32)
    d_pe = 3 + 6 * PE_BANDS
    off_dims = [d_pe + 3 * k, OFF_WIDTH, OFF_WIDTH, OFF_WIDTH, OFF_WIDTH, 3]
    rad_dims = [cfg.hash.n_levels * cfg.hash.n_feat, RAD_WIDTH, RAD_WIDTH, 4]
    off_w = [_xavier(rng_off, a, b) for a, b in zip(off_dims[:-1], off_dims[1:])]
    off_b = [rng_off.uniform(-cfg.bias_scale, cfg.bias_scale, b).astype(np.float32) for b in off_dims[1:]]
    rad_w = [_xavier(rng_rad, a, b) for a, b in zip(rad_dims[:-1], rad_dims[1:])]
    rad_b = [rng_rad.uniform(-cfg.bias_scale, cfg.bias_scale, b).astype(np.float32) for b in rad_dims[1:]]
    table = rng_tab.uniform(-cfg.table_scale, cfg.table_scale, (cfg.hash.n_entries, cfg.hash.n_feat)).astype(np.float32)
    if cfg.half:  # fp16-representable so the fp32 master and the fp16 copy start identical
        table = table.astype(np.float16).astype(np.float32)
        off_w = [w.astype(np.float16).astype(np.float32) for w in off_w]
        rad_w = [w.astype(np.float16).astype(np.float32) for w in rad_w]
    cam = orbit_camera((0.0, 0.0, 0.0), 0.0, 0.0, cfg.radius, cfg.fov_deg, cfg.width, cfg.height)
    return Scene(cfg=cfg, skeleton=skel, poses=poses, vol_logits=logits, off_w=off_w, off_b=off_b, rad_w=rad_w,
                 rad_b=rad_b, table=table, jitter_seed=int(rng_jit.integers(0, 2 ** 31)), camera=cam)


def target_image(scene: Scene, seed: int = 7):
    """Seeded smooth RGB field inside the projected body-box ellipsoid, background outside
    (config 3 training target).  Returns (H,W,3) float32 and the (H,W) bool mask."""
    cfg = scene.cfg
    rng = np.random.default_rng(np.random.SeedSequence(cfg.seed).spawn(8)[7])
    h, w = cfg.height, cfg.width
    yy, xx = np.meshgrid(np.linspace(0, 1, h), np.linspace(0, 1, w), indexing="ij")
    img = np.zeros((h, w, 3))
    for c in range(3):
        for _ in range(4):
            fx, fy = rng.uniform(0.5, 3.0, 2)
            ph = rng.uniform(0, 2 * np.pi)
            img[..., c] += np.sin(2 * np.pi * (fx * xx + fy * yy) + ph)
    img = 0.5 + 0.12 * img
    cam = scene.camera
    kinv = np.linalg.inv(cam.intrinsics)
    pix = np.stack([xx * 0 + np.arange(w)[None, :] + 0.5, yy * 0 + np.arange(h)[:, None] + 0.5, np.ones((h, w))], -1)
    d = (pix @ kinv.T) @ cam.rotation
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    o = cam.center
    # unit sphere inscribed in the [-1,1]^3 body box, scaled to an ellipsoid (0.8, 1.0, 0.6)
    s = np.array([0.8, 1.0, 0.6])
    od, dd = o / s, d / s
    a = np.sum(dd * dd, -1)
    b = 2 * np.sum(dd * od, -1)
    cc = np.sum(od * od) - 1.0
    mask = b * b - 4 * a * cc > 0
    out = np.where(mask[..., None], np.clip(img, 0, 1), np.asarray(cfg.background)[None, None, :])
    return out.astype(np.float32), mask


def opaque_subject(scene: Scene, axes=(0.45, 0.8, 0.3), level: Optional[int] = None, sigma_in: float = 90.0) -> Scene:
    """A subject with a realistic density field (stand-in for trained weights, which are
    absent: ZJU-MoCap and its checkpoints are not in the container): density ~sigma_in / m
    inside a canonical body ellipsoid with semi-axes ``axes`` (fractions of the canonical box
    half-extent) and ~5e-5 / m outside, seen through the scene's own skinning warp and
    residual offsets -- empty space around the body and rays that saturate inside it, the two
    things occupancy skipping and early termination act on.

    Built from the scene's own parameter blocks: feature 0 of dense hash level ``level`` is
    +1 at grid vertices inside the ellipsoid and -1 outside; radiance hidden unit 0 passes
    relu(4 f) through both hidden layers; the sigma logit is 25 h - 9 (softplus(h - 1) ->
    ~90 inside, 4.5e-5 outside); every other weight keeps its seeded value (colours)."""
    cfg = scene.cfg
    h = cfg.hash
    if level is None:        # the finest dense level up to 3 (C2: res 42, C1: res 20)
        level = max(l for l in range(min(4, h.n_levels)) if h.dense()[l])
    if not h.dense()[level]:
        raise ValueError(f"level {level} is hashed, opaque_subject needs a dense level")
    res, off = h.resolutions()[level], h.offsets()[level]
    table = scene.table.copy()
    s1 = res + 1
    ii = np.arange(s1) / res
    gx, gy, gz = np.meshgrid(ii, ii, ii, indexing="ij")          # normalised canonical vertex positions
    q = ((gx - 0.5) / (0.5 * axes[0])) ** 2 + ((gy - 0.5) / (0.5 * axes[1])) ** 2 + ((gz - 0.5) / (0.5 * axes[2])) ** 2
    inside = q <= 1.0
    # dense index x + y s + z s^2 (oracle.encoding / hash_index)
    idx = (np.arange(s1)[:, None, None] + np.arange(s1)[None, :, None] * s1 + np.arange(s1)[None, None, :] * s1 * s1)
    table[off + idx.reshape(-1), 0] = np.where(inside.reshape(-1), 1.0, -1.0).astype(np.float32)
    rad_w = [w.copy() for w in scene.rad_w]
    rad_b = [b.copy() for b in scene.rad_b]
    rad_w[0][:, 0] = 0.0
    rad_w[0][2 * level, 0] = 4.0
    rad_b[0][0] = 0.0
    rad_w[1][0, :] = 0.0
    rad_w[1][:, 0] = 0.0
    rad_w[1][0, 0] = 1.0
    rad_b[1][0] = 0.0
    rad_w[2][0, :] = 0.0
    rad_w[2][:, 3] = 0.0
    rad_w[2][0, 3] = sigma_in / 3.6
    rad_b[2][3] = -9.0
    if cfg.half:
        table = table.astype(np.float16).astype(np.float32)
        rad_w = [w.astype(np.float16).astype(np.float32) for w in rad_w]
    return replace(scene, table=table, rad_w=rad_w, rad_b=rad_b)


OCC_RES = 32


def ellipsoid_occupancy(box_min, box_max, seed: int = 11, axes=(0.8, 1.0, 0.6), jitter: float = 0.1) -> np.ndarray:
    """Seeded-ellipsoid 32^3 occupancy bitfield over the observation box (the C2
    run with a body-shaped skip grid next to the flat-density one).  Cell (i,j,k) -- bit
    ((i*32 + j)*32 + k) of an int32[1024], the layout of ``occ_test`` -- is set iff its
    centre lies inside the ellipsoid with semi-axes ``axes`` (x the box half-extent), each
    scaled by a seeded factor in [1 - jitter, 1 + jitter]."""
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    bmin, bmax = np.asarray(box_min, np.float64), np.asarray(box_max, np.float64)
    half, ctr = 0.5 * (bmax - bmin), 0.5 * (bmax + bmin)
    semi = np.asarray(axes) * half * rng.uniform(1.0 - jitter, 1.0 + jitter, 3)
    c = (np.arange(OCC_RES) + 0.5) / OCC_RES
    gx, gy, gz = np.meshgrid(*[bmin[j] + c * (bmax[j] - bmin[j]) for j in range(3)], indexing="ij")
    inside = ((gx - ctr[0]) / semi[0]) ** 2 + ((gy - ctr[1]) / semi[1]) ** 2 + ((gz - ctr[2]) / semi[2]) ** 2 <= 1.0
    bits = inside.reshape(-1).astype(np.uint64)
    words = (bits.reshape(-1, 32) << np.arange(32, dtype=np.uint64)).sum(1)
    return words.astype(np.uint32).view(np.int32)


@dataclass
class MultiScene:
    """Config 5: subjects (each a full single-subject Scene in its own frame) placed at
    world offsets; ``camera`` is the world camera, subject s is rendered through
    ``camera.translated(offsets[s])``."""
    cfg: SceneConfig
    subjects: List[Scene]
    offsets: np.ndarray             # (S, 3) world position of each subject frame's origin
    camera: CameraModel

    def subject_camera(self, s: int) -> CameraModel:
        return self.camera.translated(self.offsets[s])


def place_subjects(rng, n: int, extent: float, box: float = 2.0, margin: float = 0.05,
                   tries: int = 10000) -> np.ndarray:
    """Seeded subject positions on the ground plane (y = 0): x, z ~ U(-extent/2, extent/2),
    rejection-sampled until every pair of boxes is separated along x or z by >= box + margin,
    i.e. the boxes are disjoint (what makes the depth-ordered merge exact)."""
    half = extent / 2.0
    for _ in range(tries):
        xz = rng.uniform(-half, half, (n, 2))
        ok = all(max(abs(xz[i, 0] - xz[j, 0]), abs(xz[i, 1] - xz[j, 1])) >= box + margin
                 for i in range(n) for j in range(i))
        if ok:
            return np.stack([xz[:, 0], np.zeros(n), xz[:, 1]], 1)
    raise ValueError(f"could not place {n} disjoint {box} m boxes in a {extent} m square")


def make_multi_scene(cfg: SceneConfig, n_subjects: int = 4, extent: float = 4.0, pitch_deg: float = 20.0) -> MultiScene:
    """Config 5 stand-in: every subject from its own child seed (its own hash table,
    skeleton, pose, weight volume and MLPs), positions from another child."""
    ch = np.random.SeedSequence(cfg.seed).spawn(n_subjects + 1)
    subjects = [make_scene(replace(cfg, seed=int(c.generate_state(1)[0]))) for c in ch[:n_subjects]]
    offsets = place_subjects(np.random.default_rng(ch[n_subjects]), n_subjects, extent)
    cam = orbit_camera((0.0, 0.0, 0.0), 0.0, pitch_deg, cfg.radius, cfg.fov_deg, cfg.width, cfg.height)
    return MultiScene(cfg=cfg, subjects=subjects, offsets=offsets, camera=cam)
