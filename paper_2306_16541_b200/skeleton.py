"""Host-side articulated skeleton: per-frame motion bases G_i uploaded to the warp kernel.

Mirrors the reference body model (``sk:25-303``): ``T_i = T_parent(i) o translate(
rest_offset_i) o rotate(omega_i)`` and ``G_i = T_i(canonical) o T_i(observed)^-1`` mapping
observation space to canonical space (``sk:288-303``, ``S:200``).  Row-vector convention:
a transform applies as ``x @ R.T + t`` (``sk:5-6``).  Per frame this is 24 small
matrices -- host work, outside the per-sample hot path.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

# SMPL-style 24-joint kinematic tree (pelvis root; spine chain; legs; arms).
SMPL24_PARENTS = [-1, 0, 0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 9, 9, 12, 13, 14, 16, 17, 18, 19, 20, 21]


@dataclass
class Skeleton:
    parent: np.ndarray           # (K,) int, root = -1
    rest_offset: np.ndarray      # (K,3) bone origin in the parent frame
    canonical_angles: np.ndarray  # (K,3) axis-angle of the canonical pose
    canonical_root: np.ndarray   # (3,)

    def __post_init__(self):
        self.parent = np.asarray(self.parent, dtype=np.int64)
        self.rest_offset = np.asarray(self.rest_offset, dtype=np.float64)
        self.canonical_angles = np.asarray(self.canonical_angles, dtype=np.float64)
        self.canonical_root = np.asarray(self.canonical_root, dtype=np.float64)
        if int(np.sum(self.parent < 0)) != 1:
            raise ValueError("skeleton must have exactly one root")
        for i in range(self.bone_count):  # acyclic
            seen, j = set(), i
            while j >= 0:
                if j in seen:
                    raise ValueError(f"cycle in parent chain at bone {i}")
                seen.add(j)
                j = int(self.parent[j])

    @property
    def bone_count(self) -> int:
        return len(self.parent)

    def order(self) -> List[int]:
        depth = np.zeros(self.bone_count, dtype=np.int64)
        for i in range(self.bone_count):
            j = i
            while self.parent[j] >= 0:
                depth[i] += 1
                j = int(self.parent[j])
        return [int(i) for i in np.argsort(depth, kind="stable")]


@dataclass
class Pose:
    angles: np.ndarray            # (K,3) axis-angle Omega
    root_translation: np.ndarray  # (3,)

    def __post_init__(self):
        self.angles = np.asarray(self.angles, dtype=np.float64)
        self.root_translation = np.asarray(self.root_translation, dtype=np.float64)
        if not (np.all(np.isfinite(self.angles)) and np.all(np.isfinite(self.root_translation))):
            raise ValueError("pose contains non-finite entries")

    def flat(self) -> np.ndarray:
        """Omega^o flattened (K*3,) -- the pose input of the residual MLP."""
        return self.angles.reshape(-1)


def rodrigues(omega: np.ndarray) -> np.ndarray:
    """Axis-angle (K,3) -> rotations (K,3,3); Taylor branch for |w|^2 < 1e-8 (sk:186-209)."""
    w = np.atleast_2d(np.asarray(omega, dtype=np.float64))
    th2 = np.einsum("ki,ki->k", w, w)
    small = th2 < 1e-8
    th = np.sqrt(np.where(small, 1.0, th2))
    a = np.where(small, 1.0 - th2 / 6.0, np.sin(th) / th)
    b = np.where(small, 0.5 - th2 / 24.0, (1.0 - np.cos(th)) / np.where(small, 1.0, th2))
    k = np.zeros((w.shape[0], 3, 3))
    k[:, 0, 1], k[:, 0, 2], k[:, 1, 2] = -w[:, 2], w[:, 1], -w[:, 0]
    k[:, 1, 0], k[:, 2, 0], k[:, 2, 1] = w[:, 2], -w[:, 1], w[:, 0]
    return np.eye(3) + a[:, None, None] * k + b[:, None, None] * np.einsum("kij,kjl->kil", k, k)


def world_transforms(skel: Skeleton, angles: np.ndarray, root: np.ndarray):
    """(R (K,3,3), t (K,3)) of every bone; t is also the joint world position (sk:240-273)."""
    rot = rodrigues(angles)
    r_out = np.zeros((skel.bone_count, 3, 3))
    t_out = np.zeros((skel.bone_count, 3))
    for i in skel.order():
        p = int(skel.parent[i])
        if p < 0:
            r_out[i] = rot[i]
            t_out[i] = np.asarray(root, np.float64) + skel.rest_offset[i]
        else:
            r_out[i] = r_out[p] @ rot[i]
            t_out[i] = t_out[p] + r_out[p] @ skel.rest_offset[i]
    return r_out, t_out


def motion_basis(skel: Skeleton, pose: Pose):
    """G_r (K,3,3), G_t (K,3): observation -> canonical per bone (sk:288-303)."""
    rc, tc = world_transforms(skel, skel.canonical_angles, skel.canonical_root)
    ro, to = world_transforms(skel, pose.angles, pose.root_translation)
    g_r = np.einsum("kij,klj->kil", rc, ro)           # Rc Ro^T
    g_t = tc - np.einsum("kij,kj->ki", g_r, to)
    return g_r, g_t


def pack_g(g_r: np.ndarray, g_t: np.ndarray) -> np.ndarray:
    """(K,12) float32 [R row-major, t] -- the layout of fv_warp.d_g."""
    k = g_r.shape[0]
    return np.concatenate([g_r.reshape(k, 9), g_t.reshape(k, 3)], axis=1).astype(np.float32)
