"""Pinhole camera of the reference capture model (``cap:40-142``), host side.

The ray-march kernel regenerates every ray from ``K^-1``, ``R`` and the camera centre
(``fv_camera``); this module only builds those constants and the pixel traversal order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CameraModel:
    intrinsics: np.ndarray       # 3x3
    world_to_camera: np.ndarray  # 4x4 rows [R | t]
    width: int
    height: int

    def __post_init__(self):
        self.intrinsics = np.asarray(self.intrinsics, dtype=np.float64)
        self.world_to_camera = np.asarray(self.world_to_camera, dtype=np.float64)
        k = self.intrinsics
        if k.shape != (3, 3) or k[0, 0] <= 0 or k[1, 1] <= 0:
            raise ValueError("intrinsics must be 3x3 with positive focal lengths")
        r = self.world_to_camera[:3, :3]
        if np.max(np.abs(r.T @ r - np.eye(3))) > 1e-9 or abs(np.linalg.det(r) - 1) > 1e-9:
            raise ValueError("extrinsic rotation is not rigid")

    @property
    def rotation(self) -> np.ndarray:
        return self.world_to_camera[:3, :3]

    @property
    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.world_to_camera[:3, 3]

    def translated(self, offset) -> "CameraModel":
        """The same camera seen from a frame whose origin sits at world point ``offset``
        (a subject placed at ``offset``, config 5): x_local = x_world - offset, so the centre
        moves by -offset and t = R offset is added to the translation; depths along a ray
        are unchanged."""
        w2c = self.world_to_camera.copy()
        w2c[:3, 3] = w2c[:3, 3] + self.rotation @ np.asarray(offset, dtype=np.float64)
        return CameraModel(self.intrinsics.copy(), w2c, self.width, self.height)

    def kernel_consts(self):
        """float32 (K^-1, R, centre) exactly as fv_camera carries them."""
        return (np.linalg.inv(self.intrinsics).astype(np.float32), self.rotation.astype(np.float32),
                self.center.astype(np.float32))


def look_at(eye, target, up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """World-to-camera; camera +x right, +y down, +z forward (cap:113-129)."""
    eye = np.asarray(eye, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - eye
    f /= np.linalg.norm(f)
    x = np.cross(f, np.asarray(up, dtype=np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    y /= np.linalg.norm(y)
    m = np.eye(4)
    m[:3, :3] = np.stack([x, y, f])
    m[:3, 3] = -m[:3, :3] @ eye
    return m


def orbit_camera(target, yaw_deg, pitch_deg, radius, fov_deg, width, height) -> CameraModel:
    """Camera on a sphere around ``target``: yaw about +Y, pitch above horizon (cap:132-142)."""
    yaw, pitch = np.deg2rad(yaw_deg), np.deg2rad(pitch_deg)
    target = np.asarray(target, dtype=np.float64)
    eye = target + radius * np.array([np.sin(yaw) * np.cos(pitch), np.sin(pitch), np.cos(yaw) * np.cos(pitch)])
    f = 0.5 * height / np.tan(0.5 * np.deg2rad(fov_deg))
    k = np.array([[f, 0, width / 2.0], [0, f, height / 2.0], [0, 0, 1.0]])
    return CameraModel(k, look_at(eye, target), width, height)


def tiled_pixel_order(width: int, height: int, tw: int = 8, th: int = 4) -> np.ndarray:
    """Linear pixel ids in 8x4 tiles (one 32-ray block per tile) when the image tiles evenly,
    else row-major.  Neighbouring rays share cache lines in the volume / hash gathers."""
    if width % tw or height % th:
        return np.arange(width * height, dtype=np.int32)
    ty, tx, j, i = np.meshgrid(np.arange(height // th), np.arange(width // tw), np.arange(th), np.arange(tw),
                               indexing="ij")
    return ((ty * th + j) * width + tx * tw + i).reshape(-1).astype(np.int32)
