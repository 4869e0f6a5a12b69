"""Shared test helpers: product scenes, the oracle view of the same scene, layouts."""

import numpy as np

from oracle import adapter
from paper_2306_16541_b200 import scene as psc
from paper_2306_16541_b200.skeleton import motion_basis


def make(name="c1", **overrides):
    return psc.make_scene(psc.config(name, **overrides))


def oracle_scene(scene, pose_index=0, nets=None):
    """Oracle arrays fed with the product's float32 G_i (and, given ``nets``, the device's
    own softmaxed W^c) so integer outputs are comparable bit for bit."""
    g_r, g_t = motion_basis(scene.skeleton, scene.poses[pose_index])
    vol = nets.vol.detach().cpu().numpy() if nets is not None else None
    return adapter.scene_arrays(scene, pose_index, g=(g_r.astype(np.float32), g_t.astype(np.float32)), vol=vol)


def blocked_to_ray_major(a, n_rays, n):
    """(S, ...) ray-block-major sample array -> (R, N, ...)."""
    a = np.asarray(a)
    rp = (n_rays + 31) // 32 * 32
    tail = a.shape[1:]
    b = a.reshape((rp // 32, n, 32) + tail)
    b = np.swapaxes(b, 1, 2).reshape((rp, n) + tail)
    return b[:n_rays]


def trained_scene(scene, nets):
    """The scene with the model's current (trained) fp32 master parameters, for the oracle."""
    import dataclasses
    v = {k: t.detach().cpu().numpy().copy() for k, t in nets.views.items()}
    return dataclasses.replace(scene, table=v["table"], vol_logits=v["vol_logits"],
                               off_w=[v[f"off_w{i}"] for i in range(len(scene.off_w))],
                               off_b=[v[f"off_b{i}"] for i in range(len(scene.off_b))],
                               rad_w=[v[f"rad_w{i}"] for i in range(len(scene.rad_w))],
                               rad_b=[v[f"rad_b{i}"] for i in range(len(scene.rad_b))])
