"""Turn a product ``Scene`` (plain numpy arrays, duck-typed) into the oracle's scene dict.

The oracle computes the motion bases with its own restatement of the reference FK
(``oracle.skeleton``, ``sk:240-303``) unless ``g`` is given; parameters are rounded to
fp16 exactly as the GPU receives them when ``cfg.half`` is set.
"""

from __future__ import annotations

import numpy as np

from . import skeleton as osk
from .encoding import HashGridSpec


def scene_arrays(scene, pose_index: int = 0, g=None, vol=None) -> dict:
    cfg = scene.cfg
    sk = scene.skeleton
    pose = scene.poses[pose_index]
    if g is None:
        g_r, g_t = osk.motion_basis(sk.parent, sk.rest_offset, sk.canonical_angles, sk.canonical_root,
                                    pose.angles, pose.root_translation)
    else:
        g_r, g_t = g
    q = (lambda a: np.asarray(a, np.float32).astype(np.float16).astype(np.float32)) if cfg.half else \
        (lambda a: np.asarray(a, np.float32))
    if vol is None:  # softmax0 of the logits (ad:711-721); tests pass the device's own W^c
        z = scene.vol_logits.astype(np.float64)
        e = np.exp(z - z.max(axis=0, keepdims=True))
        vol = (e / e.sum(axis=0, keepdims=True)).astype(np.float32)
    h = cfg.hash
    return {
        "g_r": np.asarray(g_r, np.float32), "g_t": np.asarray(g_t, np.float32),
        "pose_vec": np.asarray(pose.angles, np.float32).reshape(-1),
        "vol": q(vol), "wbox_min": scene.wbox_min, "wbox_max": scene.wbox_max,
        "obox_min": scene.obox_min, "obox_max": scene.obox_max,
        "off_w": [q(w) for w in scene.off_w], "off_b": [np.asarray(b, np.float32) for b in scene.off_b],
        "rad_w": [q(w) for w in scene.rad_w], "rad_b": [np.asarray(b, np.float32) for b in scene.rad_b],
        "table": q(scene.table), "bg": np.asarray(cfg.background, np.float32),
        "hash_spec": HashGridSpec(h.n_levels, h.n_feat, h.log2_T, h.base_res, h.max_res),
    }


def settings(cfg, **kw) -> dict:
    out = {"n_samples": cfg.n_samples, "jitter": cfg.jitter, "seed": 0, "pe_bands": 6, "pe_alpha": 6.0,
           "offset_enabled": True, "eps_w": 1e-4, "eps_t": 0.0, "occupancy": None}
    out.update(kw)
    return out
