"""Multi-subject scenes (BASELINE config 5) -- TEST INFRASTRUCTURE (oracle).

Builder-defined, PARITY UNPINNED: the reference has no multi-subject code (``S:8``; the
paper lists multi-person capture as future work, ``P:303``).  Definition restated here:

* subject ``s`` lives in its own frame, placed at world ``offset_s``; it is rendered by the
  single-subject path (``pipeline.render_rays``: ``S:410-446``) through the world camera
  shifted by ``-offset_s`` with background 0, giving per ray its premultiplied colour
  ``C_s`` and ``alpha_s = 1 - T_s`` over its box;
* subject boxes are disjoint, so along a ray their sample intervals are disjoint and the
  front-to-back composite of ALL samples (``S:428-437`` over the t-sorted union) equals
  ``C = sum_s (prod_{j before s} T_j) C_s + (prod_s T_s) bg``, ``alpha = 1 - prod_s T_s``
  with subjects ordered by their float32 slab entry depth.

``merge_subjects`` is that product in the kernel's float32 order (csrc/scene_merge.cu);
``union_composite`` is the brute-force definition (one composite over the merged, depth-
sorted sample streams) used to pin the factorisation.
"""

from __future__ import annotations

import numpy as np

from . import camera, composite as comp, pipeline

F32 = np.float32


def entry_depths(cc_list, pix, width, box_min, box_max):
    """(t_enter (S,R), hit (S,R)) of every subject's box, float32 kernel order."""
    te, hits = [], []
    for cc in cc_list:
        o, d = camera.rays_f32(cc, pix, width)
        t0, _, hit = camera.slab_f32(o, d, box_min, box_max)
        te.append(t0)
        hits.append(hit)
    return np.stack(te), np.stack(hits)


def merge_subjects(rgb, alpha, t_enter, hit, bg):
    """rgb (S,R,3), alpha (S,R) per-subject composites with background 0 -> (rgb (R,3),
    alpha (R)); subjects composited front to back by entry depth (stable in s on ties)."""
    s_n, r = alpha.shape
    out = np.zeros((r, 3), F32)
    a_out = np.zeros(r, F32)
    bg = np.asarray(bg, F32)
    for p in range(r):
        order = sorted((float(t_enter[s, p]), s) for s in range(s_n) if hit[s, p])
        t = F32(1.0)
        c = np.zeros(3, F32)
        for _, s in order:
            c = (c + (t * rgb[s, p]).astype(F32)).astype(F32)
            t = F32(t * F32(F32(1.0) - alpha[s, p]))
        out[p] = (c + (t * bg).astype(F32)).astype(F32)
        a_out[p] = F32(F32(1.0) - t)
    return out, a_out


def render_scene_rays(subject_scenes, cc_list, pix, width, settings_list, bg, dtype=np.float32):
    """Per-subject oracle renders (background 0) + depth-ordered merge.  Returns the merged
    (rgb, alpha) and the per-subject render dicts."""
    renders = []
    for sc, cc, st in zip(subject_scenes, cc_list, settings_list):
        sc0 = dict(sc, bg=np.zeros(3, np.float32))
        renders.append(pipeline.render_rays(sc0, cc, pix, width, st, dtype))
    box_min, box_max = subject_scenes[0]["obox_min"], subject_scenes[0]["obox_max"]
    te, hit = entry_depths(cc_list, pix, width, box_min, box_max)
    rgb = np.stack([r["rgb"] for r in renders]).astype(F32)
    alpha = np.stack([r["alpha"] for r in renders]).astype(F32)
    out_rgb, out_alpha = merge_subjects(rgb, alpha, te, hit, bg)
    return {"rgb": out_rgb, "alpha": out_alpha, "renders": renders, "t_enter": te, "hit": hit}


def union_composite(renders, bg, eps_w=comp.EPS_W):
    """Brute-force definition: per ray, concatenate all subjects' samples, sort by depth t
    and run ONE front-to-back composite (float64)."""
    r = renders[0]["sigma"].shape[0]
    rgb = np.zeros((r, 3))
    alpha = np.zeros(r)
    for p in range(r):
        t = np.concatenate([rd["t"][p] for rd in renders])
        order = np.argsort(t, kind="stable")
        sig = np.concatenate([rd["sigma"][p] for rd in renders])[order]
        col = np.concatenate([rd["color"][p] for rd in renders])[order]
        dl = np.concatenate([rd["delta"][p] for rd in renders])[order]
        lk = np.concatenate([rd["lik"][p] for rd in renders])[order]
        res = comp.composite(sig[None], col[None], dl[None], lk[None], bg, eps_w, 0.0, np.float64)
        rgb[p] = res["rgb"][0]
        alpha[p] = res["alpha"][0]
    return rgb, alpha
