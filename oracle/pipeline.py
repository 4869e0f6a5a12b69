"""The composed per-ray-sample path (oracle): SPEC ``render_image`` (``S:438-446``).

per pixel: ray (``cap:73-82``) -> slab + stratified samples (``S:410-413``) -> occupancy
skip -> ``warp_point`` = skeleton warp (``S:327-336``) + residual offset MLP on
``[posenc(x_skel, alpha), Omega^o]`` (``S:346-358``) -> hash-grid features -> radiance MLP
+ heads (``S:419-427``) -> composite (``S:428-437``).

Samples that are outside the box, in an empty occupancy cell or background
(``L <= eps_w``) carry ``sigma = 0`` ("contribute zero density downstream", SPEC
motion-field invariants) and are never evaluated by the field.

``scene`` is a plain dict of numpy arrays (see ``paper_2306_16541_b200.scene``):
``g_r, g_t, pose_vec, vol, wbox_min, wbox_max, obox_min, obox_max, off_w, off_b, rad_w,
rad_b, table, bg`` plus the ``HashGridSpec`` under ``hash_spec``.
"""

from __future__ import annotations

import numpy as np

from . import camera, composite as comp, encoding, mlp, warp

F32 = np.float32


def _field(scene, x_skel, settings, dtype):
    dt = np.dtype(dtype).type
    pe = encoding.posenc(x_skel, settings["pe_bands"], settings["pe_alpha"], dtype)
    if settings.get("offset_enabled", True):
        pose = np.broadcast_to(np.asarray(scene["pose_vec"], dt), (x_skel.shape[0], len(scene["pose_vec"])))
        off_in = np.concatenate([pe, pose], axis=1).astype(dt)
        x_res, off_acts = mlp.mlp_forward(off_in, scene["off_w"], scene["off_b"], dtype, keep=True)
    else:
        off_in, off_acts = None, None
        x_res = np.zeros_like(x_skel)
    x_final = (x_skel + x_res).astype(dt)
    cinv = (1.0 / (np.asarray(scene["wbox_max"], np.float64) - np.asarray(scene["wbox_min"], np.float64))).astype(F32)
    feat = encoding.hash_encode(scene["hash_spec"], x_final, np.asarray(scene["wbox_min"], F32), cinv,
                                scene["table"], dtype)
    h, rad_acts = mlp.mlp_forward(feat, scene["rad_w"], scene["rad_b"], dtype, keep=True)
    c, sigma = mlp.radiance_heads(h)
    return {"pe": pe, "off_in": off_in, "off_acts": off_acts, "x_res": x_res, "x_final": x_final,
            "feat": feat, "h": h, "rad_acts": rad_acts, "c": c, "sigma": sigma, "cinv": cinv}


def render_rays(scene, cc, pix, width, settings, dtype=np.float32):
    """Render the rays of linear pixel indices ``pix``; returns every intermediate."""
    dt = np.dtype(dtype).type
    pix = np.asarray(pix, dtype=np.int64)
    n = settings["n_samples"]
    o, d = camera.rays_f32(cc, pix, width)
    t_enter, t_exit, hit = camera.slab_f32(o, d, scene["obox_min"], scene["obox_max"])
    t, delta, count = camera.stratified_f32(t_enter, t_exit, hit, pix, n, settings["jitter"],
                                            settings["seed"])
    x = camera.positions_f32(o, d, t)
    valid = np.broadcast_to(hit[:, None], (len(pix), n)).copy()
    occ_bits = settings.get("occupancy")
    if occ_bits is not None:
        cell = camera.occ_cell(x, scene["obox_min"], camera.occ_scale(scene["obox_min"], scene["obox_max"]))
        valid &= camera.occ_test(occ_bits, cell)
    flat = np.nonzero(valid.ravel())[0]
    xv = x.reshape(-1, 3)[flat]
    wr = warp.skeleton_warp(xv, scene["g_r"], scene["g_t"], scene["vol"], scene["wbox_min"],
                            scene["wbox_max"], settings.get("eps_w", warp.EPS_W), dtype)
    fg_flat = flat[wr["fg"]]
    field = _field(scene, wr["x_skel"][wr["fg"]], settings, dtype)

    rn = len(pix) * n
    sigma = np.zeros(rn, dt)
    color = np.zeros((rn, 3), dt)
    lik = np.zeros(rn, dt)
    sigma[fg_flat] = field["sigma"]
    color[fg_flat] = field["c"]
    lik[flat] = wr["L"]
    res = comp.composite(sigma.reshape(-1, n), color.reshape(-1, n, 3), delta, lik.reshape(-1, n),
                         scene["bg"], settings.get("eps_w", warp.EPS_W), settings.get("eps_t", 0.0), dtype)
    fgm = np.zeros(rn, bool)
    fgm[fg_flat] = True
    return {"o": o, "d": d, "t_enter": t_enter, "t_exit": t_exit, "hit": hit, "count": count,
            "t": t, "delta": delta, "x": x, "valid": valid, "flat": flat, "warp": wr,
            "fg": fgm.reshape(-1, n), "fg_flat": fg_flat, "field": field,
            "sigma": sigma.reshape(-1, n), "color": color.reshape(-1, n, 3),
            "lik": lik.reshape(-1, n), "rgb": res["rgb"], "alpha": res["alpha"], "comp": res}


def loss_and_grads(scene, cc, pix, width, settings, target, dtype=np.float32, patch=None):
    """MSE loss over the rays (or, with ``patch = (size, lam_mse, lam_perc)`` and patch-major
    rays, the SPEC patch loss ``oracle.loss.patch_loss``) and float64 gradients of
    every trainable block.

    Blocks: ``table``; ``off_w[i]``/``off_b[i]``; ``rad_w[i]``/``rad_b[i]``; ``vol`` (the
    softmaxed weight volume; chain into logits with ``warp.softmax0_bwd``).
    """
    r = render_rays(scene, cc, pix, width, settings, dtype)
    rgb = r["rgb"].astype(np.float64)
    if patch is None:
        diff = rgb - np.asarray(target, np.float64)
        loss = float(np.mean(diff * diff))
        d_rgb = 2.0 * diff / diff.size
    else:
        from . import loss as oloss
        size, lam_mse, lam_perc = patch
        shp = (-1, size, size, 3)
        loss, _, _, g = oloss.patch_loss(rgb.reshape(shp), np.asarray(target, np.float64).reshape(shp), lam_mse, lam_perc)
        d_rgb = g.reshape(-1, 3)
    d_alpha = np.zeros(len(rgb))
    n = settings["n_samples"]
    d_sigma, d_color = comp.composite_bwd(r["comp"], r["sigma"], r["color"], r["delta"], r["lik"],
                                          scene["bg"], d_rgb, d_alpha, settings.get("eps_w", warp.EPS_W))
    fgf = r["fg_flat"]
    f = r["field"]
    ds = d_sigma.reshape(-1)[fgf]
    dc = d_color.reshape(-1, 3)[fgf]
    dh = mlp.radiance_heads_bwd(f["h"], dc, ds)
    dfeat, grad_rad_w, grad_rad_b = mlp.mlp_backward(f["rad_acts"], scene["rad_w"], dh)
    dtab, dxf = encoding.hash_encode_bwd(scene["hash_spec"], f["x_final"], scene["wbox_min"], f["cinv"],
                                         scene["table"], dfeat)
    grads = {"table": dtab, "rad_w": grad_rad_w, "rad_b": grad_rad_b}
    dxs = dxf.copy()
    if settings.get("offset_enabled", True):
        din, gw, gb = mlp.mlp_backward(f["off_acts"], scene["off_w"], dxf)
        npe = f["pe"].shape[1]
        dxs += encoding.posenc_bwd(r["warp"]["x_skel"][r["warp"]["fg"]], settings["pe_bands"],
                                   settings["pe_alpha"], din[:, :npe])
        grads["off_w"], grads["off_b"] = gw, gb
    wr = r["warp"]
    d_xskel_valid = np.zeros((len(r["flat"]), 3))
    d_xskel_valid[wr["fg"]] = dxs
    grads["vol"] = warp.skeleton_warp_bwd(wr, d_xskel_valid, np.asarray(scene["vol"]).shape,
                                          scene["wbox_min"], scene["wbox_max"])
    # motion bases (A4) and the pose vector through the residual MLP's first layer
    x_valid = r["x"].reshape(-1, 3)[r["flat"]]
    grads["g_r"], grads["g_t"] = warp.skeleton_warp_bwd_g(wr, x_valid, d_xskel_valid, scene["vol"],
                                                          scene["wbox_min"], scene["wbox_max"])
    if settings.get("offset_enabled", True):
        npe = f["pe"].shape[1]
        grads["pose_vec"] = np.asarray(scene["off_w"][0], np.float64)[npe:] @ grads["off_b"][0]
    return loss, grads, r


def occupancy_points(obox_min, obox_max):
    """2x2x2 probe points of every 32^3 cell (x-major cells), float32 kernel order."""
    res = camera.OCC_RES
    bmin = np.asarray(obox_min, F32)
    cw = ((np.asarray(obox_max, F32) - bmin).astype(F32) / F32(res)).astype(F32)
    cell = np.arange(res ** 3)
    c = np.stack([cell // (res * res), (cell // res) % res, cell % res], axis=1)
    j = np.arange(8)
    sub = np.stack([(j >> 2) & 1, (j >> 1) & 1, j & 1], axis=1)
    off = np.where(sub == 1, F32(0.75), F32(0.25)).astype(F32)
    q = (c[:, None, :].astype(F32) + off[None, :, :]).astype(F32)
    return (bmin + (q * cw).astype(F32)).astype(F32).reshape(-1, 3)


def occupancy_build(scene, settings, threshold, dtype=np.float32):
    """32^3 bitfield (uint32[1024]): bit set iff any probe point is foreground with
    sigma > threshold (builder-defined; PARITY UNPINNED).  Also returns per-point sigma."""
    pts = occupancy_points(scene["obox_min"], scene["obox_max"])
    wr = warp.skeleton_warp(pts, scene["g_r"], scene["g_t"], scene["vol"], scene["wbox_min"], scene["wbox_max"],
                            settings.get("eps_w", warp.EPS_W), dtype)
    sig = np.zeros(len(pts), dtype)
    f = _field(scene, wr["x_skel"][wr["fg"]], settings, dtype)
    sig[wr["fg"]] = f["sigma"]
    on = (wr["fg"] & (sig > threshold)).reshape(-1, 8).any(axis=1)
    bits = np.zeros(1024, np.uint32)
    idx = np.nonzero(on)[0]
    np.bitwise_or.at(bits, idx >> 5, (np.uint32(1) << (idx & 31).astype(np.uint32)))
    return bits, sig.reshape(-1, 8)
