"""Generate the golden vectors that pin the oracle to the REAL reference.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the reference package ``freeview`` from /root/reference/pkg/src, evaluates
its own primitives (and compositions of them, for SPEC operations the package only
specifies) on small seeded inputs, and writes ``tests/golden/ref_primitives.npz``.
The .npz is committed; tests never import the reference at run time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("FREEVIEW_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from freeview import autodiff as ad  # noqa: E402
from freeview import capture as cap  # noqa: E402
from freeview import fused as fu  # noqa: E402
from freeview import skeleton as sk  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_primitives.npz")
SMPL24 = [-1, 0, 0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 9, 9, 12, 13, 14, 16, 17, 18, 19, 20, 21]


def grads(fn, *tensors):
    for t in tensors:
        t.requires_grad = True
        t.zero_grad()
    with ad.Tape() as tape:
        y = fn(*tensors)
        tape.backward(y)
    return [t.grad.copy() for t in tensors]


def main():
    rng = np.random.default_rng(2306)
    g = {}

    # --- sample_bone_channels (ad:728-808): values and both gradients, f64 and f32
    vol = rng.uniform(0, 1, (5, 8, 8, 8))
    pts = rng.uniform(-1.3, 1.3, (4, 200, 3))
    pts[0, :5] = [[-1, -1, -1], [1, 1, 1], [0, 0, 0], [5, 5, 5], [-1.05, 0.2, 0.3]]
    up = rng.normal(size=(4, 200))
    bmin, bmax = np.array([-1.0, -1.0, -1.0]), np.array([1.0, 1.0, 1.0])
    g["sbc_vol"], g["sbc_pts"], g["sbc_up"] = vol, pts, up
    g["sbc_out"] = ad.sample_bone_channels(ad.Tensor(vol), ad.Tensor(pts), bmin, bmax).data
    g["sbc_out_f32"] = ad.sample_bone_channels(ad.Tensor(vol.astype(np.float32)), ad.Tensor(pts.astype(np.float32)),
                                               bmin, bmax).data
    gv, gp = grads(lambda v, p: ad.tsum(ad.mul(ad.sample_bone_channels(v, p, bmin, bmax), ad.Tensor(up))),
                   ad.Tensor(vol.copy()), ad.Tensor(pts.copy()))
    g["sbc_dvol"], g["sbc_dpts"] = gv, gp

    # --- posenc (ad:574-615)
    p = rng.uniform(-1, 1, (20, 3))
    for tag, alpha in (("full", 6.0), ("win", 2.3)):
        up = rng.normal(size=(20, ad.posenc_dim(6)))
        g[f"pe_{tag}_p"], g[f"pe_{tag}_up"] = p, up
        g[f"pe_{tag}_out"] = ad.posenc(ad.Tensor(p), 6, alpha).data
        g[f"pe_{tag}_out_f32"] = ad.posenc(ad.Tensor(p.astype(np.float32)), 6, alpha).data
        g[f"pe_{tag}_dp"] = grads(lambda t: ad.tsum(ad.mul(ad.posenc(t, 6, alpha), ad.Tensor(up))),
                                  ad.Tensor(p.copy()))[0]
    g["hann_23"] = ad.hann_band_weights(6, 2.3)

    # --- softmax0 (ad:711-721)
    x = rng.normal(size=(6, 3, 3, 3))
    up = rng.normal(size=x.shape)
    g["sm_x"], g["sm_up"], g["sm_out"] = x, up, ad.softmax0(ad.Tensor(x)).data
    g["sm_dx"] = grads(lambda t: ad.tsum(ad.mul(ad.softmax0(t), ad.Tensor(up))), ad.Tensor(x.copy()))[0]

    # --- transmittance (ad:815-837)
    at = rng.uniform(0, 1, (5, 9))
    at[1, 3] = 0.0
    up = rng.normal(size=(5, 10))
    g["tr_x"], g["tr_up"], g["tr_out"] = at, up, ad.transmittance(ad.Tensor(at)).data
    g["tr_dx"] = grads(lambda t: ad.tsum(ad.mul(ad.transmittance(t), ad.Tensor(up))), ad.Tensor(at.copy()))[0]

    # --- heads (ad:200-222)
    h = rng.normal(scale=3.0, size=(50,))
    g["hd_x"], g["hd_sig"], g["hd_sp"] = h, ad.sigmoid(ad.Tensor(h)).data, ad.softplus(ad.Tensor(h)).data

    # --- MLP: FusedMlp.random(32,4,depth=2) + naive_forward (fu:124-142), linear bwd (ad:403-425)
    mlp = fu.FusedMlp.random(32, 4, depth=2, seed=3)
    xin = rng.uniform(-1, 1, (100, 32)).astype(np.float32)
    for i, (w, b) in enumerate(zip(mlp.weights, mlp.biases)):
        g[f"mlp_w{i}"], g[f"mlp_b{i}"] = w, b
    g["mlp_x"], g["mlp_out"] = xin, fu.naive_forward(mlp, xin)
    ws = [ad.Tensor(w.astype(np.float64)) for w in mlp.weights]
    bs = [ad.Tensor(b.astype(np.float64)) for b in mlp.biases]
    up = rng.normal(size=(100, 4))
    g["mlp_up"] = up

    def mlp_loss(x, w0, w1, w2, b0, b1, b2):
        h1 = ad.linear(x, w0, b0, "relu")
        h2 = ad.linear(h1, w1, b1, "relu")
        return ad.tsum(ad.mul(ad.linear(h2, w2, b2, "none"), ad.Tensor(up)))

    gr = grads(mlp_loss, ad.Tensor(xin.astype(np.float64)), *ws, *bs)
    for name, val in zip(["dx", "dw0", "dw1", "dw2", "db0", "db1", "db2"], gr):
        g[f"mlp_{name}"] = val

    # --- Adam (ad:880-912): three steps, two blocks, distinct lrs
    p0 = rng.normal(size=(7,))
    p1 = rng.normal(size=(3, 2))
    gs = [(rng.normal(size=(7,)), rng.normal(size=(3, 2))) for _ in range(3)]
    g["adam_p0"], g["adam_p1"] = p0.copy(), p1.copy()
    for i, (a, b) in enumerate(gs):
        g[f"adam_g{i}_0"], g[f"adam_g{i}_1"] = a, b
    t0, t1 = ad.Tensor(p0.copy()), ad.Tensor(p1.copy())
    st = ad.AdamState([t0], beta1=0.9, beta2=0.99)
    st1 = ad.AdamState([t1], beta1=0.9, beta2=0.99)
    for a, b in gs:
        ad.adam_step([t0], [a], st, lr=5e-4)
        ad.adam_step([t1], [b], st1, lr=5e-5)
    g["adam_out0"], g["adam_out1"] = t0.data, t1.data

    # --- motion_basis / FK (sk:186-303) for a seeded 24-joint skeleton
    rest = rng.uniform(-1, 1, (24, 3))
    offs = rest.copy()
    par = np.array(SMPL24)
    offs[1:] = rest[1:] - rest[par[1:]]
    names = [f"j{i}" for i in range(24)]
    skel = sk.Skeleton(names=names, parent=par, rest_offset=offs, canonical_angles=np.zeros((24, 3)),
                       canonical_root=np.zeros(3), tip=np.zeros((24, 3)))
    ang = rng.normal(0, 0.2, (24, 3))
    root = np.array([0.05, -0.02, 0.1])
    gr_, gt_ = sk.motion_basis(skel, ad.Tensor(ang), ad.Tensor(root))
    g["mb_parent"], g["mb_offs"], g["mb_ang"], g["mb_root"] = par, offs, ang, root
    g["mb_gr"], g["mb_gt"] = gr_.data, gt_.data
    rw, tw = sk.forward_kinematics_np(skel, ang, root)
    g["fk_r"], g["fk_t"] = rw, tw

    # --- camera rays (cap:73-142)
    cam = cap.orbit_camera((0.0, 0.1, 0.0), 30.0, 10.0, 3.0, 45.0, 8, 6)
    o, d = cam.rays()
    g["cam_k"], g["cam_w2c"], g["cam_o"], g["cam_d"] = cam.intrinsics, cam.world_to_camera, o, d
    cam3 = cap.orbit_camera((0.0, 0.0, 0.0), 0.0, 0.0, 3.0, 45.0, 64, 64)
    g["cam3_k"], g["cam3_w2c"] = cam3.intrinsics, cam3.world_to_camera

    # --- composite composed from reference ops; grads through the Tape
    R, N, eps = 6, 10, 1e-4
    sig = rng.uniform(0, 3, (R, N))
    dl = rng.uniform(0.01, 0.3, (R, N))
    lik = rng.uniform(0, 1, (R, N))
    lik[0, 2], lik[1, :] = 0.0, 5e-5
    col = rng.uniform(0, 1, (R, N, 3))
    bg = np.array([[0.2, 0.4, 0.6]])
    ur, ua = rng.normal(size=(R, 3)), rng.normal(size=(R, 1))

    def comp(sigma, color):
        a = ad.sub(ad.Tensor(np.ones((R, N))), ad.exp(ad.neg(ad.mul(sigma, ad.Tensor(dl)))))
        gate = ad.clamp(ad.div(ad.Tensor(lik), ad.Tensor(np.full((R, N), eps))), 0.0, 1.0)
        ab = ad.mul(a, gate)
        tr = ad.transmittance(ad.sub(ad.Tensor(np.ones((R, N))), ab))
        w = ad.mul(ad.slice_cols(tr, 0, N), ab)
        tn = ad.slice_cols(tr, N, N + 1)
        rgb = ad.add(ad.weighted_sum1(w, color), ad.matmul(tn, ad.Tensor(bg)))
        alpha = ad.sub(ad.Tensor(np.ones((R, 1))), tn)
        return rgb, alpha

    rgb, alpha = comp(ad.Tensor(sig), ad.Tensor(col))
    g["cp_sigma"], g["cp_delta"], g["cp_lik"], g["cp_color"], g["cp_bg"] = sig, dl, lik, col, bg[0]
    g["cp_rgb"], g["cp_alpha"], g["cp_ur"], g["cp_ua"] = rgb.data, alpha.data[:, 0], ur, ua

    def comp_loss(sigma, color):
        rgb_, alpha_ = comp(sigma, color)
        return ad.add(ad.tsum(ad.mul(rgb_, ad.Tensor(ur))), ad.tsum(ad.mul(alpha_, ad.Tensor(ua))))

    g["cp_dsigma"], g["cp_dcolor"] = grads(comp_loss, ad.Tensor(sig.copy()), ad.Tensor(col.copy()))

    # --- skeleton warp (S:327-336 / Eqs 7-9) composed from reference ops, grads into logits
    K, M = 4, 64
    logits = rng.uniform(0, 1, (K + 1, 8, 8, 8))
    grw = sk.rodrigues_np(rng.normal(0, 0.3, (K, 3)))
    gtw = rng.normal(0, 0.2, (K, 3))
    xw = rng.uniform(-0.9, 0.9, (M, 3))
    pw = np.einsum("kij,nj->kni", grw, xw) + gtw[:, None, :]
    vol_sm = ad.softmax0(ad.Tensor(logits)).data
    w_all = ad.sample_bone_channels(ad.Tensor(vol_sm), ad.Tensor(pw), bmin, bmax).data
    fgm = w_all.sum(axis=0) > eps
    upx = rng.normal(size=(int(fgm.sum()), 3))

    def warp(lg):
        v = ad.softmax0(lg)
        w = ad.sample_bone_channels(v, ad.Tensor(pw[:, fgm]), bmin, bmax)
        L = ad.sum0(w)
        wn = ad.div(w, ad.stack0([L] * K))
        return ad.weighted_sum0(wn, ad.Tensor(pw[:, fgm])), L

    xs, L = warp(ad.Tensor(logits))
    g["wp_logits"], g["wp_gr"], g["wp_gt"], g["wp_x"] = logits, grw, gtw, xw
    g["wp_fg"], g["wp_xskel"], g["wp_L"], g["wp_up"] = fgm, xs.data, L.data, upx
    g["wp_dlogits"] = grads(lambda lg: ad.tsum(ad.mul(warp(lg)[0], ad.Tensor(upx))), ad.Tensor(logits.copy()))[0]

    # --- SPEC compute_loss composed from reference ops: lam_mse * MSE + lam_perc *
    # multi-scale gradient difference (diff_axis ad:844, avgpool2 ad:862, absval, tmean)
    pr = rng.uniform(0, 1, (3, 8, 8, 3))
    pt = rng.uniform(0, 1, (3, 8, 8, 3))

    def patch_loss(r, t, lam_mse=0.2, lam_perc=1.0):
        e = ad.sub(r, t)
        mse = ad.tmean(ad.mul(e, e))
        terms = []
        for lvl in range(2):
            if lvl:
                r, t = ad.avgpool2(r), ad.avgpool2(t)
            for ax in (2, 1):
                terms.append(ad.tmean(ad.absval(ad.sub(ad.diff_axis(r, ax), ad.diff_axis(t, ax)))))
        perc = ad.add(ad.add(terms[0], terms[1]), ad.add(terms[2], terms[3]))
        return ad.add(ad.mul_scalar(mse, lam_mse), ad.mul_scalar(perc, lam_perc)), mse, perc

    tot, mse, perc = patch_loss(ad.Tensor(pr), ad.Tensor(pt))
    g["pl_r"], g["pl_t"] = pr, pt
    g["pl_loss"], g["pl_mse"], g["pl_perc"] = tot.data, mse.data, perc.data
    g["pl_dr"] = grads(lambda r: patch_loss(r, ad.Tensor(pt))[0], ad.Tensor(pr.copy()))[0]
    g["pl_offset_loss"] = patch_loss(ad.Tensor(pt + 0.1), ad.Tensor(pt))[0].data   # S:502 known answer

    # --- conv_transpose3d (ad:633-699), the weight-volume generator's layer
    cx = rng.normal(size=(3, 4, 4, 4))
    cw = rng.normal(size=(3, 2, 4, 4, 4))
    cup = rng.normal(size=(2, 8, 8, 8))
    g["ct_x"], g["ct_w"], g["ct_up"] = cx, cw, cup
    g["ct_out"] = ad.conv_transpose3d(ad.Tensor(cx), ad.Tensor(cw), 2, 1).data
    g["ct_dx"], g["ct_dw"] = grads(lambda a, b: ad.tsum(ad.mul(ad.conv_transpose3d(a, b, 2, 1), ad.Tensor(cup))),
                                   ad.Tensor(cx.copy()), ad.Tensor(cw.copy()))

    # --- gradients into the motion bases and the pose (A4: dL/dG_i of the skinning warp,
    # chained through motion_basis to the joint angles) -- the reference's own Tape
    xf = xw[fgm]
    mf = xf.shape[0]

    def warp_g(rr, tt):
        xk = ad.Tensor(np.broadcast_to(xf, (K, mf, 3)).copy())
        pts = ad.add(ad.bmm(xk, ad.transpose_last2(rr)), ad.bmm(ad.Tensor(np.ones((K, mf, 1))), tt))
        v = ad.Tensor(ad.softmax0(ad.Tensor(logits)).data)
        w = ad.sample_bone_channels(v, pts, bmin, bmax)
        L = ad.sum0(w)
        wn = ad.div(w, ad.stack0([L] * K))
        return ad.weighted_sum0(wn, pts)

    g["wg_dgr"], g["wg_dgt"] = grads(lambda rr, tt: ad.tsum(ad.mul(warp_g(rr, tt), ad.Tensor(upx))),
                                     ad.Tensor(grw.copy()), ad.Tensor(gtw.reshape(K, 1, 3).copy()))
    ugr, ugt = rng.normal(size=(24, 3, 3)), rng.normal(size=(24, 3))

    def mb_loss(a, r0):
        gr__, gt__ = sk.motion_basis(skel, a, r0)
        return ad.add(ad.tsum(ad.mul(gr__, ad.Tensor(ugr))), ad.tsum(ad.mul(gt__, ad.Tensor(ugt))))

    g["mb_ugr"], g["mb_ugt"] = ugr, ugt
    g["mb_dang"], g["mb_droot"] = grads(mb_loss, ad.Tensor(ang.copy()), ad.Tensor(root.copy()))

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1024:.1f} KiB, {len(g)} arrays)")


if __name__ == "__main__":
    main()
