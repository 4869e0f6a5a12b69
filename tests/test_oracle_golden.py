"""Pin the oracle to the real reference: golden vectors from tests/golden/make_golden.py."""

import os

import numpy as np
import pytest

from oracle import adam as oadam
from oracle import camera as ocam
from oracle import composite as ocomp
from oracle import encoding as oenc
from oracle import mlp as omlp
from oracle import skeleton as osk
from oracle import warp as owarp

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_primitives.npz"))
BMIN, BMAX = np.array([-1.0] * 3), np.array([1.0] * 3)


def test_sample_bone_channels_f64_bitexact():
    out = owarp.sample_bone_channels(G["sbc_vol"][:4], G["sbc_pts"], BMIN, BMAX, np.float64)
    assert np.array_equal(out, G["sbc_out"])


def test_sample_bone_channels_f32_close():
    out = owarp.sample_bone_channels(G["sbc_vol"][:4].astype(np.float32), G["sbc_pts"].astype(np.float32),
                                     BMIN, BMAX, np.float32)
    assert np.max(np.abs(out - G["sbc_out_f32"])) < 2e-6


def test_sample_bone_channels_gradients():
    dvol, dpts = owarp.sample_bone_channels_bwd(G["sbc_vol"].shape, G["sbc_pts"], BMIN, BMAX, G["sbc_up"],
                                                np.float64, vol=G["sbc_vol"])
    assert np.max(np.abs(dvol - G["sbc_dvol"])) < 1e-12
    assert np.max(np.abs(dpts - G["sbc_dpts"])) < 1e-12


@pytest.mark.parametrize("tag,alpha", [("full", 6.0), ("win", 2.3)])
def test_posenc(tag, alpha):
    p = G[f"pe_{tag}_p"]
    assert np.max(np.abs(oenc.posenc(p, 6, alpha, np.float64) - G[f"pe_{tag}_out"])) < 1e-15
    assert np.max(np.abs(oenc.posenc(p.astype(np.float32), 6, alpha, np.float32) - G[f"pe_{tag}_out_f32"])) == 0.0
    assert np.max(np.abs(oenc.posenc_bwd(p, 6, alpha, G[f"pe_{tag}_up"]) - G[f"pe_{tag}_dp"])) < 1e-12


def test_hann():
    assert np.max(np.abs(oenc.hann_band_weights(6, 2.3) - G["hann_23"])) == 0.0


def test_softmax0():
    out = owarp.softmax0(G["sm_x"])
    assert np.max(np.abs(out - G["sm_out"])) < 1e-15
    assert np.max(np.abs(owarp.softmax0_bwd(out, G["sm_up"]) - G["sm_dx"])) < 1e-15


def test_heads():
    assert np.max(np.abs(omlp.sigmoid(G["hd_x"]) - G["hd_sig"])) == 0.0
    assert np.max(np.abs(omlp.softplus(G["hd_x"]) - G["hd_sp"])) == 0.0


def test_mlp_forward_and_backward():
    ws = [G[f"mlp_w{i}"] for i in range(3)]
    bs = [G[f"mlp_b{i}"] for i in range(3)]
    out = omlp.mlp_forward(G["mlp_x"], ws, bs, np.float32)
    assert np.max(np.abs(out - G["mlp_out"])) < 1e-5
    _, acts = omlp.mlp_forward(G["mlp_x"], ws, bs, np.float64, keep=True)
    gx, gws, gbs = omlp.mlp_backward(acts, ws, G["mlp_up"])
    assert np.max(np.abs(gx - G["mlp_dx"])) < 1e-10
    for i in range(3):
        assert np.max(np.abs(gws[i] - G[f"mlp_dw{i}"])) < 1e-10
        assert np.max(np.abs(gbs[i] - G[f"mlp_db{i}"])) < 1e-10


def test_transmittance_matches_composite_scan():
    # the compositor's exclusive scan is the reference transmittance (ad:815-826)
    x = G["tr_x"]
    t = np.ones((x.shape[0], x.shape[1] + 1))
    for i in range(x.shape[1]):
        t[:, i + 1] = t[:, i] * x[:, i]
    assert np.max(np.abs(t - G["tr_out"])) < 1e-15


def test_composite_forward_and_backward():
    out = ocomp.composite(G["cp_sigma"], G["cp_color"], G["cp_delta"], G["cp_lik"], G["cp_bg"], dtype=np.float64)
    assert np.max(np.abs(out["rgb"] - G["cp_rgb"])) < 1e-12
    assert np.max(np.abs(out["alpha"] - G["cp_alpha"])) < 1e-12
    ds, dc = ocomp.composite_bwd(out, G["cp_sigma"], G["cp_color"], G["cp_delta"], G["cp_lik"], G["cp_bg"],
                                 G["cp_ur"], G["cp_ua"][:, 0])
    assert np.max(np.abs(ds - G["cp_dsigma"])) < 1e-12
    assert np.max(np.abs(dc - G["cp_dcolor"])) < 1e-12


def test_adam_three_steps():
    p0, p1 = G["adam_p0"].copy(), G["adam_p1"].copy()
    s0, s1 = oadam.AdamState([p0]), oadam.AdamState([p1])
    for i in range(3):
        oadam.adam_step([p0], [G[f"adam_g{i}_0"]], s0, 5e-4)
        oadam.adam_step([p1], [G[f"adam_g{i}_1"]], s1, 5e-5)
    assert np.max(np.abs(p0 - G["adam_out0"])) < 1e-15
    assert np.max(np.abs(p1 - G["adam_out1"])) < 1e-15


def test_adam_nonfinite_names_block():
    p = np.ones(2)
    with pytest.raises(FloatingPointError, match="radiance.l0.W"):
        oadam.adam_step([p], [np.array([np.nan, 0.0])], oadam.AdamState([p]), 0.1, names=["radiance.l0.W"])


def test_motion_basis_and_fk():
    r, t = osk.forward_kinematics(G["mb_parent"], G["mb_offs"], G["mb_ang"], G["mb_root"])
    assert np.max(np.abs(r - G["fk_r"])) < 1e-13 and np.max(np.abs(t - G["fk_t"])) < 1e-13
    gr, gt = osk.motion_basis(G["mb_parent"], G["mb_offs"], np.zeros((24, 3)), np.zeros(3), G["mb_ang"], G["mb_root"])
    assert np.max(np.abs(gr - G["mb_gr"])) < 1e-13 and np.max(np.abs(gt - G["mb_gt"])) < 1e-13


def test_camera_rays():
    o, d = ocam.rays_f64(G["cam_k"], G["cam_w2c"], 8, 6)
    assert np.max(np.abs(o - G["cam_o"])) < 1e-14 and np.max(np.abs(d - G["cam_d"])) < 1e-14
    k, w2c = ocam.orbit_camera((0, 0, 0), 0.0, 0.0, 3.0, 45.0, 64, 64)
    assert np.max(np.abs(k - G["cam3_k"])) == 0 and np.max(np.abs(w2c - G["cam3_w2c"])) == 0
    cc = ocam.camera_consts(G["cam_k"], G["cam_w2c"])
    o32, d32 = ocam.rays_f32(cc, np.arange(48), 8)
    assert np.max(np.abs(d32 - G["cam_d"])) < 1e-6 and np.max(np.abs(o32 - G["cam_o"])) < 1e-6


def test_skeleton_warp_forward_and_volume_gradient():
    lg = G["wp_logits"]
    vol = owarp.softmax0(lg)
    out = owarp.skeleton_warp(G["wp_x"], G["wp_gr"], G["wp_gt"], vol, BMIN, BMAX, dtype=np.float64)
    fg = G["wp_fg"]
    assert np.array_equal(out["fg"], fg)
    assert np.max(np.abs(out["x_skel"][fg] - G["wp_xskel"])) < 1e-12
    assert np.max(np.abs(out["L"][fg] - G["wp_L"])) < 1e-12
    d = np.zeros((len(fg), 3))
    d[fg] = G["wp_up"]
    dvol = owarp.skeleton_warp_bwd(out, d, vol.shape, BMIN, BMAX)
    dlog = owarp.softmax0_bwd(vol, dvol)
    assert np.max(np.abs(dlog - G["wp_dlogits"])) < 1e-12


def test_patch_loss_matches_reference_composition():
    from oracle import loss as oloss
    tot, mse, perc, dr = oloss.patch_loss(G["pl_r"], G["pl_t"])
    assert abs(tot - float(G["pl_loss"])) < 1e-12
    assert abs(mse - float(G["pl_mse"])) < 1e-12 and abs(perc - float(G["pl_perc"])) < 1e-12
    assert np.max(np.abs(dr - G["pl_dr"])) < 1e-12
    # S:500-503 known answers: identical patches -> 0; constant offset -> 0.2 * 0.01; symmetry
    t = G["pl_t"]
    assert oloss.patch_loss(t, t)[0] == 0.0
    off = oloss.patch_loss(t + 0.1, t)
    assert abs(off[0] - float(G["pl_offset_loss"])) < 1e-15 and abs(off[0] - 0.002) < 1e-12 and off[2] < 1e-12
    assert abs(oloss.patch_loss(G["pl_r"], t)[0] - oloss.patch_loss(t, G["pl_r"])[0]) < 1e-12


def test_weight_volume_generator_layer_matches_reference():
    """The generator's transposed convolution (torch/cuDNN) is the reference's
    conv_transpose3d (ad:633-699): values and both gradients."""
    import torch
    x = torch.tensor(G["ct_x"][None], requires_grad=True)
    w = torch.tensor(G["ct_w"], requires_grad=True)
    out = torch.nn.functional.conv_transpose3d(x, w, stride=2, padding=1)
    assert np.max(np.abs(out[0].detach().numpy() - G["ct_out"])) < 1e-12
    (out[0] * torch.tensor(G["ct_up"])).sum().backward()
    assert np.max(np.abs(x.grad[0].numpy() - G["ct_dx"])) < 1e-12
    assert np.max(np.abs(w.grad.numpy() - G["ct_dw"])) < 1e-12


def test_weight_volume_generator_shape_and_softmax():
    import torch
    from paper_2306_16541_b200.weightnet import WeightVolumeNet
    net = WeightVolumeNet(25, seed=3)
    with torch.no_grad():
        logits = net()
    assert tuple(logits.shape) == (25, 32, 32, 32)                      # S:295-296 known answer
    wc = torch.softmax(logits, 0)
    assert float((wc.sum(0) - 1).abs().max()) < 1e-6
    with torch.no_grad():
        assert torch.equal(WeightVolumeNet(25, seed=3)(), logits)         # constant latent: deterministic


def test_warp_gradient_into_motion_bases():
    """dL/dG_i of the skinning warp (A4) vs the reference Tape (golden wg_*)."""
    K = G["wp_gr"].shape[0]
    vol = owarp.softmax0(G["wp_logits"])
    xf = G["wp_x"][G["wp_fg"]]
    wr = owarp.skeleton_warp(xf, G["wp_gr"], G["wp_gt"], vol, BMIN, BMAX, 1e-4, np.float64)
    assert wr["fg"].all()
    dgr, dgt = owarp.skeleton_warp_bwd_g(wr, xf, G["wp_up"], vol, BMIN, BMAX)
    assert np.max(np.abs(dgr - G["wg_dgr"])) < 1e-10
    assert np.max(np.abs(dgt - G["wg_dgt"].reshape(K, 3))) < 1e-10


def test_torch_motion_basis_and_pose_gradient_match_reference():
    """pose.motion_basis (float64 torch, used to train the pose refiner) reproduces the
    reference's motion bases and its Tape gradient into the joint angles (golden mb_*)."""
    import torch
    from paper_2306_16541_b200.pose import motion_basis as mb_t
    from paper_2306_16541_b200.skeleton import Skeleton
    skel = Skeleton(parent=G["mb_parent"], rest_offset=G["mb_offs"], canonical_angles=np.zeros((24, 3)),
                    canonical_root=np.zeros(3))
    ang = torch.tensor(G["mb_ang"], requires_grad=True)
    root = torch.tensor(G["mb_root"], requires_grad=True)
    gr, gt = mb_t(skel, ang, root)
    assert np.max(np.abs(gr.detach().numpy() - G["mb_gr"])) < 1e-12
    assert np.max(np.abs(gt.detach().numpy() - G["mb_gt"])) < 1e-12
    ((gr * torch.tensor(G["mb_ugr"])).sum() + (gt * torch.tensor(G["mb_ugt"])).sum()).backward()
    assert np.max(np.abs(ang.grad.numpy() - G["mb_dang"])) < 1e-10
    assert np.max(np.abs(root.grad.numpy() - G["mb_droot"])) < 1e-10


def test_pose_refiner_known_answers():
    """SPEC refine_pose examples: fresh net -> identity exactly; rotation
    composition about a shared axis; joints untouched."""
    import torch
    from paper_2306_16541_b200.pose import PoseRefinerNet, rodrigues, rotation_log
    net = PoseRefinerNet(24, seed=1)
    om = torch.tensor(np.random.default_rng(0).normal(0, 0.3, (24, 3)))
    assert torch.equal(net.refine(om), om)
    w = torch.tensor([[0.0, 0.0, np.pi / 4]], dtype=torch.float64)
    dw = torch.tensor([[0.0, 0.0, np.pi / 2]], dtype=torch.float64)
    comp = rotation_log(rodrigues(dw) @ rodrigues(w))
    assert np.max(np.abs(comp.numpy() - [[0.0, 0.0, 3 * np.pi / 4]])) < 1e-9
    r = rodrigues(om)
    assert float((rotation_log(r) - om).abs().max()) < 1e-12
