"""SPEC known-answer examples on the sm_100a kernels (the same answers
tests/test_oracle_spec.py checks on the oracle):

* skeleton_warp ``S:331-336`` (``fv_warp_fwd``): identity at theta^c within 1e-6, single
  bone exact, far points background, normalised weights sum to 1 within 1e-5;
* positional_encode ``S:342-345`` (``fv_posenc_fwd``);
* composite ``S:433-437`` (``fv_composite_fwd``, ``fv_render_fwd``): sigma = 0 ->
  background, sigma delta = 20 -> c_1, homogeneous medium within 1e-3 at N = 128 through the
  render path's own sampler, zero likelihood contributes exactly 0, alpha + T = 1.
"""

import numpy as np
import pytest
import torch

from oracle import camera as ocam
from oracle import warp as owarp
from paper_2306_16541_b200.autodiff import posenc
from paper_2306_16541_b200.model import FreeviewModel
from paper_2306_16541_b200.render import RenderSettings, composite, skeleton_warp, stratified_sample

from helpers import make, oracle_scene

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _x(n, lo, hi, seed):
    return torch.from_numpy(np.random.default_rng(seed).uniform(lo, hi, (n, 3)).astype(np.float32)).to(DEV)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_warp_identity_at_canonical_pose(cfg):
    sc = make(cfg)
    nets = FreeviewModel(sc)
    k = nets.n_bones
    nets.set_pose_bases(np.broadcast_to(np.eye(3), (k, 3, 3)).copy(), np.zeros((k, 3)), np.zeros(3 * k))
    x = _x(8000, -0.9, 0.9, 1)
    xs, lik, fg = skeleton_warp(nets, x)
    fg = fg.cpu().numpy()
    assert fg.mean() > 0.9
    assert np.abs(xs.cpu().numpy()[fg] - x.cpu().numpy()[fg]).max() < 1e-6


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_warp_single_bone_exact_far_background_and_normalisation(cfg):
    sc = make(cfg)
    nets = FreeviewModel(sc)
    osc = oracle_scene(sc, nets=nets)
    # normalisation on the seeded W^c: weights from fv_warp_fwd's optional w output
    x = _x(20000, -1.2, 1.2, 4)
    n = x.shape[0]
    w = torch.empty((nets.n_bones, n), device=DEV)
    xs_ = torch.empty((n, 3), device=DEV)
    lik = torch.empty(n, device=DEV)
    fgb = torch.empty(n, dtype=torch.uint8, device=DEV)
    import ctypes as C
    from paper_2306_16541_b200 import _lib
    ws = nets.warp_struct()
    _lib.check(nets.lib.fv_warp_fwd(C.byref(ws), 1e-4, x.data_ptr(), n, xs_.data_ptr(), lik.data_ptr(),
                                    fgb.data_ptr(), w.data_ptr(), _lib.stream_ptr()))
    fg = fgb.cpu().numpy().astype(bool)
    assert 0.1 < fg.mean() < 1.0
    s = (w.cpu().numpy()[:, fg] / lik.cpu().numpy()[fg]).sum(axis=0)
    assert np.abs(s - 1.0).max() < 1e-5
    # far outside under every G_i
    d = np.random.default_rng(3).normal(size=(2000, 3))
    far = torch.from_numpy((50.0 * d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)).to(DEV)
    _, lk, fgf = skeleton_warp(nets, far)
    assert torch.all(lk == 0) and not bool(fgf.any())
    # single bone j with w^c = 1, others 0: x_skel = G_j(x) exactly where the bone
    # point is one voxel inside the grid
    j = 5
    logits = nets.views["vol_logits"]
    logits.fill_(-1e4)
    logits[j].fill_(0.0)
    nets.refresh()
    x = _x(20000, -0.9, 0.9, 2)
    xs, lk, fg = skeleton_warp(nets, x)
    p = owarp.bone_points(x.cpu().numpy(), osc["g_r"], osc["g_t"], np.float32)[j]
    g = nets.vol_res
    u = (p - osc["wbox_min"]) * (g - 1) / (osc["wbox_max"] - osc["wbox_min"])
    interior = np.all((u >= 1.0) & (u <= g - 2.0), axis=1)
    assert interior.sum() > 1000
    assert np.all(lk.cpu().numpy()[interior] == 1.0)
    assert np.array_equal(xs.cpu().numpy()[interior], p[interior])


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_warp_grid_boundaries_bitexact(cfg):
    """The grid-coordinate edge cases of ad:746-753 (inside iff 0 <= u <= G+1, floor clamped
    to [0, G]) on the kernel's bit-pattern inside test and round-down floor: runs of
    consecutive float32 points across u = 0, 1, G, G+1 on each axis (identity bones, so the
    bone point is x itself), plus NaN / inf coordinates, bit-exact against the oracle."""
    sc = make(cfg)
    nets = FreeviewModel(sc)
    k = nets.n_bones
    eye, zero = np.broadcast_to(np.eye(3, dtype=np.float32), (k, 3, 3)).copy(), np.zeros((k, 3), np.float32)
    nets.set_pose_bases(eye, zero, np.zeros(3 * k))
    osc = oracle_scene(sc, nets=nets)
    g = nets.vol_res
    wmin = np.asarray(osc["wbox_min"], np.float32)
    scale = ((np.float32(g) - np.float32(1.0)) / (np.asarray(osc["wbox_max"], np.float32) - wmin)).astype(np.float32)
    pts = []
    for ax in range(3):
        for u_edge in (0.0, 1.0, float(g), float(g + 1)):
            xb = np.float32(wmin[ax] + (u_edge - 1.0) / scale[ax])
            run = [xb]
            for _ in range(40):
                run.append(np.nextafter(run[-1], np.float32(np.inf), dtype=np.float32))
                run.insert(0, np.nextafter(run[0], np.float32(-np.inf), dtype=np.float32))
            p = np.zeros((len(run), 3), np.float32)
            p[:, ax] = run
            p[:, (ax + 1) % 3] = 0.1
            p[:, (ax + 2) % 3] = -0.2
            pts.append(p)
    odd = np.array([[np.nan, 0, 0], [0, np.inf, 0], [0, 0, -np.inf], [np.inf, np.inf, np.inf]], np.float32)
    x = np.concatenate(pts)
    xs, lik, fg = skeleton_warp(nets, torch.from_numpy(x).to(DEV))
    wr = owarp.skeleton_warp(x, eye, zero, osc["vol"], osc["wbox_min"], osc["wbox_max"], 1e-4, np.float32)
    assert np.array_equal(lik.cpu().numpy(), wr["L"])
    assert np.array_equal(fg.cpu().numpy(), wr["fg"])
    m = wr["fg"]
    assert 0.2 < m.mean() < 1.0
    assert np.array_equal(xs.cpu().numpy()[m], wr["x_skel"][m])
    # non-finite coordinates: every bone outside (NaN fails both comparisons of ad:746-753),
    # the clamped cell keeps the gather in bounds (the oracle's integer cast is undefined there)
    _, lk, fgo = skeleton_warp(nets, torch.from_numpy(odd).to(DEV))
    assert torch.all(lk == 0) and not bool(fgo.any())


def test_posenc_known_answers():
    pe = posenc(torch.zeros((1, 3), device=DEV), 6, 6.0).cpu().numpy()[0]
    assert np.all(pe[:3] == 0)
    for k in range(6):
        assert np.all(pe[3 + 6 * k: 6 + 6 * k] == 0.0) and np.all(pe[6 + 6 * k: 9 + 6 * k] == 1.0)
    pe = posenc(torch.tensor([[0.5, 0.0, 0.0]], device=DEV), 1, 1.0).cpu().numpy()[0]
    assert abs(pe[3] - 1.0) < 1e-6 and abs(pe[6]) < 1e-6
    pe = posenc(_x(10, -1, 1, 0), 6, 0.0).cpu().numpy()
    assert np.all(pe[:, 3:] == 0.0)


def _col(r, n, seed):
    return np.random.default_rng(seed).uniform(0, 1, (r, n, 3)).astype(np.float32)


def _c(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(DEV)


def test_composite_known_answers():
    r, n = 256, 128
    bg = (0.2, 0.4, 0.6)
    col = _col(r, n, 1)
    dl = np.full((r, n), 0.01, np.float32)
    one = np.ones((r, n), np.float32)
    rgb, alpha = composite(_c(np.zeros((r, n))), _c(col), _c(dl), _c(one), bg)
    assert torch.all(alpha == 0)
    assert np.array_equal(rgb.cpu().numpy(), np.broadcast_to(np.asarray(bg, np.float32), (r, 3)))
    sig = np.random.default_rng(2).uniform(0, 5, (r, n)).astype(np.float32)
    sig[:, 0] = 20.0 / dl[:, 0]
    rgb, alpha = composite(_c(sig), _c(col), _c(dl), _c(one), bg)
    assert np.abs(rgb.cpu().numpy() - col[:, 0]).max() < 1e-8
    assert np.abs(alpha.cpu().numpy() - 1.0).max() < 1e-8
    lik = np.where(np.random.default_rng(3).uniform(size=(r, n)) < 0.3, 0.0, 1.0).astype(np.float32)
    a_rgb, a_alpha = composite(_c(sig * (lik > 0)), _c(col), _c(dl), _c(one), bg)
    b_rgb, b_alpha = composite(_c(sig), _c(col), _c(dl), _c(lik), bg)
    assert torch.equal(a_rgb, b_rgb) and torch.equal(a_alpha, b_alpha)


def test_homogeneous_medium_through_the_render_sampler():
    """Constant sigma over each ray's [t_enter, t_exit] with the deltas of the render path's
    own stratified sampler (fv_march_warp): alpha within 1e-3 of 1 - exp(-sigma (t_f - t_n))
    at N = 128 (and no worse than at N = 32)."""
    sc = make("c1")
    nets = FreeviewModel(sc)
    osc = oracle_scene(sc)
    cc = ocam.camera_consts(sc.camera.intrinsics, sc.camera.world_to_camera)
    pix = np.arange(64 * 64)
    o, d = ocam.rays_f32(cc, pix, 64)
    t0, t1, hit = ocam.slab_f32(o, d, osc["obox_min"], osc["obox_max"])
    h = (t1 - t0).astype(np.float64)
    sigma = 1.3
    errs = []
    for n in (32, 128):
        st = RenderSettings(n_samples=n, jitter=True, seed=9)
        _, delta, count = stratified_sample(nets, sc.camera, torch.arange(64 * 64, dtype=torch.int32, device=DEV), st)
        assert np.array_equal(count.cpu().numpy() > 0, hit)
        dl = delta[torch.from_numpy(hit).to(DEV)]
        r = dl.shape[0]
        rgb, alpha = composite(torch.full_like(dl, sigma), torch.full((r, n, 3), 0.7, device=DEV), dl,
                               torch.ones_like(dl), (0.0, 0.0, 0.0))
        errs.append(np.abs(alpha.cpu().numpy() - (1.0 - np.exp(-sigma * h[hit]))).max())
    assert errs[1] < 1e-3 and errs[1] <= errs[0] + 1e-6
