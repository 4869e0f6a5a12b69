"""SPEC known-answer examples (SURVEY §4 "SPEC known-answer examples that no test
implements") as self-tests of the CPU oracle, float64 and float32 kernel order.

* skeleton_warp ``S:331-336``: identity at theta^c, single bone, far points, normalisation;
* positional_encode ``S:342-345``;
* composite ``S:433-437``: sigma = 0, sigma delta = 20, homogeneous medium at N = 128,
  zero likelihood; plus the telescoping invariant ``S:449``.
"""

import numpy as np
import pytest

from oracle import camera as ocam
from oracle import composite as ocomp
from oracle import encoding as oenc
from oracle import warp as owarp

from helpers import make, oracle_scene

EPS_W = 1e-4


@pytest.fixture(scope="module")
def c1():
    sc = make("c1")
    return sc, oracle_scene(sc)


def _inside_points(osc, n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-0.9, 0.9, (n, 3)).astype(np.float32)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_skeleton_warp_identity_at_canonical_pose(c1, dtype):
    """theta^o = theta^c and x inside the subject -> x_skel = x within 1e-6."""
    sc, osc = c1
    k = sc.cfg.n_bones
    eye, zero = np.broadcast_to(np.eye(3), (k, 3, 3)).copy(), np.zeros((k, 3))
    x = _inside_points(osc, 5000, 1)
    wr = owarp.skeleton_warp(x, eye, zero, osc["vol"], osc["wbox_min"], osc["wbox_max"], EPS_W, dtype)
    assert wr["fg"].mean() > 0.9
    assert np.abs(wr["x_skel"][wr["fg"]] - x[wr["fg"]]).max() < 1e-6


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_skeleton_warp_single_bone_is_exact(c1, dtype):
    """one bone with w^c = 1, the others 0 -> x_skel = G_i(x) exactly (points whose
    bone point is one voxel inside the grid, where the trilinear sample is exactly 1)."""
    sc, osc = c1
    vol = np.zeros_like(osc["vol"])
    j = 5
    vol[j] = 1.0
    x = _inside_points(osc, 20000, 2)
    wr = owarp.skeleton_warp(x, osc["g_r"], osc["g_t"], vol, osc["wbox_min"], osc["wbox_max"], EPS_W, dtype)
    p = owarp.bone_points(x, osc["g_r"], osc["g_t"], dtype)[j]
    g = vol.shape[1]
    u = (p - osc["wbox_min"]) * (g - 1) / (osc["wbox_max"] - osc["wbox_min"])
    interior = np.all((u >= 1.0) & (u <= g - 2.0), axis=1)
    assert interior.sum() > 1000
    if dtype is np.float32:     # the kernel's lerp form: a blend of equal corners is exact
        assert np.all(wr["L"][interior] == 1.0)
        assert np.array_equal(wr["x_skel"][interior], p[interior])
    else:                       # the reference's product-weight sum (ad:767-773): 1 to an ulp
        assert np.abs(wr["L"][interior] - 1.0).max() < 1e-14
        assert np.abs(wr["x_skel"][interior] - p[interior]).max() < 1e-14


def test_skeleton_warp_far_points_are_background(c1):
    """x far outside the canonical box under all G_i -> likelihood 0, background."""
    sc, osc = c1
    rng = np.random.default_rng(3)
    d = rng.normal(size=(2000, 3))
    x = (50.0 * d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    for dt in (np.float64, np.float32):
        wr = owarp.skeleton_warp(x, osc["g_r"], osc["g_t"], osc["vol"], osc["wbox_min"], osc["wbox_max"], EPS_W, dt)
        assert np.all(wr["L"] == 0) and not wr["fg"].any()


def test_skeleton_warp_normalised_weights_sum_to_one(c1):
    """normalised weights sum to 1 within 1e-5 wherever likelihood > eps_w."""
    sc, osc = c1
    x = np.random.default_rng(4).uniform(-1.2, 1.2, (20000, 3)).astype(np.float32)
    wr = owarp.skeleton_warp(x, osc["g_r"], osc["g_t"], osc["vol"], osc["wbox_min"], osc["wbox_max"], EPS_W,
                             np.float32)
    fg = wr["fg"]
    assert 0.1 < fg.mean() < 1.0
    s = (wr["w"][:, fg] / wr["L"][fg]).sum(axis=0)
    assert np.abs(s - 1.0).max() < 1e-5


def test_positional_encode_known_answers():
    """S:343-345."""
    pe = oenc.posenc(np.zeros((1, 3)), 6, 6.0, np.float64)[0]
    assert np.all(pe[:3] == 0)
    for k in range(6):
        assert np.all(pe[3 + 6 * k: 6 + 6 * k] == 0.0) and np.all(pe[6 + 6 * k: 9 + 6 * k] == 1.0)
    pe = oenc.posenc(np.array([[0.5, 0.0, 0.0]]), 1, 1.0, np.float64)[0]
    assert abs(pe[3] - 1.0) < 1e-12 and abs(pe[6]) < 1e-12
    pe = oenc.posenc(np.random.default_rng(0).uniform(-1, 1, (10, 3)), 6, 0.0, np.float64)
    assert np.all(pe[:, 3:] == 0.0)


def _col(r, n, seed):
    return np.random.default_rng(seed).uniform(0, 1, (r, n, 3))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_composite_known_answers(dtype):
    """S:434-437 on the oracle compositor."""
    r, n = 64, 128
    bg = np.array([0.2, 0.4, 0.6])
    col = _col(r, n, 1)
    dl = np.full((r, n), 0.01)
    one = np.ones((r, n))
    # all sigma = 0 -> background, alpha 0
    out = ocomp.composite(np.zeros((r, n)), col, dl, one, bg, dtype=dtype)
    assert np.all(out["alpha"] == 0) and np.allclose(out["rgb"], bg[None], atol=0)
    # sigma_1 delta_1 = 20, likelihood 1 -> rgb = c_1 within 1e-8, alpha ~ 1
    sig = np.random.default_rng(2).uniform(0, 5, (r, n))
    sig[:, 0] = 20.0 / dl[:, 0]
    out = ocomp.composite(sig, col, dl, one, bg, dtype=dtype)
    assert np.abs(out["rgb"] - col[:, 0].astype(dtype)).max() < 1e-8    # c_1 as the dtype holds it
    assert np.abs(out["alpha"] - 1.0).max() < 1e-8
    # likelihood 0 contributes exactly 0: same result as that sample's sigma set to 0
    lik = np.where(np.random.default_rng(3).uniform(size=(r, n)) < 0.3, 0.0, 1.0)
    a = ocomp.composite(sig * (lik > 0), col, dl, one, bg, dtype=dtype)
    b = ocomp.composite(sig, col, dl, lik, bg, dtype=dtype)
    assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["alpha"], b["alpha"])
    # telescoping: alpha + final transmittance = 1 exactly
    assert np.array_equal(b["alpha"] + b["T"][:, -1], np.ones(r, dtype))


def test_composite_homogeneous_medium_through_the_sampler():
    """constant sigma and colour over [t_n, t_f], N = 128 stratified jittered samples
    (the repo's delta rule) -> alpha within 1e-3 of 1 - exp(-sigma (t_f - t_n)),
    converging as N grows."""
    sc = make("c1")
    osc = oracle_scene(sc)
    cc = ocam.camera_consts(sc.camera.intrinsics, sc.camera.world_to_camera)
    pix = np.arange(64 * 64)
    o, d = ocam.rays_f32(cc, pix, 64)
    t0, t1, hit = ocam.slab_f32(o, d, osc["obox_min"], osc["obox_max"])
    errs = []
    for n in (32, 128):
        _, dl, _ = ocam.stratified_f32(t0, t1, hit, pix, n, True, 9)
        dl, h = dl[hit], (t1 - t0)[hit]
        sigma = 1.3
        out = ocomp.composite(np.full(dl.shape, sigma), np.full(dl.shape + (3,), 0.7), dl, np.ones(dl.shape),
                              np.zeros(3), dtype=np.float32)
        errs.append(np.abs(out["alpha"] - (1.0 - np.exp(-sigma * h.astype(np.float64)))).max())
    assert errs[1] < 1e-3 and errs[1] <= errs[0] + 1e-6
