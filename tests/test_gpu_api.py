"""The reference-named operator layer: ``autodiff.{sample_bone_channels, posenc,
transmittance, softmax0}``, ``fused.{FusedMlp, fused_forward}`` and the SPEC functions
``positional_encode``, ``residual_offset``, ``stratified_sample`` -- each one CUDA kernel
chain through the C ABI -- against the CPU oracle on the same seeded inputs, plus the
reference's error behaviour (DimensionError on bad shapes, no CPU fallback)."""

import numpy as np
import pytest
import torch

from oracle import camera as ocam
from oracle import encoding as oenc
from oracle import mlp as omlp
from oracle import pipeline as opipe
from oracle import warp as owarp
from oracle.adapter import settings as osettings
from paper_2306_16541_b200 import autodiff, fused
from paper_2306_16541_b200.errors import DimensionError
from paper_2306_16541_b200.model import FreeviewModel
from paper_2306_16541_b200.render import (RenderSettings, positional_encode, residual_offset,
                                          stratified_sample)

from helpers import make, oracle_scene

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def c1():
    sc = make("c1", table_scale=0.5, bias_scale=0.05)
    nets = FreeviewModel(sc)
    return sc, nets, oracle_scene(sc, nets=nets)


@pytest.mark.parametrize("half", [False, True])
def test_sample_bone_channels_matches_oracle(half):
    """fp32 volume: bit-exact with the oracle's float32 lerp form; fp16-packed volume
    (config 2): bit-exact against the oracle on the fp16-rounded volume."""
    sc = make("c2" if half else "c1", width=16, height=16, table_scale=0.5)
    nets = FreeviewModel(sc)
    osc = oracle_scene(sc, nets=nets)
    k = nets.n_bones
    rng = np.random.default_rng(3)
    lo, hi = np.asarray(osc["wbox_min"]), np.asarray(osc["wbox_max"])
    pts = rng.uniform(lo - 0.15, hi + 0.15, (k, 4000, 3)).astype(np.float32)   # incl. outside the padded grid
    got = autodiff.sample_bone_channels(nets, torch.from_numpy(pts).to(DEV)).cpu().numpy()
    ref = owarp.sample_bone_channels(osc["vol"][:k], pts, osc["wbox_min"], osc["wbox_max"], np.float32)
    assert got.shape == (k, 4000)
    assert np.array_equal(got, ref)
    assert (ref == 0).mean() > 0.02 and (ref > 0).mean() > 0.5
    with pytest.raises(DimensionError):
        autodiff.sample_bone_channels(nets, torch.zeros((k + 1, 5, 3), device=DEV))


@pytest.mark.parametrize("alpha", [6.0, 3.5, 0.0])
def test_posenc_and_positional_encode_match_oracle(alpha):
    rng = np.random.default_rng(5)
    p = rng.uniform(-1.2, 1.2, (5000, 3)).astype(np.float32)
    got = autodiff.posenc(torch.from_numpy(p).to(DEV), 6, alpha).cpu().numpy()
    ref = oenc.posenc(p, 6, alpha, np.float32)
    assert got.shape == (5000, 39)
    assert np.array_equal(got[:, :3], ref[:, :3])               # raw columns copied
    assert np.max(np.abs(got - ref)) < 2e-6                     # sincosf vs numpy sin/cos
    spec = positional_encode(torch.from_numpy(p).to(DEV), 6, alpha).cpu().numpy()
    assert np.array_equal(spec, got)
    with pytest.raises(DimensionError):
        autodiff.posenc(torch.zeros((4, 2), device=DEV), 6)
    with pytest.raises(DimensionError):
        autodiff.posenc(torch.zeros((4, 3)), 6)                 # CPU tensor: no fallback


def test_transmittance_matches_running_product():
    rng = np.random.default_rng(7)
    a = rng.uniform(0, 0.3, (700, 96)).astype(np.float32)
    a[::7, 40:] = 1.0                                           # fully opaque samples
    got = autodiff.transmittance(torch.from_numpy(a).to(DEV)).cpu().numpy()
    ref = np.concatenate([np.ones((700, 1), np.float32), np.cumprod(np.float32(1) - a, axis=1, dtype=np.float32)], 1)
    assert got.shape == (700, 97)
    assert np.array_equal(got, ref)
    assert np.all(got[::7, 41:] == 0)
    assert autodiff.transmittance(torch.zeros((0, 5), device=DEV)).shape == (0, 6)


def test_softmax0_matches_oracle():
    rng = np.random.default_rng(9)
    z = rng.uniform(0, 1, (25, 12, 12, 12)).astype(np.float32)
    got = autodiff.softmax0(torch.from_numpy(z).to(DEV)).cpu().numpy()
    ref = owarp.softmax0(z.astype(np.float64))
    assert np.max(np.abs(got - ref)) < 1e-6
    assert np.allclose(got.sum(0), 1.0, atol=1e-6)


def test_fused_forward_matches_naive_and_is_chunk_invariant():
    """fu:182-193 / t_fused:48-86: equivalence with the naive MLP (fp32-accurate here, bar
    2e-5 of the output scale instead of the reference's 1e-3) and bitwise chunk invariance."""
    mlp = fused.FusedMlp.random(32, 4, depth=2, width=64, seed=1)
    rng = np.random.default_rng(2)
    x = rng.standard_normal((10000, 32)).astype(np.float32)
    xt = torch.from_numpy(x).to(DEV)
    y = fused.fused_forward(mlp, xt).cpu().numpy()
    ws = [w.cpu().numpy().astype(np.float64) for w in mlp.weights]
    bs = [b.cpu().numpy().astype(np.float64) for b in mlp.biases]
    ref = omlp.mlp_forward(x.astype(np.float64), ws, bs, np.float64)
    assert np.max(np.abs(y - ref)) <= 2e-5 * np.abs(ref).max()
    for a, b in [(0, 1), (17, 300), (5000, 10000)]:
        part = fused.fused_forward(mlp, xt[a:b].clone()).cpu().numpy()
        assert np.array_equal(part, y[a:b])
    with pytest.raises(DimensionError):
        fused.fused_forward(mlp, xt[0])                          # 1-D batch
    with pytest.raises(DimensionError):
        fused.fused_forward(mlp, xt[:, :31])                     # wrong width
    with pytest.raises(DimensionError):
        fused.fused_forward(mlp, xt[:0])                         # empty batch


def test_residual_offset_matches_oracle(c1):
    sc, nets, osc = c1
    rng = np.random.default_rng(11)
    xs = rng.uniform(-1, 1, (3000, 3)).astype(np.float32)
    nets.set_pose(sc.poses[0])
    got = residual_offset(nets, torch.from_numpy(xs).to(DEV)).cpu().numpy()
    ref = opipe._field(osc, xs, osettings(sc.cfg), np.float64)["x_res"]
    scale = np.abs(ref).max()
    assert scale > 1e-3
    assert np.max(np.abs(got - ref)) <= 1e-5 * max(scale, 1.0)
    off = residual_offset(nets, torch.from_numpy(xs).to(DEV), stage=False).cpu().numpy()
    assert np.array_equal(off, np.zeros_like(off))              # stage disabled: exactly 0


def test_stratified_sample_bitexact(c1):
    sc, nets, osc = c1
    r, n = 64 * 64, 64
    pix = torch.arange(r, dtype=torch.int32, device=DEV)
    st = RenderSettings(n_samples=n, jitter=True, seed=99)
    x, delta, count = stratified_sample(nets, sc.camera, pix, st)
    cc = ocam.camera_consts(sc.camera.intrinsics, sc.camera.world_to_camera)
    o, d = ocam.rays_f32(cc, np.arange(r), 64)
    t0, t1, hit = ocam.slab_f32(o, d, osc["obox_min"], osc["obox_max"])
    t, dl, cnt = ocam.stratified_f32(t0, t1, hit, np.arange(r), n, True, 99)
    xo = ocam.positions_f32(o, d, t)
    assert x.shape == (r, n, 3) and delta.shape == (r, n)
    assert np.array_equal(count.cpu().numpy(), cnt)
    assert np.array_equal(x.cpu().numpy()[hit], xo[hit])
    assert np.array_equal(delta.cpu().numpy()[hit], dl[hit])
    assert hit.mean() > 0.25
