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


def test_sample_bone_channels_matches_oracle():
    """Reference signature sample_bone_channels(vol, pts, box_min, box_max) on a model's own
    W^c: bit-exact with the oracle's float32 lerp form, incl. points outside the padded grid."""
    sc = make("c1", width=16, height=16)
    nets = FreeviewModel(sc)
    osc = oracle_scene(sc, nets=nets)
    k = nets.n_bones
    rng = np.random.default_rng(3)
    lo, hi = np.asarray(osc["wbox_min"]), np.asarray(osc["wbox_max"])
    pts = rng.uniform(lo - 0.15, hi + 0.15, (k, 4000, 3)).astype(np.float32)
    got = autodiff.sample_bone_channels(nets.vol, torch.from_numpy(pts).to(DEV), lo, hi).cpu().numpy()
    ref = owarp.sample_bone_channels(osc["vol"][:k], pts, osc["wbox_min"], osc["wbox_max"], np.float32)
    assert got.shape == (k, 4000)
    assert np.array_equal(got, ref)
    assert (ref == 0).mean() > 0.02 and (ref > 0).mean() > 0.5
    with pytest.raises(DimensionError):
        autodiff.sample_bone_channels(nets.vol, torch.zeros((k + 2, 5, 3), device=DEV), lo, hi)
    with pytest.raises(DimensionError):
        autodiff.sample_bone_channels(nets.vol, torch.zeros((k, 5, 2), device=DEV), lo, hi)


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
    """Reference semantics (ad:815-837): input = attenuations 1 - opacity, T[:, i+1] =
    T[:, i] * atten[:, i] -- bit-exact with numpy's float32 cumprod, exact zeros included."""
    rng = np.random.default_rng(7)
    at = rng.uniform(0.7, 1.0, (700, 96)).astype(np.float32)
    at[::7, 40:] = 0.0                                          # fully opaque samples
    got = autodiff.transmittance(torch.from_numpy(at).to(DEV)).cpu().numpy()
    ref = np.concatenate([np.ones((700, 1), np.float32), np.cumprod(at, axis=1, dtype=np.float32)], 1)
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
    mlp = fused.FusedMlp.random(32, 4, depth=2, seed=1)
    rng = np.random.default_rng(2)
    x = rng.standard_normal((10000, 32)).astype(np.float32)
    xt = torch.from_numpy(x).to(DEV)
    y = fused.fused_forward(mlp, xt).cpu().numpy()
    ws = [w.cpu().numpy().astype(np.float64) for w in mlp.weights]
    bs = [b.cpu().numpy().astype(np.float64) for b in mlp.biases]
    ref = omlp.mlp_forward(x.astype(np.float64), ws, bs, np.float64)
    assert np.max(np.abs(y - ref)) <= 2e-5 * np.abs(ref).max()
    assert np.max(np.abs(fused.naive_forward(mlp, xt).cpu().numpy() - ref)) <= 2e-5 * np.abs(ref).max()
    for a, b in [(0, 1), (17, 300), (5000, 10000), (127, 129)]:
        part = fused.fused_forward(mlp, xt[a:b].clone()).cpu().numpy()
        assert np.array_equal(part, y[a:b])
    with pytest.raises(DimensionError):
        fused.fused_forward(mlp, xt[0])                          # 1-D batch
    with pytest.raises(DimensionError):
        fused.fused_forward(mlp, xt[:, :31])                     # wrong width
    with pytest.raises(DimensionError):
        fused.fused_forward(mlp, xt[:0])                         # empty batch
    with pytest.raises(DimensionError):                          # reference shape rules (fu:80-96)
        fused.FusedMlp([torch.zeros((32, 64), device=DEV)])
    with pytest.raises(DimensionError):
        fused.FusedMlp([torch.zeros((65, 64), device=DEV), torch.zeros((64, 4), device=DEV)])
    with pytest.raises(DimensionError):
        fused.FusedMlp([torch.zeros((32, 48), device=DEV), torch.zeros((48, 4), device=DEV)])


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


# ----------------------------------------------------------------- backwards vs golden vectors
# tests/golden/ref_primitives.npz: the reference's own ops and Tape gradients (make_golden.py)

GOLD = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "ref_primitives.npz"))


def _leaf(a):
    return torch.tensor(np.asarray(a, np.float32), device=DEV, requires_grad=True)


def _rel(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)


def test_sample_bone_channels_autograd_matches_reference_tape():
    """Forward and both gradients (d vol, d pts: fv_sample_bone_channels_bwd) against the
    reference's own values and Tape gradients (ad:728-808; golden sbc_*)."""
    vol, pts = _leaf(GOLD["sbc_vol"]), _leaf(GOLD["sbc_pts"])
    out = autodiff.sample_bone_channels(vol, pts, (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    assert _rel(out.detach().cpu().numpy(), GOLD["sbc_out"]) < 1e-6
    (out * torch.tensor(GOLD["sbc_up"], dtype=torch.float32, device=DEV)).sum().backward()
    assert _rel(vol.grad.cpu().numpy(), GOLD["sbc_dvol"]) < 1e-5
    assert _rel(pts.grad.cpu().numpy(), GOLD["sbc_dpts"]) < 1e-5


@pytest.mark.parametrize("tag,alpha", [("full", 6.0), ("win", 2.3)])
def test_posenc_autograd_matches_reference_tape(tag, alpha):
    p = _leaf(GOLD[f"pe_{tag}_p"])
    out = autodiff.posenc(p, 6, alpha)
    assert np.abs(out.detach().cpu().numpy() - GOLD[f"pe_{tag}_out_f32"]).max() < 2e-6
    (out * torch.tensor(GOLD[f"pe_{tag}_up"], dtype=torch.float32, device=DEV)).sum().backward()
    assert _rel(p.grad.cpu().numpy(), GOLD[f"pe_{tag}_dp"]) < 1e-5
    q = _leaf(GOLD[f"pe_{tag}_p"])                              # include_raw=False: raw columns dropped
    out2 = autodiff.posenc(q, 6, alpha, include_raw=False)
    assert out2.shape == (20, 36) and autodiff.posenc_dim(6, False) == 36
    (out2 * torch.tensor(GOLD[f"pe_{tag}_up"][:, 3:], dtype=torch.float32, device=DEV)).sum().backward()
    ref = GOLD[f"pe_{tag}_dp"] - GOLD[f"pe_{tag}_up"][:, :3]     # minus the raw-column pass-through
    assert _rel(q.grad.cpu().numpy(), ref) < 1e-5


def test_softmax0_autograd_matches_reference_tape():
    x = _leaf(GOLD["sm_x"])
    out = autodiff.softmax0(x)
    assert np.abs(out.detach().cpu().numpy() - GOLD["sm_out"]).max() < 1e-6
    (out * torch.tensor(GOLD["sm_up"], dtype=torch.float32, device=DEV)).sum().backward()
    assert _rel(x.grad.cpu().numpy(), GOLD["sm_dx"]) < 1e-5


def test_transmittance_autograd_is_the_division_free_reverse_scan():
    """ad:815-837 with an exact zero attenuation (golden tr_*): the reverse scan stays finite
    and equals the reference Tape gradient."""
    x = _leaf(GOLD["tr_x"])
    out = autodiff.transmittance(x)
    assert np.abs(out.detach().cpu().numpy() - GOLD["tr_out"]).max() < 1e-6
    (out * torch.tensor(GOLD["tr_up"], dtype=torch.float32, device=DEV)).sum().backward()
    g = x.grad.cpu().numpy()
    assert np.all(np.isfinite(g))
    assert _rel(g, GOLD["tr_dx"]) < 1e-5


def test_linear_chain_autograd_matches_reference_tape():
    """The reference's 32 -> 64 -> 64 -> 4 MLP built from ``linear`` (ad:403-425) with its
    Tape gradients (golden mlp_*): forward within fp32 rounding of naive_forward, dx / dW /
    db within 1e-5 relative."""
    x = _leaf(GOLD["mlp_x"])
    ws = [_leaf(GOLD[f"mlp_w{i}"]) for i in range(3)]
    bs = [_leaf(GOLD[f"mlp_b{i}"]) for i in range(3)]
    h = autodiff.linear(x, ws[0], bs[0], "relu")
    h = autodiff.linear(h, ws[1], bs[1], "relu")
    y = autodiff.linear(h, ws[2], bs[2], "none")
    assert _rel(y.detach().cpu().numpy(), GOLD["mlp_out"]) < 2e-5
    (y * torch.tensor(GOLD["mlp_up"], dtype=torch.float32, device=DEV)).sum().backward()
    assert _rel(x.grad.cpu().numpy(), GOLD["mlp_dx"]) < 1e-5
    for i in range(3):
        assert _rel(ws[i].grad.cpu().numpy(), GOLD[f"mlp_dw{i}"]) < 1e-5
        assert _rel(bs[i].grad.cpu().numpy(), GOLD[f"mlp_db{i}"]) < 1e-5
    with pytest.raises(DimensionError):
        autodiff.linear(x, ws[1], bs[1])


def test_fused_forward_matches_reference_naive_forward_golden():
    """FusedMlp.random(32, 4, depth=2, seed=3) draws the reference's exact weights
    (fu:120-130) and fused_forward equals the reference's naive_forward (golden mlp_out)."""
    mlp = fused.FusedMlp.random(32, 4, depth=2, seed=3)
    for i in range(3):
        assert np.array_equal(mlp.weights[i].cpu().numpy(), GOLD[f"mlp_w{i}"])
        assert np.array_equal(mlp.biases[i].cpu().numpy(), GOLD[f"mlp_b{i}"])
    y = fused.fused_forward(mlp, torch.tensor(GOLD["mlp_x"], device=DEV)).cpu().numpy()
    assert _rel(y, GOLD["mlp_out"]) < 2e-5


def test_adam_step_matches_reference_and_refuses_nonfinite():
    """adam_step(params, grads, state, lr) (ad:893-912): three steps on two blocks with their
    own states and rates equal the reference's (golden adam_*); a non-finite gradient raises
    TrainingError naming the block and leaves parameters, moments and the step count alone."""
    from paper_2306_16541_b200.errors import TrainingError
    p0 = torch.tensor(GOLD["adam_p0"], dtype=torch.float32, device=DEV)
    p1 = torch.tensor(GOLD["adam_p1"], dtype=torch.float32, device=DEV)
    s0, s1 = autodiff.AdamState([p0], beta1=0.9, beta2=0.99), autodiff.AdamState([p1], beta1=0.9, beta2=0.99)
    for i in range(3):
        autodiff.adam_step([p0], [torch.tensor(GOLD[f"adam_g{i}_0"], dtype=torch.float32, device=DEV)], s0, lr=5e-4)
        autodiff.adam_step([p1], [torch.tensor(GOLD[f"adam_g{i}_1"], dtype=torch.float32, device=DEV)], s1, lr=5e-5)
    assert np.abs(p0.cpu().numpy() - GOLD["adam_out0"]).max() < 1e-6
    assert np.abs(p1.cpu().numpy() - GOLD["adam_out1"]).max() < 1e-6
    assert s0.t == 3
    before = (p0.clone(), s0.m[0].clone(), s0.v[0].clone())
    bad = torch.tensor(GOLD["adam_g0_0"], dtype=torch.float32, device=DEV)
    bad[3] = float("nan")
    with pytest.raises(TrainingError, match="table"):
        autodiff.adam_step([p0], [bad], s0, lr=5e-4, names=["table"])
    assert s0.t == 3 and torch.equal(p0, before[0]) and torch.equal(s0.m[0], before[1])
    with pytest.raises(DimensionError):
        autodiff.adam_step([p0], [bad[:3]], s0, lr=5e-4)


@pytest.mark.parametrize("n_in,n_out,depth,batch", [(1, 1, 1, 1), (64, 64, 4, 65536), (3, 4, 7, 1001),
                                                    (39, 3, 2, 129), (32, 4, 2, 127)])
def test_fused_forward_shapes(n_in, n_out, depth, batch):
    """fv_fused_mlp_fwd over the FusedMlp shape range (in/out 1..64, 2..8 layers, ragged
    batches around the 128-row chunk): equal to the layer-by-layer naive_forward to fp32
    rounding and bitwise chunk-invariant."""
    mlp = fused.FusedMlp.random(n_in, n_out, depth=depth, seed=n_in + depth)
    x = torch.randn((batch, n_in), device=DEV)
    y = fused.fused_forward(mlp, x)
    ref = fused.naive_forward(mlp, x)
    assert y.shape == (batch, n_out)
    scale = float(ref.abs().max()) + 1e-6
    assert float((y - ref).abs().max()) <= 2e-5 * scale
    if batch > 3:
        part = fused.fused_forward(mlp, x[1:batch - 1].clone())
        assert torch.equal(part, y[1:batch - 1])
