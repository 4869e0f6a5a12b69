"""Edge cases and full-size properties of the render path (SPEC S:410-446 examples)."""

import numpy as np
import pytest
import torch

from oracle import camera as ocam
from oracle import pipeline as opipe
from oracle.adapter import settings as osettings
from paper_2306_16541_b200.camera import orbit_camera
from paper_2306_16541_b200.model import FreeviewModel
from paper_2306_16541_b200.render import RenderSettings, Renderer

from helpers import make, oracle_scene

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def c2full():
    # table ~U(+-0.05): 500x the BASELINE init so the hash features matter, yet smooth enough
    # that the fp16 residual MLP's ~1e-4 x_final round-off stays below the 1e-3 render bar
    # (a +-0.5 random table amplifies it ~500x through the finest levels).
    sc = make("c2", table_scale=0.05, bias_scale=0.05, background=(0.1, 0.3, 0.8))
    return sc, FreeviewModel(sc)


def _render_pix(nets, cam, pix, st, rnd=None):
    rnd = rnd or Renderer()
    p = torch.as_tensor(np.asarray(pix, np.int32), device=DEV)
    cnt = torch.empty(len(pix), dtype=torch.int32, device=DEV)
    rgb, alpha = rnd.render_pixels(nets, cam, p, st, counts=cnt)
    torch.cuda.synchronize()
    return rgb.cpu().numpy(), alpha.cpu().numpy(), cnt.cpu().numpy()


def test_empty_ray_batch(c2full):
    sc, nets = c2full
    rgb, alpha, cnt = _render_pix(nets, sc.camera, [], RenderSettings.from_config(sc.cfg))
    assert rgb.shape == (0, 3) and alpha.shape == (0,)


def test_box_behind_camera_gives_background(c2full):
    """scene box behind the camera -> background, alpha 0, zero samples."""
    sc, nets = c2full
    cam = orbit_camera((0.0, 0.0, 6.0), 180.0, 0.0, 3.0, 45.0, 64, 64)   # at z=3 facing +z: box behind
    st = RenderSettings.from_config(sc.cfg, seed=1)
    rgb, alpha, cnt = _render_pix(nets, cam, np.arange(64 * 64), st)
    assert np.all(cnt == 0)
    assert np.all(alpha == 0.0)
    assert np.allclose(rgb, np.asarray(st.background, np.float32)[None, :], atol=0)


def test_camera_inside_box_and_single_sample(c2full):
    sc, nets = c2full
    osc = oracle_scene(sc, nets=nets)
    for cam, n in ((orbit_camera((0.0, 0.0, 0.0), 20.0, 10.0, 0.5, 60.0, 32, 32), 48),
                   (sc.camera, 1)):
        cfg = sc.cfg
        st = RenderSettings(n_samples=n, jitter=True, seed=9, background=cfg.background)
        pix = np.arange(32 * 32) if cam.width == 32 else np.arange(0, 512 * 512, 256)
        rgb, alpha, cnt = _render_pix(nets, cam, pix, st)
        cc = ocam.camera_consts(cam.intrinsics, cam.world_to_camera)
        ref = opipe.render_rays(osc, cc, pix, cam.width, osettings(cfg, n_samples=n, seed=9), np.float32)
        assert np.array_equal(cnt, ref["count"])
        assert np.abs(rgb - ref["rgb"]).max() < 1e-3 and np.abs(alpha - ref["alpha"]).max() < 1e-3


def test_untiled_resolution_row_major_path(c2full):
    sc, nets = c2full
    cam = orbit_camera((0.0, 0.0, 0.0), 0.0, 0.0, 3.0, 45.0, 37, 23)   # not a multiple of 8x4
    st = RenderSettings.from_config(sc.cfg, seed=4, occupancy=False)
    img, alpha = Renderer().render_image(nets, cam, None, st)
    torch.cuda.synchronize()
    osc = oracle_scene(sc, nets=nets)
    cc = ocam.camera_consts(cam.intrinsics, cam.world_to_camera)
    ref = opipe.render_rays(osc, cc, np.arange(37 * 23), 37, osettings(sc.cfg, seed=4), np.float32)
    assert np.abs(img.cpu().numpy().reshape(-1, 3) - ref["rgb"]).max() < 1e-3
    assert np.abs(alpha.cpu().numpy().reshape(-1) - ref["alpha"]).max() < 1e-3


def test_empty_occupancy_skips_everything(c2full):
    sc, nets = c2full
    st = RenderSettings.from_config(sc.cfg, seed=2, occupancy=False)
    rnd = Renderer()
    pix = torch.arange(4096, dtype=torch.int32, device=DEV)
    occ = torch.zeros(1024, dtype=torch.int32, device=DEV)
    rgb, alpha = rnd.render_pixels(nets, sc.camera, pix, st, occ=occ)
    torch.cuda.synchronize()
    assert torch.all(alpha == 0) and torch.allclose(rgb, torch.tensor(st.background, device=DEV).expand(4096, 3))


def test_full_frame_deterministic_and_crop_invariant(c2full):
    """fixed seed -> bitwise-identical renders; any crop equals the per-ray result."""
    sc, nets = c2full
    st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
    rnd = Renderer()
    a, _ = rnd.render_image(nets, sc.camera, None, st)
    a = a.clone()
    b, _ = rnd.render_image(nets, sc.camera, None, st)
    assert torch.equal(a, b)
    occ = rnd.occ.clone()
    yy, xx = np.meshgrid(np.arange(200, 208), np.arange(300, 308), indexing="ij")
    crop = (yy * 512 + xx).reshape(-1)
    p = torch.as_tensor(crop.astype(np.int32), device=DEV)
    rgb, _ = rnd.render_pixels(nets, sc.camera, p, st, occ=occ)
    assert torch.equal(rgb, a.reshape(-1, 3)[torch.as_tensor(crop, device=DEV)])


def test_full_size_c2_spot_parity(c2full):
    """Full 512x512 frame on the GPU; random 16x16 crops checked against the oracle per ray."""
    sc, nets = c2full
    st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
    rnd = Renderer()
    img, alpha = rnd.render_image(nets, sc.camera, None, st)
    torch.cuda.synchronize()
    img, alpha = img.cpu().numpy().reshape(-1, 3), alpha.cpu().numpy().reshape(-1)
    occ = rnd.occ.cpu().numpy().view(np.uint32)
    osc = oracle_scene(sc, nets=nets)
    cc = ocam.camera_consts(sc.camera.intrinsics, sc.camera.world_to_camera)
    rng = np.random.default_rng(0)
    for _ in range(2):
        y0, x0 = rng.integers(0, 512 - 16, 2)
        yy, xx = np.meshgrid(np.arange(y0, y0 + 16), np.arange(x0, x0 + 16), indexing="ij")
        pix = (yy * 512 + xx).reshape(-1)
        ref = opipe.render_rays(osc, cc, pix, 512, osettings(sc.cfg, seed=sc.jitter_seed, occupancy=occ), np.float32)
        assert np.abs(img[pix] - ref["rgb"]).max() < 1e-3
        assert np.abs(alpha[pix] - ref["alpha"]).max() < 1e-3


def test_launch_chunking_is_bitwise_invisible(c2full, monkeypatch):
    """Ray sets above Renderer.MAX_SAMPLES_PER_LAUNCH sample slots go in chunks of whole
    32-ray blocks (the C ABI refuses >= 2^31 slots, int32 sample ids): the full 512^2 frame
    (image-sized by-pixel outputs) and a per-ray batch with counts (sliced outputs) are
    bitwise the single-launch result in chunks of 1184 rays (37 ray blocks)."""
    sc, nets = c2full
    st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
    rnd = Renderer()
    a_rgb, a_alpha = rnd.render_image(nets, sc.camera, None, st)
    a_rgb, a_alpha = a_rgb.clone(), a_alpha.clone()
    rng = np.random.default_rng(4)
    pix = rng.choice(512 * 512, 3000, replace=False).astype(np.int32)
    b_rgb, b_alpha, b_cnt = _render_pix(nets, sc.camera, pix, st, rnd)
    monkeypatch.setattr(Renderer, "MAX_SAMPLES_PER_LAUNCH", 32 * 128 * 37 // 32 * 32 + 100)
    rnd2 = Renderer()
    c_rgb, c_alpha = rnd2.render_image(nets, sc.camera, None, st)
    torch.cuda.synchronize()
    assert torch.equal(c_rgb, a_rgb) and torch.equal(c_alpha, a_alpha)
    d_rgb, d_alpha, d_cnt = _render_pix(nets, sc.camera, pix, st, rnd2)
    assert np.array_equal(d_rgb, b_rgb) and np.array_equal(d_alpha, b_alpha) and np.array_equal(d_cnt, b_cnt)


def test_warp_specialised_radiance_repeatable(c2full):
    """k_radiance_ws hands tiles between 6 gather warpgroups and one MLP warpgroup through
    mbarriers: 20 back-to-back renders of the full 512^2 frame (33.5 M slots, ~1570 tiles per
    SM) are bitwise identical -- a missed handshake would show as a differing tile."""
    sc, nets = c2full
    st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
    rnd = Renderer()
    ref, ref_a = rnd.render_image(nets, sc.camera, None, st)
    ref, ref_a = ref.clone(), ref_a.clone()
    for _ in range(20):
        img, alpha = rnd.render_image(nets, sc.camera, None, st)
        assert torch.equal(img, ref) and torch.equal(alpha, ref_a)
