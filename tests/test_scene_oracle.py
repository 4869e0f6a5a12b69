"""Config 5 (multi-subject scene) definition, CPU: placement is disjoint and the
depth-ordered merge of per-subject composites equals one composite over the depth-sorted
union of all subjects' samples (the factorisation csrc/scene_merge.cu relies on)."""

import numpy as np

from oracle import adapter
from oracle import camera as ocam
from oracle import scene as oscene
from paper_2306_16541_b200 import scene as psc
from paper_2306_16541_b200.skeleton import motion_basis


def small_multi(n_subjects=3, width=20, n_samples=10, seed=0):
    cfg = psc.config("c5", width=width, height=width, n_samples=n_samples, half=False, occupancy=False,
                     hash=psc.HashGridConfig(log2_T=14, max_res=128), table_scale=0.5, bias_scale=0.5,
                     seed=seed, radius=7.0)
    return psc.make_multi_scene(cfg, n_subjects=n_subjects)


def oracle_inputs(ms):
    scenes, ccs, sts = [], [], []
    for s, sub in enumerate(ms.subjects):
        g_r, g_t = motion_basis(sub.skeleton, sub.poses[0])
        scenes.append(adapter.scene_arrays(sub, 0, g=(g_r.astype(np.float32), g_t.astype(np.float32))))
        cam = ms.subject_camera(s)
        ccs.append(ocam.camera_consts(cam.intrinsics, cam.world_to_camera))
        sts.append(adapter.settings(sub.cfg, seed=sub.jitter_seed))
    return scenes, ccs, sts


def test_placement_is_disjoint_and_seeded():
    a, b = small_multi(4), small_multi(4)
    assert np.array_equal(a.offsets, b.offsets)
    o = a.offsets
    for i in range(4):
        for j in range(i):
            assert max(abs(o[i, 0] - o[j, 0]), abs(o[i, 2] - o[j, 2])) >= 2.0
    assert np.all(np.abs(o[:, [0, 2]]) <= 2.0) and np.all(o[:, 1] == 0)
    # every subject has its own seeded parameters
    assert not np.array_equal(a.subjects[0].table, a.subjects[1].table)


def test_subject_camera_preserves_depths():
    ms = small_multi(2)
    cam, sub = ms.camera, ms.subject_camera(1)
    assert np.allclose(sub.center, cam.center - ms.offsets[1])
    assert np.allclose(sub.rotation, cam.rotation)


def test_depth_ordered_merge_equals_union_composite():
    ms = small_multi(3)
    scenes, ccs, sts = oracle_inputs(ms)
    pix = np.arange(ms.camera.width * ms.camera.height)
    bg = np.asarray(ms.cfg.background, np.float32)
    res = oscene.render_scene_rays(scenes, ccs, pix, ms.camera.width, sts, bg)
    hits = res["hit"].sum(0)
    assert (hits >= 2).sum() > 0, "need rays crossing two subjects to test the ordering"
    assert (hits == 0).sum() > 0
    rgb_u, alpha_u = oscene.union_composite(res["renders"], bg)
    assert np.max(np.abs(res["rgb"] - rgb_u)) < 1e-5
    assert np.max(np.abs(res["alpha"] - alpha_u)) < 1e-5
    # rays that miss every box see the background exactly
    miss = hits == 0
    assert np.array_equal(res["rgb"][miss], np.broadcast_to(bg, (miss.sum(), 3)))
    assert np.all(res["alpha"][miss] == 0)


def test_single_subject_merge_is_the_plain_render():
    ms = small_multi(1)
    scenes, ccs, sts = oracle_inputs(ms)
    pix = np.arange(ms.camera.width * ms.camera.height)
    bg = np.asarray(ms.cfg.background, np.float32)
    res = oscene.render_scene_rays(scenes, ccs, pix, ms.camera.width, sts, bg)
    from oracle import pipeline as opipe
    plain = opipe.render_rays(dict(scenes[0], bg=bg), ccs[0], pix, ms.camera.width, sts[0])
    assert np.max(np.abs(res["rgb"] - plain["rgb"])) < 1e-6
    assert np.max(np.abs(res["alpha"] - plain["alpha"])) < 1e-7


def test_ellipsoid_occupancy_bit_layout():
    """The seeded-ellipsoid skip grid (bench occupancy_variants) uses the occ_test layout:
    a point's cell bit is set iff the cell centre is inside the ellipsoid."""
    bmin, bmax = (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)
    bits = psc.ellipsoid_occupancy(bmin, bmax, seed=11)
    assert bits.dtype == np.int32 and bits.shape == (1024,)
    assert np.array_equal(bits, psc.ellipsoid_occupancy(bmin, bmax, seed=11))
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (4000, 3)).astype(np.float32)
    cell = ocam.occ_cell(x, bmin, ocam.occ_scale(bmin, bmax))
    got = ocam.occ_test(bits.view(np.uint32), cell)
    c = np.stack([cell // 1024, (cell // 32) % 32, cell % 32], -1)
    centre = -1.0 + (c + 0.5) * (2.0 / 32)
    r = np.linalg.norm(centre / np.array([0.8, 1.0, 0.6]), axis=-1)
    assert np.all(got[r < 0.85]) and not np.any(got[r > 1.15])   # seeded axis factors within +-10 %
    assert 0.15 < got.mean() < 0.35
