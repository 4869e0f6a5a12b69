"""Render service (SPEC ``serve``): request validation is total (malformed requests
only ever get 400/404, never a render or a crash), PNG encoding, /meta; on the GPU:
identical requests give byte-identical PNGs, opposite viewpoints differ, a real HTTP round
trip, and the service leaves the model parameters untouched."""

import json
import threading
import urllib.error
import urllib.request
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2306_16541_b200 import service as svc_mod
from paper_2306_16541_b200.camera import orbit_camera
from paper_2306_16541_b200.render import RenderSettings


def _stub_service():
    """A RenderService over a stand-in model whose render_png records calls (no GPU)."""
    cam = orbit_camera((0, 0, 0), 0, 0, 3.0, 45.0, 64, 64)
    scene = SimpleNamespace(poses=[object()] * 5, camera=cam, cfg=SimpleNamespace(radius=3.0, fov_deg=45.0))
    s = svc_mod.RenderService(SimpleNamespace(scene=scene), RenderSettings())
    s.calls = []
    s.render_png = lambda frame, cam, canon: (s.calls.append(canon), b"PNG")[1]
    return s


def test_png_roundtrip():
    rng = np.random.default_rng(0)
    img = rng.uniform(0, 1, (17, 23, 3))
    data = svc_mod.encode_png(img)
    back = svc_mod.decode_png_rgb(data)
    assert back.shape == (17, 23, 3)
    assert np.array_equal(back, np.clip(np.rint(img * 255), 0, 255).astype(np.uint8))


def test_meta_and_valid_requests_reach_the_renderer():
    s = _stub_service()
    code, ctype, body = s.handle("GET", "/meta")
    meta = json.loads(body)
    assert code == 200 and ctype == "application/json" and meta["frames"] == 5
    assert meta["limits"]["w"] == [16, 1024]
    code, ctype, body = s.handle("GET", "/render?frame=2&yaw=30&pitch=-10&radius=2.5&fov=40&w=32&h=48")
    assert (code, ctype, body) == (200, "image/png", b"PNG")
    assert s.calls[-1] == {"frame": 2, "yaw": 30.0, "pitch": -10.0, "radius": 2.5, "fov": 40.0, "w": 32, "h": 48}
    e = orbit_camera((0, 0, 0), 10, 5, 3, 45, 64, 64).world_to_camera
    req = {"frame": 1, "intrinsics": [[50, 0, 32], [0, 50, 32], [0, 0, 1]], "world_to_camera": e.tolist(), "w": 64, "h": 64}
    assert s.handle("POST", "/render", json.dumps(req).encode())[0] == 200


@pytest.mark.parametrize("query", [
    "frame=5", "frame=-1", "frame=x", "frame=1.5", "pitch=90", "pitch=-89.5", "radius=0", "radius=-1",
    "w=15", "h=1025", "w=abc", "fov=0", "fov=180", "yaw=nan", "yaw=inf", "radius=", "w=64.5"])
def test_invalid_orbit_requests_get_400(query):
    s = _stub_service()
    code, ctype, body = s.handle("GET", "/render?" + query)
    assert code == 400 and ctype == "application/json" and "error" in json.loads(body)
    assert not s.calls


def test_validation_is_total_under_fuzzing():
    """10^4 malformed query strings -> only 400/404 (or a render for the rare valid one)."""
    s = _stub_service()
    rng = np.random.default_rng(1)
    keys = ["frame", "yaw", "pitch", "radius", "fov", "w", "h", "junk", ""]
    vals = ["", "0", "-1", "1e309", "nan", "-inf", "abc", "3.5", "1024", "16", "99999", "%00", "[]", "{}", "0x10"]
    paths = ["/render", "/meta", "/x", "/render/", "//render", "/RENDER"]
    for _ in range(10000):
        q = "&".join(f"{rng.choice(keys)}={rng.choice(vals)}" for _ in range(rng.integers(0, 6)))
        method = "GET" if rng.random() < 0.9 else "POST"
        body = bytes(rng.integers(0, 256, rng.integers(0, 40), dtype=np.uint8)) if method == "POST" else b""
        code, _, _ = s.handle(method, f"{rng.choice(paths)}?{q}", body)
        assert code in (200, 400, 404)


def test_bad_explicit_camera_bodies_get_400():
    s = _stub_service()
    bad = [b"", b"not json", b"[1, 2]", json.dumps({"intrinsics": [[1, 0], [0, 1]]}).encode(),
           json.dumps({"intrinsics": np.eye(3).tolist(), "world_to_camera": (2 * np.eye(4)).tolist(), "w": 32,
                       "h": 32}).encode(),
           json.dumps({"intrinsics": (-np.eye(3)).tolist(), "world_to_camera": np.eye(4).tolist(), "w": 32,
                       "h": 32}).encode(),
           json.dumps({"intrinsics": np.eye(3).tolist(), "world_to_camera": np.eye(4).tolist(), "w": 8, "h": 32}).encode()]
    for b in bad:
        assert s.handle("POST", "/render", b)[0] == 400
    assert s.handle("GET", "/nowhere")[0] == 404
    assert s.handle("PUT", "/render")[0] == 400
    s.loading = True
    assert s.handle("GET", "/meta")[0] == 503


# ------------------------------------------------------------------------------ GPU

@pytest.fixture(scope="module")
def live():
    from helpers import make
    from paper_2306_16541_b200.model import FreeviewModel
    # a strongly textured field (large table values) so opposite viewpoints see different colours
    sc = make("c2", width=64, height=64, table_scale=5000.0, bias_scale=0.05, n_poses=3)
    nets = FreeviewModel(sc)
    return nets, svc_mod.RenderService(nets, RenderSettings.from_config(sc.cfg, seed=0))


@pytest.mark.gpu
def test_render_is_deterministic_and_view_dependent(live):
    nets, s = live
    before = nets.flat.clone()
    a = s.handle("GET", "/render?frame=1&yaw=0&pitch=0&w=64&h=64")
    b = s.handle("GET", "/render?frame=1&yaw=0&pitch=0&w=64&h=64")
    c = s.handle("GET", "/render?frame=1&yaw=180&pitch=0&w=64&h=64")
    assert a[0] == b[0] == c[0] == 200 and a[1] == "image/png"
    assert a[2] == b[2]                                               # byte-identical bodies
    ia, ic = svc_mod.decode_png_rgb(a[2]), svc_mod.decode_png_rgb(c[2])
    assert ia.shape == (64, 64, 3)
    assert np.abs(ia.astype(float) - ic.astype(float)).mean() / 255 > 0.01   # S:584 example
    assert bool((nets.flat == before).all())                          # read-only model


@pytest.mark.gpu
def test_http_round_trip(live):
    _, s = live
    httpd = svc_mod.serve(s, 0)
    t = threading.Thread(target=httpd.serve_forever, daemon=True)
    t.start()
    try:
        base = f"http://127.0.0.1:{httpd.server_address[1]}"
        meta = json.loads(urllib.request.urlopen(base + "/meta", timeout=60).read())
        assert meta["frames"] == 3
        png = urllib.request.urlopen(base + "/render?frame=0&yaw=45&w=32&h=48", timeout=120).read()
        assert svc_mod.decode_png_rgb(png).shape == (48, 32, 3)
        with pytest.raises(urllib.error.HTTPError) as e:
            urllib.request.urlopen(base + "/render?pitch=95", timeout=60)
        assert e.value.code == 400 and "error" in json.loads(e.value.read())
    finally:
        httpd.shutdown()
        httpd.server_close()
