"""Frame delivery service (SPEC ``serve``, ``S:577-585``): plain HTTP with PNG
bodies in front of ``render_image``.

  GET  /meta                                          -> JSON {frames, default_camera, limits, model_id}
  GET  /render?frame=&yaw=&pitch=&radius=&fov=&w=&h=  -> PNG (orbit camera around the subject)
  POST /render  {"frame", "intrinsics" 3x3, "world_to_camera" 4x4 (or 3x4), "w", "h"} -> PNG
  malformed request -> 400 {"error": ...}; unknown path -> 404; while (re)loading -> 503

RenderRequest validation (``S:562-565``): frame in [0, frames), pitch in [-89, 89], radius > 0,
fov in (0, 180), w and h in [16, 1024].  Renders are deterministic for identical requests:
the jitter seed is a hash of the canonical request.  Render execution is serialised through
one lock (the SPEC's FIFO render queue, ``S:591``); model state is read-only after load
(``S:586``).  ``RenderService.handle`` is the transport-free core (what the tests drive);
``serve`` binds it to ``http.server``.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import math
import struct
import threading
import zlib
from http.server import BaseHTTPRequestHandler, ThreadingHTTPServer
from typing import Dict, Optional, Tuple
from urllib.parse import parse_qs, urlsplit

import numpy as np

from .camera import CameraModel, orbit_camera
from .model import FreeviewModel
from .render import RenderSettings, render_image

LIMITS = {"w": [16, 1024], "h": [16, 1024], "pitch": [-89.0, 89.0], "fov": [1.0, 179.0]}


class RequestError(ValueError):
    pass


def encode_png(rgb: np.ndarray) -> bytes:
    """(H, W, 3) float in [0, 1] -> 8-bit RGB PNG (zlib level 6, filter 0 per row)."""
    img = np.clip(np.rint(np.asarray(rgb, np.float64) * 255.0), 0, 255).astype(np.uint8)
    h, w = img.shape[:2]
    raw = b"".join(b"\x00" + img[y].tobytes() for y in range(h))

    def chunk(tag: bytes, data: bytes) -> bytes:
        return struct.pack(">I", len(data)) + tag + data + struct.pack(">I", zlib.crc32(tag + data) & 0xFFFFFFFF)

    return (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0))
            + chunk(b"IDAT", zlib.compress(raw, 6)) + chunk(b"IEND", b""))


def decode_png_rgb(data: bytes) -> np.ndarray:
    """Inverse of encode_png (8-bit RGB, filter 0 rows only) -> (H, W, 3) uint8."""
    if data[:8] != b"\x89PNG\r\n\x1a\n":
        raise ValueError("not a PNG")
    pos, idat = 8, b""
    w = h = 0
    while pos < len(data):
        n = struct.unpack(">I", data[pos:pos + 4])[0]
        tag, body = data[pos + 4:pos + 8], data[pos + 8:pos + 8 + n]
        if tag == b"IHDR":
            w, h = struct.unpack(">II", body[:8])
        elif tag == b"IDAT":
            idat += body
        pos += 12 + n
    raw = np.frombuffer(zlib.decompress(idat), np.uint8).reshape(h, 1 + 3 * w)
    if np.any(raw[:, 0] != 0):
        raise ValueError("unsupported PNG filter")
    return raw[:, 1:].reshape(h, w, 3)


def _num(q: Dict[str, str], key: str, default=None, kind=float):
    if key not in q:
        if default is None:
            raise RequestError(f"missing parameter '{key}'")
        return default
    try:
        v = kind(q[key])
    except (TypeError, ValueError):
        raise RequestError(f"parameter '{key}' is not a valid {kind.__name__}")
    if kind is float and not math.isfinite(v):
        raise RequestError(f"parameter '{key}' must be finite")
    return v


class RenderService:
    """Serves frames of a loaded FreeviewModel; ``poses`` index the frames."""

    def __init__(self, nets: FreeviewModel, settings: RenderSettings, model_id: str = "freeview-b200",
                 default_camera: Optional[dict] = None):
        self.nets = nets
        self.settings = settings
        self.model_id = model_id
        self.poses = list(nets.scene.poses)
        cam = nets.scene.camera
        self.default_camera = default_camera or {"yaw": 0.0, "pitch": 0.0, "radius": nets.scene.cfg.radius,
                                                 "fov": nets.scene.cfg.fov_deg, "w": cam.width, "h": cam.height}
        self.target = np.zeros(3)
        self._lock = threading.Lock()          # the FIFO render queue (one render at a time)
        self.loading = False

    # ------------------------------------------------------------------ request parsing
    def _frame(self, v) -> int:
        try:
            f = int(v)
        except (TypeError, ValueError):
            raise RequestError("parameter 'frame' is not an integer")
        if not 0 <= f < len(self.poses):
            raise RequestError(f"frame {f} outside [0, {len(self.poses)})")
        return f

    def _size(self, w: int, h: int) -> Tuple[int, int]:
        for k, v in (("w", w), ("h", h)):
            lo, hi = LIMITS[k]
            if not lo <= v <= hi:
                raise RequestError(f"{k} = {v} outside [{lo}, {hi}]")
        return w, h

    def parse_orbit(self, query: Dict[str, str]) -> Tuple[int, CameraModel, dict]:
        d = self.default_camera
        frame = self._frame(query.get("frame", "0"))
        yaw = _num(query, "yaw", d["yaw"])
        pitch = _num(query, "pitch", d["pitch"])
        radius = _num(query, "radius", d["radius"])
        fov = _num(query, "fov", d["fov"])
        w, h = self._size(_num(query, "w", d["w"], int), _num(query, "h", d["h"], int))
        if not LIMITS["pitch"][0] <= pitch <= LIMITS["pitch"][1]:
            raise RequestError(f"pitch = {pitch} outside [-89, 89]")
        if not radius > 0:
            raise RequestError("radius must be > 0")
        if not LIMITS["fov"][0] <= fov <= LIMITS["fov"][1]:
            raise RequestError(f"fov = {fov} outside [1, 179]")
        canon = {"frame": frame, "yaw": yaw, "pitch": pitch, "radius": radius, "fov": fov, "w": w, "h": h}
        return frame, orbit_camera(self.target, yaw, pitch, radius, fov, w, h), canon

    def parse_explicit(self, body: bytes) -> Tuple[int, CameraModel, dict]:
        try:
            req = json.loads(body.decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError):
            raise RequestError("body is not valid JSON")
        if not isinstance(req, dict):
            raise RequestError("body must be a JSON object")
        frame = self._frame(req.get("frame", 0))
        try:
            k = np.asarray(req["intrinsics"], np.float64)
            e = np.asarray(req["world_to_camera"], np.float64)
            w, h = int(req["w"]), int(req["h"])
        except (KeyError, TypeError, ValueError):
            raise RequestError("need intrinsics (3x3), world_to_camera (4x4 or 3x4), w, h")
        if k.shape != (3, 3) or e.shape not in ((4, 4), (3, 4)) or not (np.all(np.isfinite(k)) and np.all(np.isfinite(e))):
            raise RequestError("intrinsics must be 3x3 and world_to_camera 4x4 or 3x4, finite")
        if e.shape == (3, 4):
            e = np.vstack([e, [0.0, 0.0, 0.0, 1.0]])
        r = e[:3, :3]
        if abs(np.linalg.det(r) - 1.0) > 1e-3 or np.max(np.abs(r @ r.T - np.eye(3))) > 1e-3:
            raise RequestError("world_to_camera rotation is not orthonormal")
        if k[0, 0] <= 0 or k[1, 1] <= 0:
            raise RequestError("focal lengths must be positive")
        w, h = self._size(w, h)
        canon = {"frame": frame, "K": k.round(9).tolist(), "E": e.round(9).tolist(), "w": w, "h": h}
        return frame, CameraModel(k, e, w, h), canon

    # ------------------------------------------------------------------ rendering
    def render_png(self, frame: int, cam: CameraModel, canon: dict) -> bytes:
        seed = int.from_bytes(hashlib.sha256(json.dumps(canon, sort_keys=True).encode()).digest()[:4], "little")
        st = dataclasses.replace(self.settings, seed=seed)
        with self._lock:
            img, _ = render_image(self.nets, cam, self.poses[frame], st)
            rgb = img.cpu().numpy()
        return encode_png(rgb)

    def meta(self) -> dict:
        return {"frames": len(self.poses), "default_camera": self.default_camera, "limits": LIMITS,
                "model_id": self.model_id}

    def handle(self, method: str, path: str, body: bytes = b"") -> Tuple[int, str, bytes]:
        """(status, content type, body) for one request; never raises."""
        def err(code, msg):
            return code, "application/json", json.dumps({"error": msg}).encode()
        try:
            if self.loading:
                return err(503, "checkpoint is loading")
            u = urlsplit(path)
            query = {k: v[-1] for k, v in parse_qs(u.query, keep_blank_values=True).items()}
            if u.path == "/meta" and method == "GET":
                return 200, "application/json", json.dumps(self.meta()).encode()
            if u.path == "/render" and method == "GET":
                return 200, "image/png", self.render_png(*self.parse_orbit(query))
            if u.path == "/render" and method == "POST":
                return 200, "image/png", self.render_png(*self.parse_explicit(body))
            if u.path in ("/meta", "/render"):
                return err(400, f"method {method} not allowed on {u.path}")
            return err(404, f"unknown path {u.path}")
        except RequestError as e:
            return err(400, str(e))
        except Exception as e:   # never crash the service on a request
            return err(500, f"{type(e).__name__}: {e}")


def serve(service: RenderService, port: int = 8080, host: str = "127.0.0.1") -> ThreadingHTTPServer:
    """Bind the service to an HTTP server (call .serve_forever() on the result)."""

    class Handler(BaseHTTPRequestHandler):
        def _reply(self, method):
            n = int(self.headers.get("Content-Length") or 0)
            body = self.rfile.read(n) if n > 0 else b""
            code, ctype, out = service.handle(method, self.path, body)
            self.send_response(code)
            self.send_header("Content-Type", ctype)
            self.send_header("Content-Length", str(len(out)))
            self.end_headers()
            self.wfile.write(out)

        def do_GET(self):
            self._reply("GET")

        def do_POST(self):
            self._reply("POST")

        def log_message(self, *args):
            pass

    return ThreadingHTTPServer((host, port), Handler)


def main(argv=None) -> int:
    """``python -m paper_2306_16541_b200.service [--config c2] [--port 8080] [--checkpoint DIR]``:
    serve a seeded model of the config (optionally with a save_checkpoint directory's
    parameters) until interrupted."""
    import argparse
    from . import scene as psc
    from .train import load_params
    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--port", type=int, default=8080)
    ap.add_argument("--host", default="127.0.0.1")
    ap.add_argument("--checkpoint", default=None)
    args = ap.parse_args(argv)
    sc = psc.make_scene(psc.config(args.config))
    nets = FreeviewModel(sc)
    if args.checkpoint:
        load_params(args.checkpoint, nets)
    svc = RenderService(nets, RenderSettings.from_config(sc.cfg, seed=0))
    httpd = serve(svc, args.port, args.host)
    print(f"serving {args.config} on http://{args.host}:{httpd.server_address[1]} (/meta, /render)", flush=True)
    try:
        httpd.serve_forever()
    except KeyboardInterrupt:
        pass
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
