"""bench.py's driver contract on the CPU: the reference arm's JSON line (CPU oracle timed on
this host, same config object as our arm), the roofline objects, and the multi-GPU launch
guards (``--gpus N`` self-launch refuses a box with fewer GPUs; a launcher's WORLD_SIZE must
equal --gpus)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2306_16541_b200 import scene as psc  # noqa: E402


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=ROOT)


def test_reference_arm_line():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-tiles", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["metric"] == bench.METRIC and line["unit"] == bench.UNIT and line["higher_is_better"] is True
    assert line["n_gpus"] == 1 and line["steps"] == 1 and line["warmup"] == 1 and line["value"] > 0
    assert line["config"] == bench.workload_config(psc.config("c2"))      # like for like with our arm
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_stage_rooflines_objects():
    cfg = psc.config("c2")
    stages = {"march_warp": 1.7, "offset": 2.9, "radiance": 4.55, "composite": 0.17}
    roofs = bench.stage_rooflines(stages, cfg, 33554432, 29747775)
    assert set(roofs) == set(stages)
    for key, r in roofs.items():
        assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
        assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12 and r["limiter"]
        n = 29747775 if key in ("offset", "radiance") else 33554432
        unit = bench.KERNEL_UNITS[key][3]
        scale = 1e12 if r["bound"] == "tensor" else 1e9
        assert abs(r["achieved"] - n * unit / (stages[key] * 1e-3) / scale) < 1e-6 * r["achieved"]
    assert roofs["offset"]["bound"] == "tensor" and "frac_vs_sustained" in roofs["offset"]


def test_gpus_n_without_enough_gpus_fails_loudly():
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"], timeout=300)
    assert r.returncode == 2 and "--gpus 2 but only" in r.stderr


def test_launcher_world_size_must_match_gpus():
    r = _run(["--gpus", "4", "--steps", "1", "--warmup", "3"],
             env_extra={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=2 but --gpus 4" in r.stderr


@pytest.mark.parametrize("argv", [[], ["--gpus", "8", "--steps", "20", "--warmup", "5"]])
def test_defaults_and_flags(argv, monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"] + argv)
    a = bench.parse()
    if not argv:
        assert a.gpus == 1 and a.impl == "ours" and a.config == "c2" and a.warmup >= 3 and 1 <= a.steps <= 50
    else:
        assert a.gpus == 8 and a.steps == 20 and a.warmup == 5


def test_reference_arm_under_torchrun_prints_one_line():
    """The driver launches the reference arm like ours for N > 1 (torchrun, one process per
    GPU): rank 0 alone runs the CPU timing and prints the line, the other ranks exit 0."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    port = bench._free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
                        "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--cpu-tiles", "1"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
