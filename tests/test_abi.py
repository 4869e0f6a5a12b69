"""The C-ABI library loads without a GPU and exports exactly what include/fv_api.h declares."""

import ctypes
import os
import re

import pytest

from paper_2306_16541_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "fv_api.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_struct_layout_and_version_without_gpu():
    lib = _lib.load()  # checks ctypes struct sizes against sizeof() in C
    assert lib.fv_version() == 100
    sizes = (ctypes.c_int64 * len(_lib.STRUCTS))()
    lib.fv_struct_sizes(sizes)
    assert all(s > 0 for s in sizes)


def test_error_codes_map_to_reference_exceptions():
    import pytest
    from paper_2306_16541_b200.errors import DimensionError
    lib = _lib.load()
    with pytest.raises(DimensionError):
        _lib.check(lib.fv_linear_fwd(None, None, None, None, -1, 0, 0, 0, None), "fv_linear_fwd")


def test_no_cpu_fallback_missing_library_and_cpu_tensors(monkeypatch):
    """The product path fails loudly: a missing libfvcuda.so raises (no silent CPU path), and
    the operators refuse CPU tensors instead of computing on the host."""
    import torch
    from paper_2306_16541_b200 import autodiff, fused
    from paper_2306_16541_b200.errors import DimensionError
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libfvcuda.so")
    with pytest.raises(RuntimeError, match="not built"):
        _lib.load()
    monkeypatch.undo()
    with pytest.raises(DimensionError):
        autodiff.posenc(torch.zeros((4, 3)), 6)
    with pytest.raises(DimensionError):
        autodiff.transmittance(torch.zeros((2, 3)))
    with pytest.raises(DimensionError):
        fused.fused_forward(fused.FusedMlp([torch.zeros((3, 64)), torch.zeros((64, 2))]), torch.zeros((4, 3)))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.ptr(torch.zeros(3))


def test_fused_mlp_random_draws_the_reference_weights():
    """FusedMlp.random follows fu:120-130's draw order (per layer: He-normal weights, then
    N(0, 0.01) biases) bit for bit (golden mlp_* from the reference), and the reference's
    shape rules raise DimensionError."""
    import numpy as np
    import torch
    from paper_2306_16541_b200 import fused
    from paper_2306_16541_b200.errors import DimensionError
    g = np.load(os.path.join(ROOT, "tests", "golden", "ref_primitives.npz"))
    mlp = fused.FusedMlp.random(32, 4, depth=2, seed=3, device="cpu")
    assert mlp.depth == 2 and mlp.in_dim == 32 and mlp.out_dim == 4
    for i in range(3):
        assert np.array_equal(mlp.weights[i].numpy(), g[f"mlp_w{i}"])
        assert np.array_equal(mlp.biases[i].numpy(), g[f"mlp_b{i}"])
    nb = fused.FusedMlp.random(32, 4, depth=2, seed=3, with_bias=False, device="cpu")
    assert all(float(b.abs().sum()) == 0.0 for b in nb.biases)
    with pytest.raises(DimensionError):
        fused.FusedMlp([torch.zeros((32, 64))])
    with pytest.raises(DimensionError):
        fused.FusedMlp([torch.zeros((32, 64)), torch.zeros((64, 65))])
    with pytest.raises(DimensionError):
        fused.FusedMlp([torch.zeros((32, 64)), torch.zeros((64, 4))], [torch.zeros(64), torch.zeros(3)])


def test_sample_slot_limit_is_a_loud_error_without_gpu():
    """Sample ids are int32 in the ABI: a launch whose padded(n_rays) x n_samples reaches
    2^31 slots is refused with FV_EDIM before anything touches the device (the Python
    Renderer splits such ray sets into chunks, tests/test_gpu_edge.py)."""
    from paper_2306_16541_b200.errors import DimensionError
    lib = _lib.load()
    cam, mar, war, hsh, fld = _lib.FvCamera(), _lib.FvMarch(), _lib.FvWarp(), _lib.FvHash(), _lib.FvField()
    war.n_bones, war.vol_res = 24, 32
    hsh.n_levels, hsh.n_feat, hsh.log2_T, hsh.d_table = 16, 2, 19, 16   # never dereferenced
    mar.n_samples = 128
    n_rays = (1 << 31) // 128 + 32                                       # just past the limit
    for fn, args in (("fv_render_fwd", (ctypes.byref(cam), ctypes.byref(mar), ctypes.byref(war), ctypes.byref(hsh),
                                         ctypes.byref(fld), n_rays, None, 0, None, None, None, None)),
                     ("fv_march_compact", (ctypes.byref(cam), ctypes.byref(mar), ctypes.byref(war), n_rays, 16, 16,
                                           16, 16, 16, None, None, None))):
        with pytest.raises(DimensionError, match="2\\^31"):
            _lib.check(getattr(lib, fn)(*args), fn)
