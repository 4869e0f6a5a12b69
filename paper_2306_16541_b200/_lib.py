"""ctypes binding of ``libfvcuda.so`` (C ABI declared in ``include/fv_api.h``).

There is no fallback: if the library or a CUDA device is missing, the product path
raises.  Status codes map to the reference's exception types (``ad:26-31``).
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

from .errors import DimensionError, TrainingError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfvcuda.so")

FV_OK, FV_EDIM, FV_ENONFINITE, FV_ELAUNCH, FV_EUNSUPPORTED = 0, 1, 2, 3, 4
MAX_BONES, MAX_LEVELS, MAX_VOL_RES = 32, 16, 128

f3 = C.c_float * 3
vp = C.c_void_p


class FvCamera(C.Structure):
    _fields_ = [("kinv", C.c_float * 9), ("rot", C.c_float * 9), ("center", f3),
                ("width", C.c_int32), ("height", C.c_int32)]


class FvMarch(C.Structure):
    _fields_ = [("obox_min", f3), ("obox_max", f3), ("n_samples", C.c_int32), ("jitter", C.c_int32),
                ("seed", C.c_uint32), ("eps_w", C.c_float), ("eps_t", C.c_float), ("bg", f3),
                ("d_occ", vp), ("occ_scale", f3), ("d_pix", vp), ("pix_offset", C.c_int32),
                ("out_by_pixel", C.c_int32), ("round_samples", C.c_int32)]


MAX_SUBJECTS = 8


class FvSceneMerge(C.Structure):
    _fields_ = [("n_subjects", C.c_int32), ("cam", FvCamera * MAX_SUBJECTS), ("box_min", f3), ("box_max", f3),
                ("d_rgb", vp * MAX_SUBJECTS), ("d_alpha", vp * MAX_SUBJECTS), ("bg", f3)]


class FvWarp(C.Structure):
    _fields_ = [("n_bones", C.c_int32), ("vol_res", C.c_int32), ("vol_half", C.c_int32),
                ("d_vol_packed", vp), ("d_g", vp), ("wbox_min", f3), ("wscale", f3)]


class FvHash(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("n_feat", C.c_int32), ("log2_T", C.c_int32),
                ("res", C.c_int32 * MAX_LEVELS), ("dense", C.c_int32 * MAX_LEVELS),
                ("offset", C.c_uint32 * MAX_LEVELS), ("table_half", C.c_int32), ("d_table", vp),
                ("cmin", f3), ("cinv", f3)]


class FvField(C.Structure):
    _fields_ = [("precision", C.c_int32), ("pe_bands", C.c_int32), ("pe_w", C.c_float * 8),
                ("offset_enabled", C.c_int32), ("d_off_w", vp * 5), ("d_off_b", vp * 5),
                ("d_rad_w", vp * 3), ("d_rad_b", vp * 3), ("d_off_b0_eff", vp), ("d_tc_pack", vp)]


STRUCTS = (FvCamera, FvMarch, FvWarp, FvHash, FvField, FvSceneMerge)

P = C.POINTER
i32, i64, f32, sz = C.c_int32, C.c_int64, C.c_float, C.c_size_t

# name -> (restype, argtypes); exactly the functions declared in include/fv_api.h
SIGNATURES = {
    "fv_version": (i32, []),
    "fv_last_error": (C.c_char_p, []),
    "fv_device_sm": (i32, []),
    "fv_struct_sizes": (None, [P(i64)]),
    "fv_warp_pack": (i32, [vp, i32, P(FvWarp), vp, vp]),
    "fv_warp_fwd": (i32, [P(FvWarp), f32, vp, i64, vp, vp, vp, vp, vp]),
    "fv_warp_bwd": (i32, [P(FvWarp), f32, vp, i64, vp, vp, vp]),
    "fv_warp_bwd_g": (i32, [P(FvWarp), f32, vp, i64, vp, vp, vp, vp]),
    "fv_hash_fwd": (i32, [P(FvHash), vp, i64, vp, vp, vp]),
    "fv_hash_bwd": (i32, [P(FvHash), vp, i64, vp, vp, vp, vp]),
    "fv_hash_index_paired": (i32, [P(FvHash), vp, i64, vp, vp, vp]),
    "fv_gather_probe": (i32, [P(FvHash), vp, i64, i32, vp, i64, vp]),
    "fv_march_compact": (i32, [P(FvCamera), P(FvMarch), P(FvWarp), i64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "fv_linear_fwd": (i32, [vp, vp, vp, vp, i64, i32, i32, i32, vp]),
    "fv_linear_bwd": (i32, [vp, vp, vp, vp, vp, vp, vp, i64, i32, i32, i32, vp]),
    "fv_fused_mlp_fwd": (i32, [vp, i64, i32, i32, i32, vp, vp, vp, vp]),
    "fv_field_pack_bytes": (sz, []),
    "fv_field_pack": (i32, [P(FvField), vp, vp]),
    "fv_offset_bias": (i32, [P(FvField), vp, i32, vp, vp]),
    "fv_field_workspace_bytes": (sz, [i64, i32]),
    "fv_residual_offset": (i32, [P(FvField), vp, i64, f32, vp, vp]),
    "fv_field_fwd": (i32, [P(FvField), P(FvHash), vp, i64, f32, vp, vp, vp, sz, vp]),
    "fv_composite_fwd": (i32, [vp, vp, vp, i32, i32, i64, i32, P(f32), f32, f32, vp, vp, vp, vp]),
    "fv_composite_bwd": (i32, [vp, vp, vp, i32, i32, vp, i64, i32, P(f32), f32, vp, vp, vp, vp]),
    "fv_posenc_fwd": (i32, [vp, i64, f32, i32, P(f32), vp, i64, vp]),
    "fv_linear_fwd_tc": (i32, [vp, i64, vp, vp, vp, i64, i64, i32, i32, i32, vp]),
    "fv_linear_bwd_tc": (i32, [vp, i64, vp, vp, i64, vp, i64, vp, vp, vp, i64, i32, i32, vp]),
    "fv_linear_fwd_tc_bits": (i32, [vp, i64, vp, vp, vp, i64, i64, i32, i32, i32, vp, vp]),
    "fv_sample_bone_channels": (i32, [P(FvWarp), vp, i64, vp, vp]),
    "fv_transmittance": (i32, [vp, i64, i32, vp, vp]),
    "fv_transmittance_bwd": (i32, [vp, vp, vp, i64, i32, vp, vp]),
    "fv_sample_bone_channels_bwd": (i32, [P(FvWarp), vp, i64, vp, vp, vp, vp]),
    "fv_linear_bwd_tc_bits": (i32, [vp, i64, vp, vp, i64, vp, i64, vp, vp, vp, i64, i32, i32, vp]),
    "fv_posenc_bwd": (i32, [vp, i64, f32, i32, P(f32), vp, i64, vp, vp]),
    "fv_xfinal": (i32, [vp, vp, i64, f32, vp, vp]),
    "fv_heads_fwd": (i32, [vp, vp, i64, f32, vp, vp]),
    "fv_heads_bwd": (i32, [vp, vp, vp, i64, f32, vp, vp]),
    "fv_softmax0_fwd": (i32, [vp, i32, i64, vp, vp]),
    "fv_softmax0_bwd": (i32, [vp, vp, i32, i64, vp, vp]),
    "fv_mse_loss": (i32, [vp, vp, vp, i64, vp, vp, vp]),
    "fv_render_workspace_bytes": (sz, [i64, i32, i32]),
    "fv_march_warp": (i32, [P(FvCamera), P(FvMarch), P(FvWarp), i64, vp, vp, vp, vp, vp]),
    "fv_patch_loss": (i32, [vp, vp, vp, i32, i32, f32, f32, vp, vp, vp]),
    "fv_scene_composite": (i32, [P(FvSceneMerge), i64, i64, vp, vp, vp]),
    "fv_render_fwd": (i32, [P(FvCamera), P(FvMarch), P(FvWarp), P(FvHash), P(FvField), i64, vp, sz,
                            vp, vp, vp, vp]),
    "fv_render_fwd_timed": (i32, [P(FvCamera), P(FvMarch), P(FvWarp), P(FvHash), P(FvField), i64, vp, sz,
                                  vp, vp, P(f32), P(i64), vp]),
    "fv_occupancy_workspace_bytes": (sz, [i32]),
    "fv_occupancy_build": (i32, [P(FvMarch), P(FvWarp), P(FvHash), P(FvField), f32, vp, sz, vp, vp]),
    "fv_check_finite": (i32, [vp, i64, i32, vp, vp]),
    "fv_adam_step": (i32, [vp, vp, vp, vp, i64, P(i64), P(f32), i32, i32, f32, f32, f32, vp, i64, i64,
                           vp, vp]),
}

_lib = None


def load() -> C.CDLL:
    """Load libfvcuda.so once; raise (never fall back) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built -- run `make` (or __graft_entry__.build())")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        sizes = (C.c_int64 * len(STRUCTS))()
        lib.fv_struct_sizes(sizes)
        want = [C.sizeof(s) for s in STRUCTS]
        if list(sizes) != want:
            raise RuntimeError(f"fv_api struct layout mismatch: C {list(sizes)} vs ctypes {want}")
        _lib = lib
    return _lib


def check(code: int, what: str = "") -> None:
    if code == FV_OK:
        return
    msg = load().fv_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if code == FV_EDIM:
        raise DimensionError(text)
    if code == FV_ENONFINITE:
        raise TrainingError(text)
    raise RuntimeError(f"libfvcuda error {code}: {text}")


def ptr(t) -> int:
    """Raw device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise RuntimeError("libfvcuda takes CUDA tensors only (no CPU fallback)")
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def farr(ctype_arr, values: Sequence[float]):
    for i, v in enumerate(values):
        ctype_arr[i] = v
    return ctype_arr
