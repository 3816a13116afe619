"""ctypes binding of libeca_b200.so (include/eca_b200.h).

The shared library is the product: there is no Python/CPU implementation to
fall back to.  Loading fails loudly when the library is missing, and every
device entry point raises when no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .params import EcaParams

LIB_PATH = Path(__file__).resolve().parent / "libeca_b200.so"

ECA_OK, ECA_ERR_ARG, ECA_ERR_CUDA, ECA_ERR_UNSUPPORTED = 0, -1, -2, -3
ACCEPTED, NO_CANDIDATES, LOW_SCORE, GEOMETRY_GATE = 0, 1, 2, 3
MAX_STRIPS, MAX_WIDTH, MAX_ATTEMPTS = 128, 4096, 8192
NET_FLOATS = 6209
BOUNDS_OVERLAP_PREVIOUS, BOUNDS_SHARE_SMS, BOUNDS_ZERO_COPY, PIPE_FRAMES_READY = 1, 2, 4, 8
LEARNED_TCGEN05, LEARNED_SIMT = 1, 2

_p = ctypes.c_void_p
_i32, _i64, _u64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
_PARAMS = ctypes.POINTER(EcaParams)
_I32P = ctypes.POINTER(ctypes.c_int32)

# name -> argtypes (all return int)
SIGNATURES = {
    "eca_strip_rows": [ctypes.c_int, ctypes.c_int, _f64, _I32P],
    "eca_triplet_table": [_u64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int16)],
    "eca_pcg64_doubles": [_u64, _i64, ctypes.POINTER(ctypes.c_double)],
    "eca_prefilter_bound": [_PARAMS, ctypes.POINTER(ctypes.c_double)],
    "eca_prefilter_selftest": [_PARAMS, _p, _p],
    "eca_points_workspace_bytes": [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)],
    "eca_points_handcrafted": [_p, ctypes.c_int, _i64, _i64, _I32P, _I32P, ctypes.c_int, _PARAMS,
                               _p, _p, _p, _p, _p],
    "eca_bounds_handcrafted": [_p, ctypes.c_int, _i64, _i64, _I32P, _I32P, ctypes.c_int, _PARAMS,
                               _p, _p, _p, _p, ctypes.c_int, _p],
    "eca_rescore_handcrafted": [ctypes.c_int, _I32P, ctypes.c_int, _PARAMS, _p, _p, _p, _p, _p],
    "eca_pipeline_bytes": [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)],
    "eca_pipeline_create": [ctypes.c_int, ctypes.c_int, ctypes.c_int, _I32P, ctypes.c_int, _PARAMS, _p,
                            _p, _i64, ctypes.POINTER(ctypes.c_void_p)],
    "eca_pipeline_step": [_p, _p, _i64, _i64, ctypes.c_int, _p, _p, ctypes.POINTER(ctypes.c_void_p)],
    "eca_pipeline_fence": [_p, _p],
    "eca_pipeline_run": [_p, _p, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_int, _p],
    "eca_pipeline_records": [_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
    "eca_pipeline_reset": [_p],
    "eca_pipeline_side_stream": [_p, ctypes.POINTER(ctypes.c_void_p)],
    "eca_pipeline_destroy": [_p],
    "eca_score_rows_handcrafted": [_p, ctypes.c_int, _i64, _i64, _I32P, _I32P, ctypes.c_int, _PARAMS,
                                   _p, _p, _p, _p, _p],
    "eca_fit": [_p, _p, _p, ctypes.c_int, ctypes.c_int, _PARAMS, _p, ctypes.c_int, _p, _p],
    "eca_estimate_batch_handcrafted": [_p, ctypes.c_int, _i64, _i64, _I32P, _I32P, ctypes.c_int, _PARAMS,
                                       _p, _p, _p, _p, _p, _p, _p, ctypes.c_int, _p],
    "eca_estimate_handcrafted": [_p, ctypes.c_int, _i64, _i64, _I32P, _I32P, ctypes.c_int, _PARAMS,
                                 _p, _p, _p, _p, _p, _p, _p],
    "eca_points_learned": [_p, ctypes.c_int, _i64, _i64, _I32P, _I32P, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, _p, _p, _p, _p, _p, _p, _p],
    "eca_points_learned_ex": [_p, ctypes.c_int, _i64, _i64, _I32P, _I32P, ctypes.c_int, ctypes.c_int,
                              ctypes.c_int, _p, _p, ctypes.c_int, _p, _p, _p, _p, _p],
    "eca_draw_mask": [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _i64, _p],
    "eca_crop_bounds": [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p],
    "eca_h2d_bands": [_p, ctypes.c_int, _i64, _i64, _I32P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                      _p, _p],
    "eca_crop_copy": [_p, ctypes.c_int, _i64, _i64, _p, _p, _p, ctypes.c_int, _p],
    "eca_nh_workspace_bytes": [ctypes.c_int, ctypes.c_int, ctypes.c_int, _f64,
                               ctypes.POINTER(ctypes.c_int64)],
    "eca_area_hausdorff": [_p, _p, _p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _f64, _p, _i64, _p,
                           _p, _p],
    "eca_boundary_points": [_p, ctypes.c_int, ctypes.c_int, _f64, _p, ctypes.c_int, _p, _p],
    "eca_hausdorff_workspace_bytes": [ctypes.c_int, ctypes.POINTER(ctypes.c_int64)],
    "eca_hausdorff_points": [_p, ctypes.c_int, _p, ctypes.c_int, _p, _i64, _p, _p, _p],
    "eca_train_workspace_bytes": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)],
    "eca_edgenet_forward": [_p, _p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p, _i64, _p, _p],
    "eca_edgenet_backward": [_p, _p, _p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p, _i64, _p, _p,
                             _p, _p],
    "eca_sgd_step": [_p, _p, ctypes.c_float, _p, _p],
}

_lib = None


class EcaError(RuntimeError):
    """A libeca_b200 call returned an error code."""


def load() -> ctypes.CDLL:
    """The loaded library (built in-tree by ``paper_2210_14771_b200.build``)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2210_14771_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_LOCAL", 0))
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        _lib = lib
    return _lib


def check(rc: int, what: str) -> int:
    if rc < 0:
        kind = {ECA_ERR_ARG: "invalid argument", ECA_ERR_CUDA: "CUDA error",
                ECA_ERR_UNSUPPORTED: "unsupported size"}.get(rc, "error")
        raise EcaError(f"{what}: {kind} (code {rc})")
    return rc
