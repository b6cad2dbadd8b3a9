"""ctypes bindings of the in-tree native libraries.

* ``libsfmcov_b200.so`` — the sm_100a CUDA library behind include/sfmcov_b200.h
  (the drop-in C ABI).  Loading it never needs a GPU; creating a handle does,
  and fails loudly without one (there is no CPU fallback).
* ``libsfmcov_synth.so`` — host-only seeded scene generators (harness).

Both are built in-tree by ``__graft_entry__.build()`` (csrc/Makefile).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libsfmcov_b200.so"
SYNTH_PATH = _HERE / "libsfmcov_synth.so"

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_int64_p = C.POINTER(C.c_int64)


class Scene(C.Structure):
    _fields_ = [
        ("n_cams", C.c_int32),
        ("n_pts", C.c_int32),
        ("n_obs", C.c_int32),
        ("cam_params", C.c_int32),
        ("cams", C.c_void_p),
        ("pts", C.c_void_p),
        ("obs_cam", C.c_void_p),
        ("obs_pt", C.c_void_p),
        ("obs_u", C.c_void_p),
        ("obs_sigma", C.c_void_p),
    ]


class Options(C.Structure):
    _fields_ = [
        ("threads", C.c_int32),
        ("point_covariances", C.c_int32),
        ("camera_cross_covariances", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Diagnostics(C.Structure):
    _fields_ = [
        ("scale_min", C.c_double),
        ("scale_max", C.c_double),
        ("min_pivot", C.c_double),
        ("max_pivot", C.c_double),
        ("inertia_positive", C.c_int32),
        ("inertia_negative", C.c_int32),
        ("negative_eigenvalue_warnings", C.c_int32),
        ("n_flagged", C.c_int32),
        ("peak_dense_bytes", C.c_int64),
        ("largest_dense_dim", C.c_int64),
        ("flagged", c_int64_p),
        ("flagged_capacity", C.c_int64),
    ]


class ErrorStruct(C.Structure):
    _fields_ = [("kind", C.c_int32), ("stage", C.c_char * 32), ("message", C.c_char * 480)]


# Every symbol include/sfmcov_b200.h declares for the CUDA library, with its
# (restype, argtypes).
CUDA_SYMBOLS = {
    "sfmcov_cuda_create": (C.c_void_p, [C.c_int32, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_destroy": (None, [C.c_void_p]),
    "sfmcov_cuda_stream": (C.c_void_p, [C.c_void_p]),
    "sfmcov_cuda_compute_covariance": (
        C.c_int32,
        [C.c_void_p, C.POINTER(Scene), C.POINTER(Options), C.c_void_p, C.POINTER(Diagnostics), C.POINTER(ErrorStruct)],
    ),
    "sfmcov_cuda_compute_covariance_full": (
        C.c_int32,
        [C.c_void_p, C.POINTER(Scene), C.POINTER(Options), C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Diagnostics),
         C.POINTER(ErrorStruct)],
    ),
    "sfmcov_cuda_compute_covariance_device": (
        C.c_int32,
        [C.c_void_p, C.POINTER(Scene), C.POINTER(Options), C.c_void_p, C.POINTER(Diagnostics), C.POINTER(ErrorStruct)],
    ),
    "sfmcov_cuda_observation_index": (
        C.c_int32,
        [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(ErrorStruct)],
    ),
    "sfmcov_cuda_jacobian": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_nullspace": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_fisher": (
        C.c_int32,
        [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
         C.POINTER(Diagnostics), C.POINTER(ErrorStruct)],
    ),
    "sfmcov_cuda_schur": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_spd_inverse_blocks": (
        C.c_int32,
        [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, c_double_p, c_double_p, C.POINTER(ErrorStruct)],
    ),
    "sfmcov_cuda_last_stage_times": (C.c_int32, [C.c_void_p, c_double_p, C.c_int32]),
    "sfmcov_cuda_stage_name": (C.c_char_p, [C.c_int32]),
    "sfmcov_cuda_last_counts": (C.c_int32, [C.c_void_p, c_int64_p, C.c_int32]),
    "sfmcov_cuda_set_profiling": (None, [C.c_void_p, C.c_int32]),
    "sfmcov_nccl_unique_id": (C.c_int32, [C.c_char_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_comm_init": (C.c_int32, [C.c_void_p, C.c_char_p, C.c_int32, C.c_int32, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_compute_covariance_sharded": (
        C.c_int32,
        [C.c_void_p, C.POINTER(Scene), C.POINTER(Options), C.c_void_p, C.POINTER(Diagnostics), C.POINTER(ErrorStruct)],
    ),
    "sfmcov_cuda_compute_covariance_sharded_device": (
        C.c_int32,
        [C.c_void_p, C.POINTER(Scene), C.POINTER(Options), C.c_void_p, C.POINTER(Diagnostics), C.POINTER(ErrorStruct)],
    ),
    "sfmcov_cuda_compute_covariance_emulated": (
        C.c_int32,
        [C.c_void_p, C.POINTER(Scene), C.POINTER(Options), C.c_int32, C.c_void_p, C.POINTER(Diagnostics),
         C.POINTER(ErrorStruct)],
    ),
    "sfmcov_plan_dense": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, c_int64_p, c_int64_p,
                                      C.c_void_p]),
    "sfmcov_plan_chunks": (C.c_int32, [C.c_int64, C.c_int32, C.c_int32, c_int64_p, c_int64_p]),
    "sfmcov_cuda_device": (C.c_int32, [C.c_void_p]),
    "sfmcov_cuda_nullspace_residual": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.c_int32, C.c_void_p,
                                                   C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_condition_columns": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                                  C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_apply_conditioning": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                   C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_schur_system": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_invert_symmetric": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                                 C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_extract_camera_blocks": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                                      C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_full_covariance": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_int64, C.c_void_p,
                                                C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_set_sharded_stage_a": (None, [C.c_void_p, C.c_int32]),
    "sfmcov_cuda_refine_covariance": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.c_int32, C.c_int32,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_pseudoinverse_covariance": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_int64, C.c_void_p, C.c_void_p,
                                                         C.c_void_p, c_double_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_worker": (C.c_void_p, [C.c_void_p, C.c_int32, C.POINTER(ErrorStruct)]),
    "sfmcov_view_graph": (C.c_int32, [C.POINTER(Scene), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                      c_int64_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_view_graph": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_int64, c_int64_p, C.POINTER(ErrorStruct)]),
    "sfmcov_extract_neighborhood": (C.c_int32, [C.POINTER(Scene), C.c_int64, C.c_int32, C.c_void_p, c_int64_p,
                                                C.c_void_p, c_int64_p, c_int32_p, C.POINTER(ErrorStruct)]),
    "sfmcov_plan_coverage": (C.c_int32, [C.POINTER(Scene), C.c_int32, C.c_uint64, C.c_void_p, C.c_int64, C.c_void_p,
                                         C.c_int64, c_int64_p, C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_approximate_covariances": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_int32, C.c_int32, C.c_uint64,
                                                        C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                                        C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_approximate_covariances_shard": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_int32, C.c_int32,
                                                              C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                                              C.c_void_p, C.c_void_p, c_int64_p,
                                                              C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_error_size_sweep": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.c_int32, C.c_int32,
                                                 C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, c_int64_p,
                                                 C.POINTER(ErrorStruct)]),
    "sfmcov_cuda_monotonicity_check": (C.c_int32, [C.c_void_p, C.POINTER(Scene), C.c_void_p, C.c_int64, C.c_void_p,
                                                   C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                                   c_int64_p, c_int64_p, C.POINTER(ErrorStruct)]),
}

SYNTH_SYMBOLS = {
    "sfmcov_synth_cube": (C.c_void_p, [C.c_uint64, C.c_double, C.c_int32]),
    "sfmcov_synth_random": (C.c_void_p, [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_double, C.c_int32]),
    "sfmcov_synth_config": (C.c_void_p, [C.c_int32, C.c_uint64]),
    "sfmcov_synth_transform": (C.c_void_p, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double]),
    "sfmcov_synth_sizes": (None, [C.c_void_p, c_int64_p, c_int64_p, c_int64_p, c_int32_p]),
    "sfmcov_synth_export": (None, [C.c_void_p] + [C.c_void_p] * 6),
    "sfmcov_synth_free": (None, [C.c_void_p]),
    "sfmcov_synth_last_error": (C.c_char_p, []),
    "sfmcov_scene_load": (C.c_void_p, [C.c_char_p, C.POINTER(ErrorStruct)]),
    "sfmcov_scene_save": (C.c_int32, [C.POINTER(Scene), C.c_char_p, C.POINTER(ErrorStruct)]),
    "sfmcov_scene_load_binary": (C.c_void_p, [C.c_char_p, C.POINTER(ErrorStruct)]),
    "sfmcov_scene_save_binary": (C.c_int32, [C.POINTER(Scene), C.c_char_p, C.POINTER(ErrorStruct)]),
    "sfmcov_covio_pack_upper_triangle": (None, [C.c_void_p, C.c_int32, C.c_void_p]),
    "sfmcov_covio_unpack_upper_triangle": (None, [C.c_void_p, C.c_int32, C.c_void_p]),
    "sfmcov_covio_save_json": (C.c_int32, [C.c_char_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                           C.POINTER(ErrorStruct)]),
    "sfmcov_covio_load_json": (C.c_int32, [C.c_char_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.POINTER(ErrorStruct)]),
    "sfmcov_covio_save_csv": (C.c_int32, [C.c_char_p, C.c_int64, C.c_int32, C.c_void_p, C.POINTER(ErrorStruct)]),
}

_cuda_lib = None
_synth_lib = None


def _bind(lib, table):
    for name, (res, args) in table.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def cuda_lib():
    """The CUDA library; raises if it has not been built (no fallback)."""
    global _cuda_lib
    if _cuda_lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(this package has no CPU fallback)")
        _cuda_lib = _bind(C.CDLL(str(LIB_PATH)), CUDA_SYMBOLS)
    return _cuda_lib


def synth_lib():
    global _synth_lib
    if _synth_lib is None:
        if not SYNTH_PATH.exists():
            raise RuntimeError(f"{SYNTH_PATH} is missing: run __graft_entry__.build()")
        _synth_lib = _bind(C.CDLL(str(SYNTH_PATH)), SYNTH_SYMBOLS)
    return _synth_lib


def ptr(a):
    """Address of a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0")
