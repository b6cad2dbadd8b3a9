"""Covariance IO (reference include/sfmcov/covariance_io.hpp,
src/covariance_io.cpp:17-122): the packed upper triangle of a camera block,
the JSON file with the diagnostics (byte-identical to the reference's
nlohmann dump) and the %.17g CSV.  Host library (libsfmcov_synth.so)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .sfmcov import CovarianceDiagnostics, CovarianceResult, _raise


def pack_upper_triangle(block: np.ndarray) -> np.ndarray:
    """(0,0),(0,1),...,(P-1,P-1) of a P x P block (covariance_io.hpp:12)."""
    b = np.ascontiguousarray(block, dtype=np.float64)
    P = b.shape[0]
    out = np.empty(P * (P + 1) // 2)
    N.synth_lib().sfmcov_covio_pack_upper_triangle(b.ctypes.data, P, out.ctypes.data)
    return out


def unpack_upper_triangle(tri: np.ndarray) -> np.ndarray:
    t = np.ascontiguousarray(tri, dtype=np.float64)
    P = int(round((np.sqrt(8 * len(t) + 1) - 1) / 2))
    out = np.empty((P, P))
    N.synth_lib().sfmcov_covio_unpack_upper_triangle(t.ctypes.data, P, out.ctypes.data)
    return out


def _diag_struct(d: CovarianceDiagnostics, keep):
    s = N.Diagnostics()
    s.scale_min, s.scale_max = d.scale_min, d.scale_max
    s.min_pivot, s.max_pivot = d.min_pivot, d.max_pivot
    s.inertia_positive, s.inertia_negative = d.inertia_positive, d.inertia_negative
    s.negative_eigenvalue_warnings = d.negative_eigenvalue_warnings
    s.peak_dense_bytes, s.largest_dense_dim = d.peak_dense_bytes, d.largest_dense_dim
    fl = np.ascontiguousarray(d.flagged_columns, dtype=np.int64)
    keep.append(fl)
    s.n_flagged = len(fl)
    s.flagged = fl.ctypes.data_as(C.POINTER(C.c_int64)) if len(fl) else None
    s.flagged_capacity = len(fl)
    return s


def save_covariance_json(result: CovarianceResult, path: str) -> None:
    cov = np.ascontiguousarray(result.camera_cov, dtype=np.float64)
    n, P = cov.shape[0], cov.shape[1]
    keep = []
    d = _diag_struct(result.diagnostics, keep)
    err = N.ErrorStruct()
    _raise(N.synth_lib().sfmcov_covio_save_json(str(path).encode(), n, P, cov.ctypes.data, C.byref(d), C.byref(err)),
           err)


def load_covariance_json(path: str, cam_params: int = 8) -> CovarianceResult:
    lib = N.synth_lib()
    err = N.ErrorStruct()
    n = C.c_int64()
    d = N.Diagnostics()
    _raise(lib.sfmcov_covio_load_json(str(path).encode(), cam_params, 0, None, C.byref(n), C.byref(d), C.byref(err)),
           err)
    cov = np.empty((max(1, n.value), cam_params, cam_params))
    fl = np.empty(max(1, d.n_flagged), np.int64)
    d.flagged = fl.ctypes.data_as(C.POINTER(C.c_int64))
    d.flagged_capacity = len(fl)
    _raise(lib.sfmcov_covio_load_json(str(path).encode(), cam_params, n.value, cov.ctypes.data, C.byref(n),
                                      C.byref(d), C.byref(err)), err)
    diag = CovarianceDiagnostics(d.scale_min, d.scale_max, fl[:d.n_flagged].tolist(), d.min_pivot, d.max_pivot,
                                 d.inertia_positive, d.inertia_negative, d.negative_eigenvalue_warnings,
                                 d.peak_dense_bytes, d.largest_dense_dim)
    return CovarianceResult(cov[:n.value], diag)


def save_covariance_csv(result: CovarianceResult, path: str) -> None:
    cov = np.ascontiguousarray(result.camera_cov, dtype=np.float64)
    err = N.ErrorStruct()
    _raise(N.synth_lib().sfmcov_covio_save_csv(str(path).encode(), cov.shape[0], cov.shape[1], cov.ctypes.data,
                                               C.byref(err)), err)
