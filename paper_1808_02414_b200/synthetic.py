"""Seeded synthetic scenes (host-side harness, libsfmcov_synth.so).

generate_cube_scene / generate_random_scene / transform_scene restate the
reference generators (src/synthetic.cpp:52-194); generate_config(1..5) builds
the BASELINE.json configurations (P = 9 cameras on a radius-20 sphere,
f = 1000, unit observation covariance, N(0, 1 px) pixel noise).  The paper's
datasets are not available here; these stand in for them.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .sfmcov import Error, ErrorKind, Reconstruction


def _take(h) -> Reconstruction:
    lib = N.synth_lib()
    if not h:
        raise Error(ErrorKind.invariant, "generate", lib.sfmcov_synth_last_error().decode())
    try:
        n, m, t, P = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        lib.sfmcov_synth_sizes(h, C.byref(n), C.byref(m), C.byref(t), C.byref(P))
        cams = np.empty((n.value, P.value))
        pts = np.empty((m.value, 3))
        oc = np.empty(t.value, np.int32)
        op = np.empty(t.value, np.int32)
        u = np.empty((t.value, 2))
        sg = np.empty((t.value, 2, 2))
        lib.sfmcov_synth_export(h, cams.ctypes.data, pts.ctypes.data, oc.ctypes.data, op.ctypes.data,
                                u.ctypes.data, sg.ctypes.data)
        return Reconstruction(cams, pts, oc, op, u, sg)
    finally:
        lib.sfmcov_synth_free(h)


def generate_cube_scene(seed: int, noise_px: float, cam_params: int = 8) -> Reconstruction:
    return _take(N.synth_lib().sfmcov_synth_cube(seed, noise_px, cam_params))


def generate_random_scene(n_cams: int, n_pts: int, visibility: float, seed: int, noise_px: float,
                          cam_params: int = 8) -> Reconstruction:
    return _take(N.synth_lib().sfmcov_synth_random(n_cams, n_pts, visibility, seed, noise_px, cam_params))


def generate_config(index: int, seed: int | None = None) -> Reconstruction:
    return _take(N.synth_lib().sfmcov_synth_config(index, index if seed is None else seed))


def transform_scene(rec: Reconstruction, R: np.ndarray, t: np.ndarray, scale: float) -> Reconstruction:
    """X' = s R X + t, C' likewise, r' = log(R(r) R^T) (src/synthetic.cpp:185-194)."""
    R = np.asarray(R, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    out = rec.copy()
    from .rotation import rotation_log, rotation_matrix
    for i in range(out.num_cameras()):
        Rc = rotation_matrix(out.cams[i, :3])
        out.cams[i, :3] = rotation_log(Rc @ R.T)
        out.cams[i, 3:6] = scale * (R @ out.cams[i, 3:6]) + t
    out.pts = scale * (out.pts @ R.T) + t
    return out
