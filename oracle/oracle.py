"""TEST INFRASTRUCTURE — ctypes wrapper of the CPU restatement (oracle/).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module, and only as the checker / CPU baseline.  Scenes are any object with
the SoA attributes of paper_1808_02414_b200.Reconstruction (cams, pts,
obs_cam, obs_pt, obs_u, obs_sigma).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle_sfmcov.so"
KINDS = {1: "io", 2: "parse", 3: "invariant", 4: "degenerate", 5: "dimension", 6: "size_guard"}


class OracleScene(C.Structure):
    _fields_ = [("n_cams", C.c_int32), ("n_pts", C.c_int32), ("n_obs", C.c_int32), ("cam_params", C.c_int32),
                ("cams", C.c_void_p), ("pts", C.c_void_p), ("obs_cam", C.c_void_p), ("obs_pt", C.c_void_p),
                ("obs_u", C.c_void_p), ("obs_sigma", C.c_void_p)]


class OracleDiag(C.Structure):
    _fields_ = [("scale_min", C.c_double), ("scale_max", C.c_double), ("min_pivot", C.c_double),
                ("max_pivot", C.c_double), ("inertia_positive", C.c_int32), ("inertia_negative", C.c_int32),
                ("negative_eigenvalue_warnings", C.c_int32), ("n_flagged", C.c_int32),
                ("peak_dense_bytes", C.c_int64), ("largest_dense_dim", C.c_int64)]


class OracleError(C.Structure):
    _fields_ = [("kind", C.c_int32), ("stage", C.c_char * 32), ("message", C.c_char * 480)]


class OracleFailure(RuntimeError):
    def __init__(self, kind, stage, what):
        super().__init__(what)
        self.kind = kind
        self.kind_name = KINDS.get(kind, str(kind))
        self.stage = stage


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX")
        L = C.CDLL(str(LIB))
        vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
        sig = {
            "oracle_blas_corename": (C.c_char_p, []),
            "oracle_blas_threads": (None, [C.c_int]),
            "oracle_validate": (i32, [vp, vp]),
            "oracle_observation_index": (i32, [vp, vp, vp, vp, vp]),
            "oracle_rotation_matrix": (None, [vp, vp]),
            "oracle_rotate_point_derivative": (None, [vp, vp, vp]),
            "oracle_sincos": (None, [C.c_double, dp, dp]),
            "oracle_observation_jacobian": (i32, [C.c_int, vp, vp, vp, vp, vp]),
            "oracle_project": (i32, [C.c_int, vp, vp, vp, vp]),
            "oracle_jacobian": (i32, [vp, C.c_int, vp, vp, vp]),
            "oracle_nullspace": (i32, [vp, vp, dp, vp]),
            "oracle_nullspace_residual": (C.c_double, [vp, vp]),
            "oracle_fisher": (i32, [vp, vp, vp, vp, vp, vp, vp, i64, vp, vp]),
            "oracle_schur": (i32, [vp, C.c_int, vp, vp]),
            "oracle_invert_schur": (i32, [vp, i64, vp, vp, vp]),
            "oracle_compute_covariance": (i32, [vp, C.c_int, vp, vp, vp, i64, vp, vp]),
            "oracle_compute_covariance_full": (i32, [vp, C.c_int, vp, vp, vp, vp, vp, i64, vp]),
            "oracle_dense_fisher": (i32, [vp, vp, vp]),
            "oracle_pseudoinverse": (i32, [vp, i64, vp, vp, vp, dp, vp]),
            "oracle_exact_camera_blocks": (i32, [vp, i64, vp, vp]),
            "oracle_trs_sample": (None, [C.c_int]),
            "oracle_trs_sample_info": (None, [vp, vp]),
            "oracle_cholesky_route": (i32, [vp, i64, C.c_int, vp, C.c_int, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _scene(rec) -> OracleScene:
    s = OracleScene()
    s.n_cams, s.n_pts, s.n_obs = rec.cams.shape[0], rec.pts.shape[0], rec.obs_cam.shape[0]
    s.cam_params = rec.cams.shape[1]
    s.cams, s.pts = rec.cams.ctypes.data, rec.pts.ctypes.data
    s.obs_cam, s.obs_pt = rec.obs_cam.ctypes.data, rec.obs_pt.ctypes.data
    s.obs_u = None if rec.obs_u is None else rec.obs_u.ctypes.data
    s.obs_sigma = None if rec.obs_sigma is None else rec.obs_sigma.ctypes.data
    return s


def _check(code, err):
    if code:
        raise OracleFailure(code, err.stage.decode(), err.message.decode())


def blas_corename() -> str:
    return lib().oracle_blas_corename().decode()


def validate(rec):
    err = OracleError()
    _check(lib().oracle_validate(C.byref(_scene(rec)), C.byref(err)), err)


def observation_index(rec):
    n, m, t = rec.cams.shape[0], rec.pts.shape[0], rec.obs_cam.shape[0]
    oc, op = np.empty(n + 1, np.int64), np.empty(m + 1, np.int64)
    ic, ip = np.empty(max(t, 1), np.int32), np.empty(max(t, 1), np.int32)
    lib().oracle_observation_index(C.byref(_scene(rec)), oc.ctypes.data, ic.ctypes.data, op.ctypes.data, ip.ctypes.data)
    return oc, ic[:t], op, ip[:t]


def rotation_matrix(r):
    r = np.ascontiguousarray(r, dtype=np.float64)
    R = np.empty((3, 3))
    lib().oracle_rotation_matrix(r.ctypes.data, R.ctypes.data)
    return R


def rotate_point_derivative(r, w):
    r = np.ascontiguousarray(r, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    D = np.empty((3, 3))
    lib().oracle_rotate_point_derivative(r.ctypes.data, w.ctypes.data, D.ctypes.data)
    return D


def sincos(x: float):
    s, c = C.c_double(), C.c_double()
    lib().oracle_sincos(float(x), C.byref(s), C.byref(c))
    return s.value, c.value


def observation_jacobian(cam, X):
    cam = np.ascontiguousarray(cam, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    P = cam.shape[0]
    jc, jp = np.empty((2, P)), np.empty((2, 3))
    err = OracleError()
    _check(lib().oracle_observation_jacobian(P, cam.ctypes.data, X.ctypes.data, jc.ctypes.data, jp.ctypes.data,
                                             C.byref(err)), err)
    return jc, jp


def project(cam, X):
    cam = np.ascontiguousarray(cam, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    u = np.empty(2)
    err = OracleError()
    _check(lib().oracle_project(cam.shape[0], cam.ctypes.data, X.ctypes.data, u.ctypes.data, C.byref(err)), err)
    return u


def jacobian(rec, threads=1):
    t, P = rec.obs_cam.shape[0], rec.cams.shape[1]
    jc, jp = np.empty((max(t, 1), 2, P)), np.empty((max(t, 1), 2, 3))
    err = OracleError()
    _check(lib().oracle_jacobian(C.byref(_scene(rec)), threads, jc.ctypes.data, jp.ctypes.data, C.byref(err)), err)
    return jc[:t], jp[:t]


def nullspace(rec):
    rows = rec.cams.shape[1] * rec.cams.shape[0] + 3 * rec.pts.shape[0]
    H = np.empty((max(rows, 1), 7))
    res = C.c_double()
    err = OracleError()
    _check(lib().oracle_nullspace(C.byref(_scene(rec)), H.ctypes.data, C.byref(res), C.byref(err)), err)
    return H[:rows], res.value


def nullspace_residual(rec, H):
    H = np.ascontiguousarray(H, dtype=np.float64)
    return lib().oracle_nullspace_residual(C.byref(_scene(rec)), H.ctypes.data)


def fisher(rec):
    n, m, t, P = rec.cams.shape[0], rec.pts.shape[0], rec.obs_cam.shape[0], rec.cams.shape[1]
    D, A, Cp = np.empty((max(n, 1), P, P)), np.empty((max(m, 1), 3, 3)), np.empty((max(t, 1), P, 3))
    sa, sb = np.empty(max(P * n + 3 * m, 1)), np.empty(7)
    fl = np.empty(max(P * n + 3 * m, 1), np.int64)
    nf = C.c_int64()
    err = OracleError()
    _check(lib().oracle_fisher(C.byref(_scene(rec)), D.ctypes.data, A.ctypes.data, Cp.ctypes.data, sa.ctypes.data,
                               sb.ctypes.data, fl.ctypes.data, fl.size, C.byref(nf), C.byref(err)), err)
    return D[:n], A[:m], Cp[:t], sa[:P * n + 3 * m], sb, fl[:nf.value].tolist()


def schur(rec, threads=1):
    dim = rec.cams.shape[1] * rec.cams.shape[0] + 7
    z = np.empty((dim, dim), order="F")
    err = OracleError()
    _check(lib().oracle_schur(C.byref(_scene(rec)), threads, z.ctypes.data, C.byref(err)), err)
    return z


def invert_schur(z):
    z = np.asfortranarray(z, dtype=np.float64)
    n = z.shape[0]
    out = np.empty((n, n), order="F")
    d = OracleDiag()
    err = OracleError()
    _check(lib().oracle_invert_schur(z.ctypes.data, n, out.ctypes.data, C.byref(d), C.byref(err)), err)
    return out, d


def compute_covariance(rec, threads=1):
    """Returns (camera_cov (n,P,P), OracleDiag, flagged, stage times dict)."""
    n, P = rec.cams.shape[0], rec.cams.shape[1]
    cov = np.empty((max(n, 1), P, P))
    d = OracleDiag()
    fl = np.empty(max(P * n + 3 * rec.pts.shape[0], 1), np.int64)
    times = np.zeros(10)
    err = OracleError()
    _check(lib().oracle_compute_covariance(C.byref(_scene(rec)), threads, cov.ctypes.data, C.byref(d), fl.ctypes.data,
                                           fl.size, times.ctypes.data, C.byref(err)), err)
    names = ["validate", "jacobian", "nullspace", "fisher", "conditioning", "schur", "dsytrf", "dsytrs2", "extract",
             "total"]
    return cov[:n], d, fl[:d.n_flagged].tolist(), dict(zip(names, times.tolist()))


def compute_covariance_full(rec, threads=1, point_covariances=True, camera_cross_covariances=True):
    """compute_covariance with the reference's optional outputs
    (covariance.cpp:283-348): returns (camera_cov (n,P,P), point_cov (m,3,3) or
    None, camera_matrix (Pn,Pn) or None, OracleDiag)."""
    n, P, m = rec.cams.shape[0], rec.cams.shape[1], rec.pts.shape[0]
    cov = np.empty((max(n, 1), P, P))
    pc = np.empty((max(m, 1), 3, 3)) if point_covariances else None
    cm = np.empty((P * n, P * n), order="F") if camera_cross_covariances else None
    d = OracleDiag()
    fl = np.empty(max(P * n + 3 * m, 1), np.int64)
    err = OracleError()
    _check(lib().oracle_compute_covariance_full(C.byref(_scene(rec)), threads, cov.ctypes.data,
                                                None if pc is None else pc.ctypes.data,
                                                None if cm is None else cm.ctypes.data, C.byref(d), fl.ctypes.data,
                                                fl.size, C.byref(err)), err)
    return cov[:n], (pc[:m] if pc is not None else None), cm, d


def dense_fisher(rec):
    N = rec.cams.shape[1] * rec.cams.shape[0] + 3 * rec.pts.shape[0]
    f = np.empty((N, N), order="F")
    err = OracleError()
    _check(lib().oracle_dense_fisher(C.byref(_scene(rec)), f.ctypes.data, C.byref(err)), err)
    return f


def pseudoinverse(rec, max_params=2000):
    n, P = rec.cams.shape[0], rec.cams.shape[1]
    N = P * n + 3 * rec.pts.shape[0]
    cov = np.empty((max(n, 1), P, P))
    sg = np.empty((N, N), order="F") if N <= max_params else None
    sv = np.empty(max(N, 1))
    gap = C.c_double()
    err = OracleError()
    _check(lib().oracle_pseudoinverse(C.byref(_scene(rec)), max_params, cov.ctypes.data,
                                      None if sg is None else sg.ctypes.data, sv.ctypes.data, C.byref(gap),
                                      C.byref(err)), err)
    return cov[:n], sg, sv[:N], gap.value


def exact_camera_blocks(rec, max_params=3000):
    """Camera blocks of the bordered Fisher inverse in long double (CPU truth
    for small scenes; validates the GPU's double-double refinement)."""
    n, P = rec.cams.shape[0], rec.cams.shape[1]
    cov = np.empty((max(n, 1), P, P))
    err = OracleError()
    _check(lib().oracle_exact_camera_blocks(C.byref(_scene(rec)), max_params, cov.ctypes.data, C.byref(err)), err)
    return cov[:n]


def cholesky_route(zp, n_cams, P, s_a_cams, blas_threads=1):
    zp = np.asfortranarray(zp, dtype=np.float64)
    sa = np.ascontiguousarray(s_a_cams, dtype=np.float64)
    cov = np.empty((n_cams, P, P))
    err = OracleError()
    _check(lib().oracle_cholesky_route(zp.ctypes.data, n_cams, P, sa.ctypes.data, blas_threads, cov.ctypes.data,
                                       C.byref(err)), err)
    return cov


def error_metric(gt, est, cams):
    """Eq. 42 of the paper (src/oracle.cpp:74-110): mean(sqrt|Δ| ⊘ O)/P²."""
    P = cams.shape[1]
    mean_abs = np.abs(cams).mean(axis=0)
    O = np.sqrt(np.outer(mean_abs, mean_abs))
    zero = [p for p in range(P) if mean_abs[p] == 0.0]
    for p in zero:
        O[p, :] = 1.0
        O[:, p] = 1.0
    per = np.array([(np.sqrt(np.abs(g - e)) / O).sum() / (P * P) for g, e in zip(gt, est)])
    srt = np.sort(per)
    n = len(per)
    median = srt[n // 2] if n % 2 else 0.5 * (srt[n // 2 - 1] + srt[n // 2])
    return per.mean(), median, per, zero
