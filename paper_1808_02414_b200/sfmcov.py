"""Python mirror of the reference ``sfmcov`` operator API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference free
functions in namespace ``sfmcov`` (include/sfmcov/*.hpp); every call runs on
the GPU through ``libsfmcov_b200.so`` (include/sfmcov_b200.h).  Scenes are
structure-of-arrays numpy buffers instead of the reference's Eigen AoS.

    reference (C++)                         this module
    ------------------------------------    -----------------------------------
    Reconstruction (types.hpp:52-66)        Reconstruction
    build_observation_index (scene.cpp:80)  build_observation_index
    assemble_jacobian (projection.hpp:54)   assemble_jacobian
    gauge_nullspace (nullspace.hpp:33)      gauge_nullspace
    build_fisher_blocks + condition_columns build_fisher_blocks
      (covariance.hpp:80-86)
    schur_reduce (covariance.hpp:94-95)     schur_reduce
    compute_covariance (covariance.hpp:110) compute_covariance
    Error / ErrorKind (error.hpp)           Error / ErrorKind
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional

import numpy as np

from . import _native as N

K_GAUGE = 7


class ErrorKind(IntEnum):
    io = 1
    parse = 2
    invariant = 3
    degenerate = 4
    dimension = 5
    size_guard = 6
    device = 7


class Error(RuntimeError):
    """sfmcov::Error: ``str(e)`` is "stage: message" like Error::what()."""

    def __init__(self, kind: int, stage: str, what: str):
        super().__init__(what)
        self.kind = ErrorKind(kind)
        self.stage = stage


def _raise(code: int, err: N.ErrorStruct):
    if code:
        raise Error(code, err.stage.decode(), err.message.decode())


@dataclass
class Reconstruction:
    """Scene of cameras, points and observations (SoA).

    cams: (n, P) float64, P = 8 (r, C, c, k) or 9 (r, C, f, k1, k2)
    pts: (m, 3); obs_cam / obs_pt: (t,) int32; obs_u: (t, 2);
    obs_sigma: (t, 2, 2) observation covariance or None (= identity).
    """

    cams: np.ndarray
    pts: np.ndarray
    obs_cam: np.ndarray
    obs_pt: np.ndarray
    obs_u: Optional[np.ndarray] = None
    obs_sigma: Optional[np.ndarray] = None

    def __post_init__(self):
        self.cams = np.ascontiguousarray(self.cams, dtype=np.float64)
        self.pts = np.ascontiguousarray(self.pts, dtype=np.float64).reshape(-1, 3)
        self.obs_cam = np.ascontiguousarray(self.obs_cam, dtype=np.int32)
        self.obs_pt = np.ascontiguousarray(self.obs_pt, dtype=np.int32)
        if self.cams.ndim != 2:
            self.cams = self.cams.reshape(-1, 8)
        if self.obs_u is not None:
            self.obs_u = np.ascontiguousarray(self.obs_u, dtype=np.float64).reshape(-1, 2)
        if self.obs_sigma is not None:
            self.obs_sigma = np.ascontiguousarray(self.obs_sigma, dtype=np.float64).reshape(-1, 2, 2)

    @property
    def cam_params(self) -> int:
        return int(self.cams.shape[1])

    def num_cameras(self) -> int:
        return int(self.cams.shape[0])

    def num_points(self) -> int:
        return int(self.pts.shape[0])

    def num_observations(self) -> int:
        return int(self.obs_cam.shape[0])

    def num_parameters(self) -> int:
        return self.cam_params * self.num_cameras() + 3 * self.num_points()

    def copy(self) -> "Reconstruction":
        return Reconstruction(self.cams.copy(), self.pts.copy(), self.obs_cam.copy(), self.obs_pt.copy(),
                              None if self.obs_u is None else self.obs_u.copy(),
                              None if self.obs_sigma is None else self.obs_sigma.copy())

    def c_struct(self) -> N.Scene:
        s = N.Scene()
        s.n_cams, s.n_pts, s.n_obs = self.num_cameras(), self.num_points(), self.num_observations()
        s.cam_params = self.cam_params
        s.cams, s.pts = N.ptr(self.cams), N.ptr(self.pts)
        s.obs_cam, s.obs_pt = N.ptr(self.obs_cam), N.ptr(self.obs_pt)
        s.obs_u = N.ptr(self.obs_u)
        s.obs_sigma = N.ptr(self.obs_sigma)
        return s

    # the reference validates inside compute_covariance; exposed for parity
    def validate(self) -> None:
        build_observation_index(self)


@dataclass
class CovarianceOptions:
    threads: int = 0  # accepted, ignored: results never depend on it
    point_covariances: bool = False
    camera_cross_covariances: bool = False


@dataclass
class CovarianceDiagnostics:
    scale_min: float = 0.0
    scale_max: float = 0.0
    flagged_columns: List[int] = field(default_factory=list)
    min_pivot: float = 0.0
    max_pivot: float = 0.0
    inertia_positive: int = 0
    inertia_negative: int = 0
    negative_eigenvalue_warnings: int = 0
    peak_dense_bytes: int = 0
    largest_dense_dim: int = 0


@dataclass
class CovarianceResult:
    camera_cov: np.ndarray  # (n, P, P)
    diagnostics: CovarianceDiagnostics
    point_cov: Optional[np.ndarray] = None      # (m, 3, 3) when options.point_covariances
    camera_matrix: Optional[np.ndarray] = None  # (P n, P n) when options.camera_cross_covariances

    def cross_block(self, i: int, j: int) -> np.ndarray:
        P = self.camera_cov.shape[1]
        return self.camera_matrix[P * i:P * i + P, P * j:P * j + P]


@dataclass
class ObservationIndex:
    off_cam: np.ndarray
    idx_cam: np.ndarray
    off_pt: np.ndarray
    idx_pt: np.ndarray

    @property
    def by_camera(self):
        return [self.idx_cam[self.off_cam[i]:self.off_cam[i + 1]] for i in range(len(self.off_cam) - 1)]

    @property
    def by_point(self):
        return [self.idx_pt[self.off_pt[j]:self.off_pt[j + 1]] for j in range(len(self.off_pt) - 1)]


@dataclass
class SparseJacobian:
    cam_index: np.ndarray
    point_index: np.ndarray
    cam_blocks: np.ndarray    # (t, 2, P)
    point_blocks: np.ndarray  # (t, 2, 3)
    n_cams: int
    n_pts: int

    def cols(self) -> int:
        return self.cam_blocks.shape[2] * self.n_cams + 3 * self.n_pts

    def dense(self) -> np.ndarray:
        P = self.cam_blocks.shape[2]
        t = self.cam_blocks.shape[0]
        J = np.zeros((2 * t, self.cols()))
        for k in range(t):
            ci, pj = self.cam_index[k], self.point_index[k]
            J[2 * k:2 * k + 2, P * ci:P * ci + P] = self.cam_blocks[k]
            c0 = P * self.n_cams + 3 * pj
            J[2 * k:2 * k + 2, c0:c0 + 3] = self.point_blocks[k]
        return J

    def max_abs(self) -> float:
        return float(max(np.abs(self.cam_blocks).max(initial=0.0), np.abs(self.point_blocks).max(initial=0.0)))


@dataclass
class FisherBlocks:
    cam_blocks: np.ndarray    # (n, P, P)  M[P_i, P_i]
    point_blocks: np.ndarray  # (m, 3, 3)  M[X_j, X_j]
    couplings: np.ndarray     # (t, P, 3)  M[P_i, X_j], observation order
    s_a: np.ndarray
    s_b: np.ndarray
    flagged: List[int]


class Engine:
    """One CUDA handle (device, stream, workspace).  Thread-safe."""

    def __init__(self, device: int = 0):
        lib = N.cuda_lib()
        err = N.ErrorStruct()
        h = lib.sfmcov_cuda_create(device, C.byref(err))
        if not h:
            raise Error(err.kind or ErrorKind.device, err.stage.decode() or "device", err.message.decode())
        self._h = h
        self._lib = lib
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._lib.sfmcov_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return self._lib.sfmcov_cuda_stream(self._h) or 0

    def set_sharded_stage_a(self, on: bool):
        """Multi-GPU stage A point-sharded (True) or replicated on every rank (False, default)."""
        self._lib.sfmcov_cuda_set_sharded_stage_a(self._h, 1 if on else 0)

    def set_profiling(self, on: bool):
        self._lib.sfmcov_cuda_set_profiling(self._h, 1 if on else 0)

    def stage_times(self) -> dict:
        buf = (C.c_double * 16)()
        k = self._lib.sfmcov_cuda_last_stage_times(self._h, buf, 16)
        return {self._lib.sfmcov_cuda_stage_name(i).decode(): buf[i] for i in range(k)}

    def counts(self) -> dict:
        buf = (C.c_int64 * 10)()
        self._lib.sfmcov_cuda_last_counts(self._h, buf, 10)
        keys = ["obs_pairs", "nnz_blocks", "N", "Npad", "n_obs", "n_pts", "n_cams", "P", "kernel_launches",
                "reserved"]
        return dict(zip(keys, [int(v) for v in buf]))

    # ---- pipeline -------------------------------------------------------------
    def _covariance_call(self, fn, rec: Reconstruction, options: Optional[CovarianceOptions], *extra, reorder=False):
        options = options or CovarianceOptions()
        P, n = rec.cam_params, rec.num_cameras()
        out = np.empty((n, P, P))
        flagged = np.zeros(max(1, rec.num_parameters()), dtype=np.int64)
        diag = N.Diagnostics()
        diag.flagged = flagged.ctypes.data_as(N.c_int64_p)
        diag.flagged_capacity = flagged.size
        opts = N.Options(options.threads, int(options.point_covariances), int(options.camera_cross_covariances), 0)
        err = N.ErrorStruct()
        sc = rec.c_struct()
        if reorder:  # (h, scene, opts, cam_cov, *extra outputs, diag, err)
            code = fn(self._h, C.byref(sc), C.byref(opts), out.ctypes.data, *extra, C.byref(diag), C.byref(err))
        else:
            code = fn(self._h, C.byref(sc), C.byref(opts), *extra, out.ctypes.data, C.byref(diag), C.byref(err))
        _raise(code, err)
        d = CovarianceDiagnostics(diag.scale_min, diag.scale_max, [int(v) for v in flagged[:diag.n_flagged]],
                                  diag.min_pivot, diag.max_pivot, diag.inertia_positive, diag.inertia_negative,
                                  diag.negative_eigenvalue_warnings, diag.peak_dense_bytes, diag.largest_dense_dim)
        return CovarianceResult(out, d)

    # ---- pipeline -------------------------------------------------------------
    def compute_covariance(self, rec: Reconstruction, options: Optional[CovarianceOptions] = None) -> CovarianceResult:
        options = options or CovarianceOptions()
        if not (options.point_covariances or options.camera_cross_covariances):
            return self._covariance_call(self._lib.sfmcov_cuda_compute_covariance, rec, options)
        P, n, m = rec.cam_params, rec.num_cameras(), rec.num_points()
        pc = np.empty((m, 3, 3)) if options.point_covariances else None
        cm = np.empty((P * n, P * n), order="F") if options.camera_cross_covariances else None
        res = self._covariance_call(self._lib.sfmcov_cuda_compute_covariance_full, rec, options,
                                    None if pc is None else pc.ctypes.data, None if cm is None else cm.ctypes.data,
                                    reorder=True)
        res.point_cov, res.camera_matrix = pc, cm
        return res

    # ---- multi-GPU -------------------------------------------------------------
    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """Attach this handle to rank `rank` of `nranks` (NCCL, one process per GPU)."""
        err = N.ErrorStruct()
        _raise(self._lib.sfmcov_cuda_comm_init(self._h, bytes(unique_id), nranks, rank, C.byref(err)), err)

    def compute_covariance_sharded(self, rec: Reconstruction,
                                   options: Optional[CovarianceOptions] = None) -> CovarianceResult:
        """The multi-GPU pipeline (call on every rank with the same scene)."""
        return self._covariance_call(self._lib.sfmcov_cuda_compute_covariance_sharded, rec, options)

    def compute_covariance_emulated(self, rec: Reconstruction, ranks: int,
                                    options: Optional[CovarianceOptions] = None) -> CovarianceResult:
        """The multi-GPU code path with `ranks` ranks emulated on this device."""
        return self._covariance_call(self._lib.sfmcov_cuda_compute_covariance_emulated, rec, options, ranks)

    def build_observation_index(self, rec: Reconstruction) -> ObservationIndex:
        n, m, t = rec.num_cameras(), rec.num_points(), rec.num_observations()
        oc, op = np.empty(n + 1, np.int64), np.empty(m + 1, np.int64)
        ic, ip = np.empty(max(t, 1), np.int32), np.empty(max(t, 1), np.int32)
        err = N.ErrorStruct()
        sc = rec.c_struct()
        code = self._lib.sfmcov_cuda_observation_index(self._h, C.byref(sc), oc.ctypes.data, ic.ctypes.data,
                                                        op.ctypes.data, ip.ctypes.data, C.byref(err))
        _raise(code, err)
        return ObservationIndex(oc, ic[:t], op, ip[:t])

    def assemble_jacobian(self, rec: Reconstruction) -> SparseJacobian:
        P, t = rec.cam_params, rec.num_observations()
        jc = np.empty((max(t, 1), 2, P))
        jp = np.empty((max(t, 1), 2, 3))
        err = N.ErrorStruct()
        sc = rec.c_struct()
        code = self._lib.sfmcov_cuda_jacobian(self._h, C.byref(sc), jc.ctypes.data, jp.ctypes.data, C.byref(err))
        _raise(code, err)
        return SparseJacobian(rec.obs_cam.copy(), rec.obs_pt.copy(), jc[:t], jp[:t], rec.num_cameras(),
                              rec.num_points())

    def gauge_nullspace(self, rec: Reconstruction) -> np.ndarray:
        H = np.empty((max(rec.num_parameters(), 1), K_GAUGE))
        err = N.ErrorStruct()
        sc = rec.c_struct()
        code = self._lib.sfmcov_cuda_nullspace(self._h, C.byref(sc), H.ctypes.data, C.byref(err))
        _raise(code, err)
        return H[:rec.num_parameters()]

    def build_fisher_blocks(self, rec: Reconstruction) -> FisherBlocks:
        P, n, m, t = rec.cam_params, rec.num_cameras(), rec.num_points(), rec.num_observations()
        D = np.empty((max(n, 1), P, P))
        A = np.empty((max(m, 1), 3, 3))
        Cp = np.empty((max(t, 1), P, 3))
        sa = np.empty(max(rec.num_parameters(), 1))
        sb = np.empty(K_GAUGE)
        flagged = np.zeros(max(1, rec.num_parameters()), dtype=np.int64)
        diag = N.Diagnostics()
        diag.flagged = flagged.ctypes.data_as(N.c_int64_p)
        diag.flagged_capacity = flagged.size
        err = N.ErrorStruct()
        sc = rec.c_struct()
        code = self._lib.sfmcov_cuda_fisher(self._h, C.byref(sc), D.ctypes.data, A.ctypes.data, Cp.ctypes.data,
                                            sa.ctypes.data, sb.ctypes.data, C.byref(diag), C.byref(err))
        _raise(code, err)
        return FisherBlocks(D[:n], A[:m], Cp[:t], sa[:rec.num_parameters()], sb,
                            [int(v) for v in flagged[:diag.n_flagged]])

    def schur_reduce(self, rec: Reconstruction) -> np.ndarray:
        dim = rec.cam_params * rec.num_cameras() + K_GAUGE
        z = np.empty((dim, dim), order="F")
        err = N.ErrorStruct()
        sc = rec.c_struct()
        code = self._lib.sfmcov_cuda_schur(self._h, C.byref(sc), z.ctypes.data, C.byref(err))
        _raise(code, err)
        return z

    def pseudoinverse_covariance(self, rec: Reconstruction, max_params: int = 2000, full: bool = True):
        """Dense reference covariance (oracle.hpp:33-37) on the GPU: returns
        (camera_cov (n,P,P), sigma_full (N,N) or None, singular values (N,), gauge gap)."""
        P, n = rec.cam_params, rec.num_cameras()
        npar = rec.num_parameters()
        cov = np.empty((max(1, n), P, P))
        sg = np.empty((npar, npar), order="F") if full and npar <= max_params else None
        sv = np.empty(max(1, npar))
        gap = C.c_double()
        err = N.ErrorStruct()
        sc = rec.c_struct()
        code = self._lib.sfmcov_cuda_pseudoinverse_covariance(self._h, C.byref(sc), max_params, cov.ctypes.data,
                                                              None if sg is None else sg.ctypes.data, sv.ctypes.data,
                                                              C.byref(gap), C.byref(err))
        _raise(code, err)
        return cov[:n], sg, sv[:npar], gap.value

    def nullspace_residual(self, rec: Reconstruction, H: np.ndarray) -> float:
        """max |J H| / (max |J| max |H|) (nullspace.hpp:36) with J formed on the GPU."""
        H = np.ascontiguousarray(H, dtype=np.float64)
        out = C.c_double()
        err = N.ErrorStruct()
        sc = rec.c_struct()
        _raise(self._lib.sfmcov_cuda_nullspace_residual(self._h, C.byref(sc), H.ctypes.data, H.shape[1], C.byref(out),
                                                        C.byref(err)), err)
        return out.value

    def invert_schur(self, z: np.ndarray):
        """invert_schur (covariance.hpp:100) of any symmetric nonsingular matrix:
        returns (z_inv, (min_pivot, max_pivot), (inertia_positive, inertia_negative))."""
        z = np.asfortranarray(z, dtype=np.float64)
        if z.ndim != 2 or z.shape[0] != z.shape[1] or z.shape[0] < 1:
            raise Error(ErrorKind.dimension, "factorization", "matrix must be square")
        n = z.shape[0]
        out = np.empty((n, n), order="F")
        mn, mx = C.c_double(), C.c_double()
        ip, ineg = C.c_int32(), C.c_int32()
        err = N.ErrorStruct()
        _raise(self._lib.sfmcov_cuda_invert_symmetric(self._h, z.ctypes.data, n, out.ctypes.data, C.byref(mn),
                                                      C.byref(mx), C.byref(ip), C.byref(ineg), C.byref(err)), err)
        return out, (mn.value, mx.value), (ip.value, ineg.value)

    def full_covariance(self, rec: Reconstruction, max_params: int = 2000) -> np.ndarray:
        """full_covariance (covariance.hpp:115): the (Pn+3m)^2 parameter covariance."""
        npar = rec.num_parameters()
        if npar > max_params:
            raise Error(ErrorKind.size_guard, "full-covariance",
                        f"scene has {npar} parameters, guard is {max_params}")
        sig = np.empty((npar, npar), order="F")
        err = N.ErrorStruct()
        sc = rec.c_struct()
        _raise(self._lib.sfmcov_cuda_full_covariance(self._h, C.byref(sc), max_params, sig.ctypes.data, C.byref(err)),
               err)
        return sig

    def refine_covariance(self, rec: Reconstruction, cams, iters: int = 3):
        """Verification: the selected cameras' blocks refined against the exact
        inverse of the bordered Fisher system (double-double residuals; see
        include/sfmcov_b200.h).  Returns (refined (k,P,P), product blocks
        (k,P,P), per-step max relative change (iters,))."""
        P = rec.cam_params
        sel = np.ascontiguousarray(cams, dtype=np.int32)
        k = len(sel)
        ref = np.empty((max(1, k), P, P))
        base = np.empty((max(1, k), P, P))
        hist = np.empty(iters)
        err = N.ErrorStruct()
        sc = rec.c_struct()
        code = self._lib.sfmcov_cuda_refine_covariance(self._h, C.byref(sc), sel.ctypes.data, k, iters, ref.ctypes.data,
                                                       base.ctypes.data, hist.ctypes.data, C.byref(err))
        _raise(code, err)
        return ref[:k], base[:k], hist

    def spd_inverse_blocks(self, a: np.ndarray, block: int):
        a = np.asfortranarray(a, dtype=np.float64)
        n = a.shape[0]
        out = np.empty((n // block, block, block))
        mn, mx = C.c_double(), C.c_double()
        err = N.ErrorStruct()
        code = self._lib.sfmcov_cuda_spd_inverse_blocks(self._h, a.ctypes.data, n, block, out.ctypes.data,
                                                        C.byref(mn), C.byref(mx), C.byref(err))
        _raise(code, err)
        return out, (mn.value, mx.value)


_default = None
_default_lock = threading.Lock()


def default_engine() -> Engine:
    global _default
    with _default_lock:
        if _default is None:
            _default = Engine(0)
        return _default


def compute_covariance(rec: Reconstruction, options: Optional[CovarianceOptions] = None) -> CovarianceResult:
    return default_engine().compute_covariance(rec, options)


def build_observation_index(rec: Reconstruction) -> ObservationIndex:
    return default_engine().build_observation_index(rec)


def assemble_jacobian(rec: Reconstruction, threads: int = 1) -> SparseJacobian:
    return default_engine().assemble_jacobian(rec)


def gauge_nullspace(rec: Reconstruction) -> np.ndarray:
    return default_engine().gauge_nullspace(rec)


def build_fisher_blocks(rec: Reconstruction) -> FisherBlocks:
    return default_engine().build_fisher_blocks(rec)


def schur_reduce(rec: Reconstruction) -> np.ndarray:
    return default_engine().schur_reduce(rec)


def spd_inverse_blocks(a: np.ndarray, block: int):
    return default_engine().spd_inverse_blocks(a, block)


# ---- multi-GPU helpers (host only) ----------------------------------------------
def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (rank 0 creates it, the caller distributes it)."""
    buf = C.create_string_buffer(128)
    err = N.ErrorStruct()
    _raise(N.cuda_lib().sfmcov_nccl_unique_id(buf, C.byref(err)), err)
    return buf.raw


def plan_dense(n_cams: int, cam_params: int, nranks: int, rank: int, panel_blocks: int = 3):
    """(padded dimension, local column count, cameras whose blocks this rank extracts)."""
    npad, ncols = C.c_int64(), C.c_int64()
    owned = np.zeros(max(1, n_cams), dtype=np.int32)
    code = N.cuda_lib().sfmcov_plan_dense(n_cams, cam_params, nranks, rank, panel_blocks, C.byref(npad),
                                          C.byref(ncols), owned.ctypes.data)
    if code:
        raise Error(code, "options", "invalid plan arguments")
    return npad.value, ncols.value, owned[:n_cams].astype(bool)


def plan_chunks(nchunks: int, nranks: int, rank: int):
    """Half-open chunk range [begin, end) of the sorted pair list owned by `rank`."""
    b, e = C.c_int64(), C.c_int64()
    code = N.cuda_lib().sfmcov_plan_chunks(nchunks, nranks, rank, C.byref(b), C.byref(e))
    if code:
        raise Error(code, "options", "invalid plan arguments")
    return b.value, e.value


# ---- Eq. 42 error metric (include/sfmcov/oracle.hpp:39-50, src/oracle.cpp:74-110) ---
@dataclass
class ErrorReport:
    per_camera: np.ndarray
    normalization: np.ndarray  # O, strictly positive after the fallback
    mean: float
    median: float
    zero_components: List[int]


def error_metric(gt: np.ndarray, est: np.ndarray, rec: Reconstruction) -> ErrorReport:
    """Per camera: mean over the P^2 block entries of sqrt|gt - est| divided
    element-wise by O = sqrt(e e^T), e the component-wise mean of |camera
    parameter| over the scene (zero components fall back to 1)."""
    n, P = rec.num_cameras(), rec.cam_params
    gt, est = np.asarray(gt), np.asarray(est)
    if gt.shape[0] != n or est.shape[0] != n:
        raise Error(ErrorKind.dimension, "error-metric", "covariance lists must have one block per camera")
    e = np.abs(rec.cams).mean(axis=0)
    zero = [p for p in range(P) if e[p] == 0.0]
    e = np.where(e == 0.0, 1.0, e)
    O = np.sqrt(np.outer(e, e))
    per = np.array([(np.sqrt(np.abs(g - x)) / O).sum() / (P * P) for g, x in zip(gt, est)])
    srt = np.sort(per)
    mean = float(srt.sum() / n) if n else 0.0
    median = float(srt[n // 2] if n % 2 else 0.5 * (srt[n // 2 - 1] + srt[n // 2])) if n else 0.0
    return ErrorReport(per, O, mean, median, zero)

