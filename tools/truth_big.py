"""Extended-precision truth for the camera blocks where FP64 routes disagree.

For a BASELINE config too large for a long-double inverse: the restatement's
bordered Schur matrix Z_p (one fixed FP64 matrix) is solved for the columns of
the selected cameras, X = Z_p^-1 [E_i; 0], by iterative refinement (LU solves
in FP64, residuals in 80-bit long double), then scaled by s_a like every route.
The GPU blocks (saved on the box by `compute_covariance`) and the two FP64
LAPACK routes of the restatement (dsytrf on Z_p, Cholesky on Z_aug) are
compared against it.

usage: python tools/truth_big.py CONFIG GPU_BLOCKS.npy [more.npy ...]
"""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import scipy.linalg as sl

from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S


def rel_blocks(a, b):
    return np.linalg.norm((a - b).reshape(len(a), -1), axis=1) / np.linalg.norm(b.reshape(len(b), -1), axis=1)


def residual_ld(zp, B, X):
    """B - zp @ X in 80-bit long double (tools/ldresid.c, OpenMP)."""
    so = "/tmp/sfmcov_ldresid.so"
    if not os.path.exists(so):
        src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ldresid.c")
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", so, src])
    lib = C.CDLL(so)
    lib.ld_residual.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_void_p, C.c_long, C.c_void_p]
    zp = np.asfortranarray(zp)
    X = np.asfortranarray(X, dtype=np.longdouble)
    B = np.asfortranarray(B, dtype=np.float64)
    out = np.empty(X.shape, dtype=np.longdouble, order="F")
    for j0 in range(0, X.shape[1], 64):  # the helper takes <= 64 columns
        x, b = np.asfortranarray(X[:, j0:j0 + 64]), np.asfortranarray(B[:, j0:j0 + 64])
        o = np.empty(x.shape, dtype=np.longdouble, order="F")
        lib.ld_residual(zp.ctypes.data, zp.shape[0], x.ctypes.data, b.ctypes.data, x.shape[1], o.ctypes.data)
        out[:, j0:j0 + 64] = o
    return out


def main():
    cfg = int(sys.argv[1])
    gpu = {os.path.basename(p): np.load(p) for p in sys.argv[2:]}
    cores = os.cpu_count() or 1
    rec = S.generate_config(cfg)
    P, n = rec.cam_params, rec.num_cameras()
    N = P * n
    O.lib().oracle_blas_threads(cores)
    t0 = time.time()
    dsy, _, _, _ = O.compute_covariance(rec, threads=cores)
    zp = O.schur(rec, threads=cores)
    sa = O.fisher(rec)[3][:N]
    chol = O.cholesky_route(zp, n, P, sa, cores)
    print(f"restatement routes {time.time() - t0:.0f} s", flush=True)
    routes = {"dsytrf": dsy, "cholesky": chol, **gpu}
    cams = set()
    names = list(routes)
    for i, a in enumerate(names):
        for b in names[i + 1:]:
            r = rel_blocks(routes[a], routes[b])
            cams.update(np.argsort(r)[-3:].tolist())
            print(f"{a} vs {b}: max {r.max():.3e}, blocks > 1e-9: {int((r > 1e-9).sum())}", flush=True)
    cams = sorted(cams)
    print("cameras", cams, flush=True)
    t0 = time.time()
    lu = sl.lu_factor(zp, overwrite_a=False, check_finite=False)
    B = np.zeros((N + 7, P * len(cams)))
    for k, c in enumerate(cams):
        B[P * c:P * c + P, P * k:P * k + P] = np.eye(P)
    X = sl.lu_solve(lu, B, check_finite=False).astype(np.longdouble)
    for it in range(3):
        r = residual_ld(zp, B, X)
        d = sl.lu_solve(lu, np.asarray(r, dtype=np.float64), check_finite=False)
        X = X + d.astype(np.longdouble)
        print(f"refinement {it}: |correction| / |X| = {np.abs(d).max() / float(np.abs(X).max()):.2e}", flush=True)
    print(f"truth {time.time() - t0:.0f} s", flush=True)
    truth = np.empty((len(cams), P, P))
    for k, c in enumerate(cams):
        blk = np.asarray(X[P * c:P * c + P, P * k:P * k + P], dtype=np.float64)
        s = sa[P * c:P * c + P]
        truth[k] = (s[:, None] * blk) * s[None, :]
    for name, v in routes.items():
        r = rel_blocks(v[cams], truth)
        print(f"{name:>16} vs truth: " + " ".join(f"{c}:{x:.1e}" for c, x in zip(cams, r)) + f"  max {r.max():.2e}",
              flush=True)


if __name__ == "__main__":
    main()
