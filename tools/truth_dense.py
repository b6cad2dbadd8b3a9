"""Accuracy of the dense stage alone at a BASELINE size: the GPU's
Cholesky + triangular inverse + block extraction (`spd_inverse_blocks`) and
LAPACK's Cholesky on ONE fixed SPD matrix Z_aug (formed from the restatement's
Z_p), against the extended-precision truth of that matrix for a few cameras
(iterative refinement with long-double residuals, tools/ldresid.c).

usage: python tools/truth_dense.py CONFIG CAM [CAM ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import scipy.linalg as sl

from oracle import oracle as O
from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import synthetic as S
from truth_big import residual_ld


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def main():
    cfg, cams = int(sys.argv[1]), [int(c) for c in sys.argv[2:]]
    cores = os.cpu_count() or 1
    rec = S.generate_config(cfg)
    P, n = rec.cam_params, rec.num_cameras()
    N = P * n
    t0 = time.time()
    zp = O.schur(rec, threads=cores)
    Z, Gm, E = zp[:N, :N], zp[:N, N:], zp[N:, N:]
    A = Z - Gm @ np.linalg.solve(E, Gm.T)
    del zp, Z
    A = np.asfortranarray(0.5 * (A + A.T))
    print(f"Z_aug formed ({time.time() - t0:.0f} s)", flush=True)
    eng = F.Engine(0)
    t0 = time.time()
    g, _ = eng.spd_inverse_blocks(A, P)
    print(f"gpu spd_inverse_blocks {time.time() - t0:.1f} s", flush=True)
    B = np.zeros((N, P * len(cams)))
    for k, c in enumerate(cams):
        B[P * c:P * c + P, P * k:P * k + P] = np.eye(P)
    t0 = time.time()
    ch = sl.cho_factor(A, lower=True, check_finite=False)
    X0 = sl.cho_solve(ch, B, check_finite=False)
    X = X0.astype(np.longdouble)
    for it in range(3):
        d = sl.cho_solve(ch, np.asarray(residual_ld(A, B, X), dtype=np.float64), check_finite=False)
        X = X + d.astype(np.longdouble)
        print(f"refinement {it}: |correction| / |X| = {np.abs(d).max() / float(np.abs(X).max()):.2e}", flush=True)
    print(f"truth {time.time() - t0:.0f} s", flush=True)
    for k, c in enumerate(cams):
        t = np.asarray(X[P * c:P * c + P, P * k:P * k + P], dtype=np.float64)
        lap = X0[P * c:P * c + P, P * k:P * k + P]
        print(f"camera {c}: lapack cholesky {rel(lap, t):.2e}  gpu {rel(g[c], t):.2e}", flush=True)


if __name__ == "__main__":
    main()
