"""Error vs an extended-precision reference on leading principal submatrices of
config 2's Z_aug: isolates the diagonal-tile kernel (n = 126 -> one tile)."""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, scipy.linalg as sl
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
rec = S.generate_config(2)
P, n = rec.cam_params, rec.num_cameras(); N = P * n
zp = O.schur(rec)
Z, Gm, E = zp[:N, :N], zp[:N, N:], zp[N:, N:]
A0 = Z - Gm @ np.linalg.solve(E, Gm.T); A0 = 0.5 * (A0 + A0.T)
eng = F.Engine(0)
for m in (126, 252, 504, 900):
    A = A0[:m, :m].copy(); nb = m // P
    X = np.linalg.inv(A).astype(np.longdouble); Al = A.astype(np.longdouble); I = np.eye(m, dtype=np.longdouble)
    for _ in range(2): X = X + X @ (I - Al @ X)
    truth = np.stack([np.asarray(X[P*i:P*i+P, P*i:P*i+P], dtype=np.float64) for i in range(nb)])
    c = sl.cho_factor(A, lower=True); inv = sl.cho_solve(c, np.eye(m))
    lap = np.stack([inv[P*i:P*i+P, P*i:P*i+P] for i in range(nb)])
    g, _ = eng.spd_inverse_blocks(np.asfortranarray(A), P)
    print(m, f"cond {np.linalg.cond(A):.1e}", "lapack", f"{rel(lap, truth):.2e}", "gpu", f"{rel(g, truth):.2e}", flush=True)
