"""Accuracy against an extended-precision reference on a small config: the
inverse diagonal blocks of Z_aug refined with Newton steps in long double."""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, scipy.linalg as sl
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
def worst(a, b): return max(rel(x, y) for x, y in zip(a, b))
rec = S.generate_config(int(sys.argv[1]))
P, n = rec.cam_params, rec.num_cameras(); N = P * n
zp = O.schur(rec)
Z, Gm, E = zp[:N, :N], zp[:N, N:], zp[N:, N:]
A = Z - Gm @ np.linalg.solve(E, Gm.T); A = 0.5 * (A + A.T)
X = np.linalg.inv(A).astype(np.longdouble); Al = A.astype(np.longdouble); I = np.eye(N, dtype=np.longdouble)
for _ in range(2):
    X = X + X @ (I - Al @ X)
truth = np.stack([np.asarray(X[P*i:P*i+P, P*i:P*i+P], dtype=np.float64) for i in range(n)])
c = sl.cho_factor(A, lower=True); inv = sl.cho_solve(c, np.eye(N))
lap = np.stack([inv[P*i:P*i+P, P*i:P*i+P] for i in range(n)])
eng = F.Engine(0)
g, _ = eng.spd_inverse_blocks(np.asfortranarray(A), P)
print("cond", np.linalg.cond(A))
print("lapack vs truth: worst", worst(lap, truth), "overall", rel(lap, truth))
print("gpu vs truth:    worst", worst(g, truth), "overall", rel(g, truth))
