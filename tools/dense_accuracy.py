"""Isolates the dense stage's FP64 error on config 3: Z_aug = Z - Γ E^-1 Γ^T
from the restatement's bordered Schur matrix, inverse diagonal blocks by
LAPACK (scipy dpotrf/dpotri) vs the GPU spd_inverse_blocks (same kernels as
the pipeline)."""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, scipy.linalg as sl
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
def worst(a, b): return max(rel(x, y) for x, y in zip(a, b))
rec = S.generate_config(3)
P, n = rec.cam_params, rec.num_cameras(); N = P * n
zp = O.schur(rec)
Z, Gm, E = zp[:N, :N], zp[:N, N:], zp[N:, N:]
A = Z - Gm @ np.linalg.solve(E, Gm.T)
A = 0.5 * (A + A.T)
c, low = sl.cho_factor(A, lower=True)
inv = sl.cho_solve((c, low), np.eye(N))
ref = np.stack([inv[P*i:P*i+P, P*i:P*i+P] for i in range(n)])
# second CPU route: explicit inverse of L (dtrtri) then X^T X blocks
L = np.tril(c)
X = sl.lapack.dtrtri(L, lower=1)[0]
ref2 = np.stack([X[:, P*i:P*i+P].T @ X[:, P*i:P*i+P] for i in range(n)])
eng = F.Engine(0)
blocks, (mn, mx) = eng.spd_inverse_blocks(np.asfortranarray(A), P)
print("cho_solve vs dtrtri route: worst", worst(ref2, ref), "overall", rel(ref2, ref))
print("gpu vs cho_solve: worst", worst(blocks, ref), "overall", rel(blocks, ref))
print("gpu vs dtrtri route: worst", worst(blocks, ref2), "overall", rel(blocks, ref2))
print("cond estimate", np.linalg.cond(A) if N <= 9000 else None)
