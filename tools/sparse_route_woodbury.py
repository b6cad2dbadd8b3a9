"""Sparse (envelope) route study: the camera blocks of (Z + G G^T)^-1 through a
gauge-fixed M = Z + K K^T (K on anchor camera pairs) and the Woodbury
correction, against the dense Cholesky route (numpy, CPU).
usage: python tools/sparse_route_woodbury.py CONFIG SCALES ANCHOR_COUNTS (e.g. 3 0.3,1 4,16)"""
import sys; sys.path.insert(0, '.')
import numpy as np, time, scipy.linalg as sl
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S
cfg = int(sys.argv[1]); scales = [float(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else [1.0]
rec = S.generate_config(cfg)
P, n = rec.cam_params, rec.num_cameras(); N = P * n
t0=time.time()
zp = O.schur(rec, threads=8)
Z, Gm, E = zp[:N, :N].copy(), zp[:N, N:].copy(), zp[N:, N:].copy(); del zp
Z = 0.5*(Z+Z.T)
LF = np.linalg.cholesky(-E); G = np.linalg.solve(LF, Gm.T).T
H, _ = O.nullspace(rec)
_, _, _, sa, sb, _ = O.fisher(rec)
Hc = H[:N] / sa[:N, None]          # null(Z_s) = S_c^-1 H_c
print("setup", time.time()-t0, "|Z Hc| / |Z||Hc|", np.linalg.norm(Z @ Hc) / np.linalg.norm(Z) / np.linalg.norm(Hc), flush=True)
Zaug = Z + G @ G.T
t0=time.time()
Li = sl.solve_triangular(np.linalg.cholesky(Zaug), np.eye(N), lower=True)
ref = np.stack([Li[:, P*i:P*i+P].T @ Li[:, P*i:P*i+P] for i in range(n)]); del Li
print("dense ref", time.time()-t0, flush=True)
def err(b):
    r = np.array([np.linalg.norm(b[i]-ref[i])/np.linalg.norm(ref[i]) for i in range(n)]); return r.max(), np.median(r)
cov = np.abs(Z).reshape(n, P, n, P).sum(axis=(1, 3))
qs = [int(x) for x in sys.argv[3].split(',')] if len(sys.argv) > 3 else [1]
for q in qs:
  anchors = [int(round(x)) for x in np.linspace(0, n - 1, q + 2)[1:-1]]
  for scale in scales:
    Ks = []
    for c0 in anchors:
        c1 = [int(j) for j in np.argsort(-cov[c0]) if j != c0][0]
        K = np.zeros((N, 7))
        for c in (c0, c1): K[P*c:P*c+P] = Hc[P*c:P*c+P]
        K *= scale * np.sqrt(np.mean(np.diag(Z)[np.r_[P*c0:P*c0+P, P*c1:P*c1+P]])) / np.sqrt(np.mean(np.sum(K*K, axis=0)))
        Ks.append(K)
    Kall = np.hstack(Ks)
    M = Z + Kall @ Kall.T
    L = np.linalg.cholesky(M)
    Li = sl.solve_triangular(L, np.eye(N), lower=True)
    Mdiag = np.stack([Li[:, P*i:P*i+P].T @ Li[:, P*i:P*i+P] for i in range(n)]); del Li
    U = np.hstack([G, Kall]); Sg = np.diag([1.0]*7 + [-1.0]*(7*q))
    Y = sl.cho_solve((L, True), U)
    C = np.linalg.inv(Sg + U.T @ Y)
    blocks = np.stack([Mdiag[i] - Y[P*i:P*i+P] @ C @ Y[P*i:P*i+P].T for i in range(n)])
    ratio = np.max([np.linalg.norm(Mdiag[i])/np.linalg.norm(ref[i]) for i in range(n)])
    print(f"q {q} scale {scale}: max |M^-1_ii|/|Sigma_ii| {ratio:.2e}, cond(C) {np.linalg.cond(C):.2e}, woodbury vs dense chol", err(blocks), flush=True)
