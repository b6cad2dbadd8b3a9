"""Sparse (envelope) route study, S-transformation variant: M = Z + K K^T with a
rank-7 K on a cluster of cameras, (Z + G G^T)^-1 = P_G M^-1 P_G^T + N (G^T N)^-1 (N^T G)^-1 N^T
(N = S_c^-1 H_c, the analytic null basis), against the dense Cholesky route.
usage: python tools/sparse_route_stransform.py CONFIG CLUSTER_SIZE SCALE"""
import sys; sys.path.insert(0, '.')
import numpy as np, time, scipy.linalg as sl
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S
cfg = int(sys.argv[1]); q = int(sys.argv[2]) if len(sys.argv) > 2 else 16; scale = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
rec = S.generate_config(cfg)
P, n = rec.cam_params, rec.num_cameras(); N = P * n
zp = O.schur(rec, threads=8)
Z, Gm, E = zp[:N, :N].copy(), zp[:N, N:].copy(), zp[N:, N:].copy(); del zp
Z = 0.5*(Z+Z.T)
LF = np.linalg.cholesky(-E); G = np.linalg.solve(LF, Gm.T).T
H, _ = O.nullspace(rec); _, _, _, sa, sb, _ = O.fisher(rec)
Nc = H[:N] / sa[:N, None]
Zaug = Z + G @ G.T
Lz = np.linalg.cholesky(Zaug); del Zaug
Li = sl.solve_triangular(Lz, np.eye(N), lower=True); del Lz
ref = np.stack([Li[:, P*i:P*i+P].T @ Li[:, P*i:P*i+P] for i in range(n)]); del Li
def err(b):
    r = np.array([np.linalg.norm(b[i]-ref[i])/np.linalg.norm(ref[i]) for i in range(n)]); return r.max(), np.median(r)
cov = np.abs(Z).reshape(n, P, n, P).sum(axis=(1, 3))
c0 = int(np.argmax((cov > 0).sum(1)))
cl = [c0] + [int(j) for j in np.argsort(-cov[c0]) if j != c0][:q - 1]   # q = cluster size
Kall = np.zeros((N, 7))
for c in cl: Kall[P*c:P*c+P] = Nc[P*c:P*c+P]
Kall *= scale * np.sqrt(np.mean(np.diag(Z)[np.concatenate([np.arange(P*c, P*c+P) for c in cl])])) / np.sqrt(np.mean(np.sum(Kall*Kall, axis=0)))
M = Z + Kall @ Kall.T
L = np.linalg.cholesky(M); del M
Li = sl.solve_triangular(L, np.eye(N), lower=True)
Md = np.stack([Li[:, P*i:P*i+P].T @ Li[:, P*i:P*i+P] for i in range(n)]); del Li
Q = sl.cho_solve((L, True), G)          # M^-1 G
GN = G.T @ Nc                            # 7x7
GNi = np.linalg.inv(GN)
B = GNi @ Q.T                            # A M^-1 = (G^T N)^-1 G^T M^-1   (7 x N)
AMA = GNi @ (G.T @ Q) @ GNi.T            # A M^-1 A^T
W = GNi @ GNi.T                          # (G^T N)^-1 (N^T G)^-1
blocks = []
for i in range(n):
    sl_ = slice(P*i, P*i+P); Ni = Nc[sl_]; Bi = B[:, sl_]
    blocks.append(Md[i] - Ni @ Bi - Bi.T @ Ni.T + Ni @ (AMA + W) @ Ni.T)
blocks = np.stack(blocks)
ratio = np.max([np.linalg.norm(Md[i])/np.linalg.norm(ref[i]) for i in range(n)])
print(f"cfg {cfg} cluster {q} scale {scale}: max|M^-1_ii|/|S_ii| {ratio:.2e}, cond(G^T N) {np.linalg.cond(GN):.2e}, S-transform vs dense chol", err(blocks), flush=True)
