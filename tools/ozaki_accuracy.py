"""FP64 emulation by int8 slices (Ozaki scheme) inside the blocked Cholesky:
accuracy against plain FP64 (numpy, CPU; the go/no-go study of DESIGN §4).
usage: python tools/ozaki_accuracy.py CONFIG PANEL_WIDTH SLICES (e.g. 3 384 7,8,9)"""
import numpy as np, time, scipy.linalg as sl
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S
cfg = int(sys.argv[1]); W = int(sys.argv[2]); slices = [int(x) for x in sys.argv[3].split(',')]
rec = S.generate_config(cfg)
P, n = rec.cam_params, rec.num_cameras(); N = P * n
t=time.time(); zp = O.schur(rec, threads=16); print("schur", time.time()-t, flush=True)
Z, Gm, E = zp[:N, :N], zp[:N, N:], zp[N:, N:]
A0 = Z - Gm @ np.linalg.solve(E, Gm.T); A0 = 0.5 * (A0 + A0.T); del zp, Z
def split(M, s, bits=7):
    mx = np.abs(M).max(axis=1)
    e = np.where(mx > 0, np.ceil(np.log2(np.where(mx > 0, mx, 1))), 0)
    r = M * np.exp2(-e)[:, None]
    sl_ = []
    for t in range(1, s + 1):
        a = np.trunc(r * 2.0 ** (bits * t)); r = r - a * 2.0 ** (-bits * t); sl_.append(a)
    return e, sl_
def ozgemm(A, B, s, bits=7):
    ea, sa = split(A, s, bits); eb, sb = split(B, s, bits)
    acc = np.zeros((A.shape[0], B.shape[0]))
    for d in range(2, s + 2):
        g = np.zeros_like(acc)
        for t in range(1, d):
            u = d - t
            if t <= s and u <= s: g += sa[t-1] @ sb[u-1].T
        acc += g * 2.0 ** (-bits * d)
    return acc * np.exp2(ea)[:, None] * np.exp2(eb)[None, :]
def chol(A, gemm):
    T = np.tril(A)
    for c0 in range(0, N, W):
        c1 = min(c0 + W, N)
        L11 = np.linalg.cholesky(T[c0:c1, c0:c1]); T[c0:c1, c0:c1] = L11
        if c1 < N:
            T[c1:, c0:c1] = sl.solve_triangular(L11, T[c1:, c0:c1].T, lower=True).T
            Lp = T[c1:, c0:c1]
            T[c1:, c1:] -= np.tril(gemm(Lp, Lp))
    return np.tril(T)
def blocks(L):
    Y = sl.solve_triangular(L, np.eye(N), lower=True)
    return np.stack([Y[:, P*i:P*i+P].T @ Y[:, P*i:P*i+P] for i in range(n)])
t=time.time(); ref = blocks(chol(A0, lambda a, b: a @ b.T)); print("fp64", time.time()-t, flush=True)
for s in slices:
    t = time.time(); b = blocks(chol(A0, lambda a, b: ozgemm(a, b, s)))
    r = np.array([np.linalg.norm(b[i]-ref[i])/np.linalg.norm(ref[i]) for i in range(n)])
    print("ozaki s=%d vs fp64: worst %.3e median %.3e" % (s, r.max(), np.median(r)), time.time()-t, flush=True)
