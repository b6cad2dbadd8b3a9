"""Cholesky update order vs accuracy on config 2 (numpy): right-looking, left-looking, blocked; reference = long-double refinement."""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, scipy.linalg as sl
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
rec = S.generate_config(2)
P, n = rec.cam_params, rec.num_cameras(); N = P * n
zp = O.schur(rec)
Z, Gm, E = zp[:N, :N], zp[:N, N:], zp[N:, N:]
A0 = Z - Gm @ np.linalg.solve(E, Gm.T); A0 = 0.5 * (A0 + A0.T)
for m in (126, 252):
    A = A0[:m, :m].copy()
    X = np.linalg.inv(A).astype(np.longdouble); Al = A.astype(np.longdouble); I = np.eye(m, dtype=np.longdouble)
    for _ in range(2): X = X + X @ (I - Al @ X)
    truth = np.stack([np.asarray(X[P*i:P*i+P, P*i:P*i+P], dtype=np.float64) for i in range(m // P)])
    def blocks(L):
        Y = sl.solve_triangular(L, np.eye(L.shape[0]), lower=True)
        return np.stack([Y[:, P*i:P*i+P].T @ Y[:, P*i:P*i+P] for i in range(m // P)])
    print(m, "lapack L:", rel(blocks(np.linalg.cholesky(A)), truth))
    # unblocked right-looking with division
    T = np.tril(A.copy())
    for j in range(m):
        T[j, j] = np.sqrt(T[j, j]); T[j+1:, j] /= T[j, j]
        T[j+1:, j+1:] -= np.tril(np.outer(T[j+1:, j], T[j+1:, j]))
    print(m, "unblocked right-looking:", rel(blocks(np.tril(T)), truth))
    # left-looking (dot-product) Cholesky in long double -> exact-ish L rounded to double
    Ll = np.linalg.cholesky(A.astype(np.float64))
    Lx = np.linalg.cholesky(np.asarray(A, dtype=np.longdouble).astype(np.float64))
    # L from extended precision: Cholesky of longdouble matrix via manual
    Al2 = A.astype(np.longdouble); Le = np.zeros_like(Al2)
    for j in range(m):
        s = Al2[j, j] - np.dot(Le[j, :j], Le[j, :j]); Le[j, j] = np.sqrt(s)
        Le[j+1:, j] = (Al2[j+1:, j] - Le[j+1:, :j] @ Le[j, :j]) / Le[j, j]
    print(m, "L computed in long double, rounded:", rel(blocks(np.asarray(Le, dtype=np.float64)), truth))
    # left-looking in double (dot products)
    Ad = A.copy(); Ld = np.zeros_like(Ad)
    for j in range(m):
        s = Ad[j, j] - np.dot(Ld[j, :j], Ld[j, :j]); Ld[j, j] = np.sqrt(s)
        Ld[j+1:, j] = (Ad[j+1:, j] - Ld[j+1:, :j] @ Ld[j, :j]) / Ld[j, j]
    print(m, "left-looking double:", rel(blocks(Ld), truth))
    # right-looking with the update accumulated first then subtracted (delayed): per 8-block panel
    for nb in (8, 32, 128):
        T = np.tril(A.copy())
        for c0 in range(0, m, nb):
            c1 = min(c0 + nb, m)
            # left-looking within panel using all previous columns (dot form), i.e. blocked left-looking
            for j in range(c0, c1):
                s = T[j, j] - np.dot(T[j, :j], T[j, :j]) if False else None
            # blocked left-looking: update panel with all previous columns at once
            T[c0:, c0:c1] = np.tril(A[c0:, c0:c1], -c0) if False else T[c0:, c0:c1]
            upd = T[c0:, :c0] @ T[c0:c1, :c0].T
            T[c0:, c0:c1] = A[c0:, c0:c1] - upd
            for j in range(c0, c1):
                T[j, j] = np.sqrt(T[j, j]); T[j+1:, j] /= T[j, j]
                T[j+1:, j+1:c1] -= np.outer(T[j+1:, j], T[j+1:c1, j])
            T = np.tril(T)
        print(m, f"blocked left-looking nb={nb}:", rel(blocks(np.tril(T)), truth))
