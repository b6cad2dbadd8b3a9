import sys; sys.path.insert(0, '.')
import numpy as np, scipy.linalg as sl
from paper_1808_02414_b200 import sfmcov as F
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
eng = F.Engine(0); rng = np.random.default_rng(5)
def truth_blocks(A, P):
    m = A.shape[0]
    X = np.linalg.inv(A).astype(np.longdouble); Al = A.astype(np.longdouble); I = np.eye(m, dtype=np.longdouble)
    for _ in range(2): X = X + X @ (I - Al @ X)
    return np.stack([np.asarray(X[P*i:P*i+P, P*i:P*i+P], dtype=np.float64) for i in range(m // P)])
for m, cond, span in ((128, 1e4, 0), (128, 1e4, 3), (128, 1e4, 6), (512, 1e4, 3)):
    Q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    B = (Q * np.geomspace(1.0, cond, m)) @ Q.T
    d = 10.0 ** rng.uniform(-span / 2, span / 2, m) if span else np.ones(m)
    A = (d[:, None] * B) * d[None, :]; A = 0.5 * (A + A.T)
    truth = truth_blocks(A, 8)
    c = sl.cho_factor(A, lower=True); inv = sl.cho_solve(c, np.eye(m))
    lap = np.stack([inv[8*i:8*i+8, 8*i:8*i+8] for i in range(m // 8)])
    g, _ = eng.spd_inverse_blocks(np.asfortranarray(A), 8)
    print(m, f"cond {cond:.0e} span 1e{span}", "lapack", f"{rel(lap, truth):.2e}", "gpu", f"{rel(g, truth):.2e}", flush=True)
