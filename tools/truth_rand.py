import sys; sys.path.insert(0, '.')
import numpy as np, scipy.linalg as sl
from paper_1808_02414_b200 import sfmcov as F
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
def worst(a, b): return max(rel(x, y) for x, y in zip(a, b))
eng = F.Engine(0); rng = np.random.default_rng(3)
for n, cond in ((128, 1e6), (512, 1e6), (1024, 1e8)):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (Q * np.geomspace(1.0, cond, n)) @ Q.T; A = 0.5 * (A + A.T)
    X = np.linalg.inv(A).astype(np.longdouble); Al = A.astype(np.longdouble); I = np.eye(n, dtype=np.longdouble)
    for _ in range(2): X = X + X @ (I - Al @ X)
    truth = np.stack([np.asarray(X[8*i:8*i+8, 8*i:8*i+8], dtype=np.float64) for i in range(n // 8)])
    c = sl.cho_factor(A, lower=True); inv = sl.cho_solve(c, np.eye(n))
    lap = np.stack([inv[8*i:8*i+8, 8*i:8*i+8] for i in range(n // 8)])
    g, _ = eng.spd_inverse_blocks(np.asfortranarray(A), 8)
    print(n, f"{cond:.0e}", "lapack", f"{rel(lap, truth):.2e}", "gpu", f"{rel(g, truth):.2e}", flush=True)
