import sys; sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import sfmcov as F
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
eng = F.Engine(0)
rng = np.random.default_rng(1)
for n in (128, 256, 1024, 4096):
    for cond in (1e1, 1e6):
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        ev = np.geomspace(1.0, cond, n)
        A = (Q * ev) @ Q.T
        A = 0.5 * (A + A.T)
        inv = np.linalg.inv(A)
        ref = np.stack([inv[8*i:8*i+8, 8*i:8*i+8] for i in range(n // 8)])
        g, _ = eng.spd_inverse_blocks(np.asfortranarray(A), 8)
        print(n, f"{cond:.0e}", "overall", rel(g, ref), "worst", max(rel(x, y) for x, y in zip(g, ref)), flush=True)
