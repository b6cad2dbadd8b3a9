import sys, os
sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import sfmcov as F
eng = F.Engine(0)
rng = np.random.default_rng(0)
for n in [126, 270, 400, 1008]:
    M = rng.standard_normal((n, n)); A = M @ M.T / n + np.eye(n)
    blocks, piv = eng.spd_inverse_blocks(A, 9)
    Ai = np.linalg.inv(A)
    w = max(np.linalg.norm(blocks[i] - Ai[9*i:9*i+9, 9*i:9*i+9]) / np.linalg.norm(Ai[9*i:9*i+9, 9*i:9*i+9]) for i in range(n // 9))
    L = np.linalg.cholesky(A)
    print("G", os.environ.get("SFMCOV_PANEL"), "n", n, "worst", w, "piv", piv, (np.diag(L)**2).min(), (np.diag(L)**2).max(), flush=True)
