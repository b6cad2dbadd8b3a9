import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
import oracle.oracle as O
eng = F.Engine(0)
for cfg in [1, 2, 2, 2, 1, 2, 2]:
    rec = S.generate_config(cfg)
    H, _ = O.nullspace(rec)
    for rep in range(3):
        Hg = eng.gauge_nullspace(rec)
        d = np.abs(H - Hg); rows = np.nonzero(d.max(1))[0]
        print(cfg, rep, "nullspace rows differing", len(rows), rows[:10], d.max(), flush=True)
