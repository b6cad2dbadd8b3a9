"""Repeat the full pipeline to flush out nondeterminism / races."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rec = S.generate_config(cfg)
eng = F.Engine(0)
ref = eng.compute_covariance(rec).camera_cov
bad = 0
for i in range(reps):
    eng.set_profiling(i % 2 == 0)
    try:
        c = eng.compute_covariance(rec).camera_cov
        same = np.array_equal(c, ref)
        if not same:
            bad += 1
            print(i, "DIFFERENT", np.abs(c - ref).max(), flush=True)
    except Exception as e:
        bad += 1
        print(i, "ERROR", e, flush=True)
print("done", reps, "bad", bad)
