"""Per-stage device times of compute_covariance on one BASELINE config (profiling aid).

usage: stage_probe.py CONFIG [REPS]   (env switches such as SFMCOV_PANEL / SFMCOV_RING apply)"""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rec = S.generate_config(cfg)
eng = F.Engine(0)
eng.set_profiling(True)
acc = {}
for r in range(reps):
    eng.compute_covariance(rec)
    if r == 0:
        continue
    for k, v in eng.stage_times().items():
        acc.setdefault(k, []).append(v)
tag = " ".join(f"{k}={os.environ[k]}" for k in sorted(os.environ) if k.startswith("SFMCOV_"))
tots = np.sum([v for v in acc.values()], axis=0)
ch = np.array(acc["cholesky"])
print(f"config {cfg} [{tag}] total min {tots.min():.3f} med {np.median(tots):.3f} max {tots.max():.3f} | "
      f"cholesky min {ch.min():.3f} med {np.median(ch):.3f} max {ch.max():.3f} | "
      + " ".join(f"{k} {np.median(v):.3f}" for k, v in acc.items() if k != "cholesky"), flush=True)
