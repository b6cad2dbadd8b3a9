"""Run the full pipeline on one BASELINE config a few times (profiling aid)."""
import sys, time
sys.path.insert(0, '.')
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rec = S.generate_config(cfg)
eng = F.Engine(0)
for _ in range(reps):
    t0 = time.time(); eng.compute_covariance(rec); print(f"e2e {time.time()-t0:.4f}s", flush=True)
