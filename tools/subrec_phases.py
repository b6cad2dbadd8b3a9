"""Phase times and throughput of approximate_covariances on config 3
(k_bar 100, 3 coverings); SFMCOV_SUBREC_TIMING=1 prints the phases,
SFMCOV_SUBREC_BATCH=0 selects the one-sub-scene-at-a-time path."""
import sys, time; sys.path.insert(0, '.')
from paper_1808_02414_b200 import synthetic as S, sfmcov as F, subrec as R
rec = S.generate_config(3); eng = F.Engine(0)
for w in (4,):
    R.approximate_covariances(rec, 100, 3, 7, workers=w, engine=eng)
    t0 = time.perf_counter(); a = R.approximate_covariances(rec, 100, 3, 7, workers=w, engine=eng); print("workers", w, time.perf_counter() - t0, flush=True)
