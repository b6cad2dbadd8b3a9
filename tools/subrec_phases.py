import sys, time; sys.path.insert(0, '.')
from paper_1808_02414_b200 import synthetic as S, sfmcov as F, subrec as R
rec = S.generate_config(3); eng = F.Engine(0)
for w in (1, 4, 8, 16):
    R.approximate_covariances(rec, 100, 3, 7, workers=w, engine=eng)
    t0 = time.perf_counter(); R.approximate_covariances(rec, 100, 3, 7, workers=w, engine=eng); print("workers", w, time.perf_counter() - t0, flush=True)
