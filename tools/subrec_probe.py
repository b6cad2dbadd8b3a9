import sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F, subrec as R
rec = S.generate_config(3); eng = F.Engine(0)
eng.set_profiling(True)
R.approximate_covariances(rec, 100, 3, 7, workers=4, engine=eng)
t0 = time.perf_counter(); a = R.approximate_covariances(rec, 100, 3, 7, workers=4, engine=eng); print("total", time.perf_counter() - t0, flush=True)
