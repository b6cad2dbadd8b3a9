"""Dense-stage time of config 3 (profiling events) for the current env settings."""
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
rec = S.generate_config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
eng = F.Engine(0); eng.set_profiling(True)
ts = []
for i in range(6):
    try: eng.compute_covariance(rec)
    except Exception as e: pass
    st = eng.stage_times(); ts.append(st["cholesky"] + st["trtri"])
print("dense ms", np.median(ts[2:]))
