"""Run one big BASELINE config end to end (timings, no oracle)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
cfg = int(sys.argv[1])
t0 = time.time(); rec = S.generate_config(cfg); print(f"gen {time.time()-t0:.1f}s", rec.cams.shape, rec.pts.shape, rec.obs_cam.shape, flush=True)
eng = F.Engine(0)
eng.set_profiling(True)
for it in range(2):
    t0 = time.time(); res = eng.compute_covariance(rec); dt = time.time() - t0
    print(f"e2e {dt:.3f}s", eng.counts(), flush=True)
    print({k: round(v, 2) for k, v in eng.stage_times().items()}, flush=True)
c = res.camera_cov
print("finite", np.isfinite(c).all(), "min diag", min(np.diag(b).min() for b in c), "sym", max(np.abs(b - b.T).max() / np.abs(b).max() for b in c), flush=True)
print("diag", res.diagnostics, flush=True)
