"""Where the time of one small compute_covariance goes (a sub-scene of
config 3, k_bar = 100: N ~ 900): host wall time of the host-API call vs the
device stage times and the launch count."""
import sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F, subrec as R
rec = S.generate_config(3)
eng = F.Engine(0)
plan = R.plan_coverage(rec, 100, 7)
cams = plan[0]
m = np.isin(rec.obs_cam, cams); cnt = np.bincount(rec.obs_pt[m], minlength=rec.num_points())
sub = R.induced_scene(rec, cams, np.nonzero(cnt >= 2)[0].astype(np.int32))
print("sub-scene", sub.num_cameras(), sub.num_points(), sub.num_observations())
for prof in (False, True):
    eng.set_profiling(prof)
    for _ in range(3): eng.compute_covariance(sub)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); eng.compute_covariance(sub); ts.append(time.perf_counter() - t0)
    print("profiling" if prof else "plain", "wall ms median", 1e3 * float(np.median(ts)))
print({k: round(v, 3) for k, v in eng.stage_times().items()}, eng.counts()["kernel_launches"])
