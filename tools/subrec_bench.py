"""Batched sub-reconstruction covariances (approximate_covariances) on config N,
k_bar 100, 3 coverings: throughput (best of 3 timed calls after a warm-up)
and the reference's serial cost (the restatement on one sub-scene, 1 thread)."""
import sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F, subrec as R
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
k_bar = int(sys.argv[2]) if len(sys.argv) > 2 else 100
rec = S.generate_config(cfg)
eng = F.Engine(0)
plans = [R.plan_coverage(rec, k_bar, 7 + d) for d in range(3)]
nsub = sum(len(p) for p in plans)
sizes = [len(c) for p in plans for c in p]
print(f"config {cfg}: k_bar {k_bar}, 3 decompositions -> {nsub} subsets, mean {np.mean(sizes):.1f} cameras (N ~ {9*np.mean(sizes):.0f})")
R.approximate_covariances(rec, k_bar, 3, 7, workers=4, engine=eng)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); R.approximate_covariances(rec, k_bar, 3, 7, workers=4, engine=eng); ts.append(time.perf_counter() - t0)
dt = min(ts)
print(f"approximate_covariances: {dt:.3f} s ({nsub / dt:.1f} sub-scenes/s; runs {', '.join(f'{t:.3f}' for t in ts)})")
from oracle import oracle as O
cams = plans[0][0]
m = np.isin(rec.obs_cam, cams); cnt = np.bincount(rec.obs_pt[m], minlength=rec.num_points())
sub = R.induced_scene(rec, cams, np.nonzero(cnt >= 2)[0].astype(np.int32))
O.lib().oracle_blas_threads(1)
t0 = time.perf_counter(); O.compute_covariance(sub); dt1 = time.perf_counter() - t0
print(f"restatement, one sub-scene, 1 thread (the reference's pinned BLAS): {dt1:.3f} s -> {nsub * dt1:.1f} s for all")
# Multi-GPU job sharding: each rank's share timed alone on this one GPU
# (the shares are independent; the slowest one bounds an R-GPU run).
for nr in (2, 4, 8):
    per = []
    for r in range(nr):
        R.approximate_covariances_shard(rec, k_bar, 3, 7, nr, r, workers=4, engine=eng)
        t0 = time.perf_counter(); R.approximate_covariances_shard(rec, k_bar, 3, 7, nr, r, workers=4, engine=eng)
        per.append(time.perf_counter() - t0)
    print(f"{nr} ranks: per-rank share {min(per):.3f}-{max(per):.3f} s -> {nsub / max(per):.1f} sub-scenes/s "
          f"(x{dt / max(per):.2f} over one GPU)")
