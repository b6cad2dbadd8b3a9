"""Config-N point / cross covariances: GPU vs the restatement, with timings."""
import sys, time; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
def worst(a, b): return max(rel(x, y) for x, y in zip(a, b))
rec = S.generate_config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
eng = F.Engine(0)
opts = F.CovarianceOptions(point_covariances=True, camera_cross_covariances=True)
for i in range(3):
    t0 = time.perf_counter(); r = eng.compute_covariance(rec, opts); t1 = time.perf_counter()
print(f"gpu full outputs e2e {t1 - t0:.4f} s (camera blocks only: ", end="")
t0 = time.perf_counter(); eng.compute_covariance(rec); print(f"{time.perf_counter() - t0:.4f} s)")
O.lib().oracle_blas_threads(0)
t0 = time.perf_counter(); cov, pc, cm, _ = O.compute_covariance_full(rec, threads=16); t1 = time.perf_counter()
print(f"restatement full outputs {t1 - t0:.2f} s")
P, n = rec.cam_params, rec.num_cameras()
print("camera worst", worst(r.camera_cov, cov), "point worst", worst(r.point_cov, pc), "matrix rel", rel(r.camera_matrix, cm))
print("diag bitwise", all(np.array_equal(r.cross_block(i, i), r.camera_cov[i]) for i in range(n)))
