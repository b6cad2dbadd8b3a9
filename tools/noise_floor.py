"""FP64 noise floor of the camera blocks (config 3 by default): the restatement's dsytrf
route against its Cholesky route, and both against the GPU paths."""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
def worst(a, b):
    r = np.array([rel(x, y) for x, y in zip(a, b)])
    return f"{r.max():.3e} (camera {int(r.argmax())}, {int((r > 1e-9).sum())} blocks > 1e-9, median {np.median(r):.2e})"
rec = S.generate_config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
O.lib().oracle_blas_threads(0)
cov, d, _, _ = O.compute_covariance(rec, threads=16)
zp = O.schur(rec)
_, _, _, sa, _, _ = O.fisher(rec)
P, n = rec.cam_params, rec.num_cameras()
covc = O.cholesky_route(zp, n, P, sa[:P * n], 16)
eng = F.Engine(0)
g1 = eng.compute_covariance(rec).camera_cov
g2 = eng.compute_covariance_emulated(rec, 2).camera_cov
print("oracle dsytrf vs oracle cholesky: worst", worst(covc, cov), "overall", rel(covc, cov))
print("gpu single vs dsytrf: worst", worst(g1, cov), "overall", rel(g1, cov))
print("gpu single vs cholesky: worst", worst(g1, covc), "overall", rel(g1, covc))
print("gpu dist2 vs dsytrf: worst", worst(g2, cov), "overall", rel(g2, cov))
print("gpu dist2 vs cholesky: worst", worst(g2, covc), "overall", rel(g2, covc))
