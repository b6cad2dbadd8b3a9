import sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
eng = F.Engine(0)
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
for name, rec in [("cube8", S.generate_cube_scene(1, 0.5)), ("config1", S.generate_config(1)), ("config2", S.generate_config(2)),
                  ("config3", S.generate_config(3))]:
    ref = eng.compute_covariance(rec)
    for R in (1, 2, 3, 4):
        try:
            t0 = time.time(); r = eng.compute_covariance_emulated(rec, R); dt = time.time() - t0
            print(name, R, "rel", rel(r.camera_cov, ref.camera_cov), "piv", r.diagnostics.min_pivot, ref.diagnostics.min_pivot,
                  r.diagnostics.max_pivot, ref.diagnostics.max_pivot, "warn", r.diagnostics.negative_eigenvalue_warnings, f"{dt:.3f}s", flush=True)
        except Exception as e:
            print(name, R, "ERROR", e, flush=True)
