"""Quick GPU parity/timing check (development aid)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
from oracle import oracle as O

def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)

eng = F.Engine(0)
scenes = [("cube", S.generate_cube_scene(1, 0.5)), ("ring12", S.generate_random_scene(12, 90, 0.4, 9, 0.5)),
          ("cfg1", S.generate_config(1)), ("cfg2", S.generate_config(2))]
for name, rec in scenes:
    print("==", name, rec.cams.shape, rec.pts.shape, rec.obs_cam.shape, flush=True)
    jc, jp = O.jacobian(rec)
    J = eng.assemble_jacobian(rec)
    print(" jac bitexact", np.array_equal(J.cam_blocks, jc), np.array_equal(J.point_blocks, jp), flush=True)
    H, _ = O.nullspace(rec)
    Hg = eng.gauge_nullspace(rec)
    print(" H bitexact", np.array_equal(H, Hg), np.abs(H - Hg).max(), flush=True)
    D, A, Cp, sa, sb, fl = O.fisher(rec)
    fb = eng.build_fisher_blocks(rec)
    print(" fisher D", np.array_equal(D, fb.cam_blocks), "A", np.array_equal(A, fb.point_blocks), "Cp", np.array_equal(Cp, fb.couplings),
          "sa", np.array_equal(sa, fb.s_a), "sb", rel(fb.s_b, sb), flush=True)
    z = O.schur(rec)
    zg = eng.schur_reduce(rec)
    print(" schur rel", rel(zg, z), flush=True)
    t0 = time.time(); cov, d, fl, tm = O.compute_covariance(rec); t1 = time.time()
    res = eng.compute_covariance(rec); t2 = time.time()
    worst = max(rel(a, b) for a, b in zip(res.camera_cov, cov))
    print(f" cov worst rel {worst:.3e}  oracle {t1-t0:.3f}s gpu {t2-t1:.3f}s", flush=True)
    print(" diag", res.diagnostics.inertia_positive, res.diagnostics.inertia_negative, res.diagnostics.largest_dense_dim,
          res.diagnostics.min_pivot, res.diagnostics.max_pivot, d.min_pivot, d.max_pivot, flush=True)

# dense path on a random SPD matrix
rng = np.random.default_rng(0)
for n in [126, 270, 1008, 2700]:
    M = rng.standard_normal((n, n)); A = M @ M.T + n * np.eye(n)
    blocks, piv = eng.spd_inverse_blocks(A, 9)
    Ai = np.linalg.inv(A)
    w = max(rel(blocks[i], Ai[9*i:9*i+9, 9*i:9*i+9]) for i in range(n // 9))
    print("spd", n, w, flush=True)

for cfg in [3]:
    rec = S.generate_config(cfg)
    print("== cfg", cfg, rec.cams.shape, rec.pts.shape, rec.obs_cam.shape, flush=True)
    eng.set_profiling(True)
    for it in range(3):
        t0 = time.time(); res = eng.compute_covariance(rec); t1 = time.time()
        print(f" gpu e2e {t1-t0:.4f}s", eng.counts(), flush=True)
        print(" ", {k: round(v, 3) for k, v in eng.stage_times().items()}, flush=True)
