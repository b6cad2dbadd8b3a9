"""The reference's acceptance criteria (tests/acceptance.cpp), run through
the B200 path.  The dense reference covariance is the GPU pseudoinverse
oracle; the Eq. 42 metric and |J H| residual come from the test
infrastructure (oracle/)."""
import time

import numpy as np
import pytest

from conftest import rel
from oracle import oracle as O
from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import subrec as R
from paper_1808_02414_b200 import synthetic as S
from paper_1808_02414_b200.rotation import random_rotation

pytestmark = pytest.mark.gpu


def reference_scenes():  # acceptance.cpp:72-79
    return [S.generate_cube_scene(1, 0.5), S.generate_random_scene(10, 60, 0.3, 11, 0.5),
            S.generate_random_scene(30, 100, 1.0 / 3.0, 12, 0.5), S.generate_random_scene(64, 200, 0.40625, 13, 0.5)]


def test_criteria_1_and_4_accuracy_and_moore_penrose(engine):  # acceptance.cpp:91-123
    worst_mean, worst_identity = 0.0, 0.0
    for rec in reference_scenes():
        gt, sigma, _, _ = engine.pseudoinverse_covariance(rec)
        fast = engine.compute_covariance(rec).camera_cov
        worst_mean = max(worst_mean, O.error_metric(gt, fast, rec.cams)[0])
        m = O.dense_fisher(rec)
        worst_identity = max(worst_identity, rel(m @ sigma @ m, m), rel(sigma @ m @ sigma, sigma))
    assert worst_mean < 1e-4
    assert worst_identity < 1e-6


def test_criterion_2_gauge_nullspace_residual(engine):  # acceptance.cpp:125-149
    rng = np.random.default_rng(2025)
    worst = 0.0
    for seed in range(100):
        if seed % 3 == 0:
            rec = S.generate_cube_scene(seed, 0.5)
        else:
            rec = S.generate_random_scene(5 + seed % 12, 40 + 3 * (seed % 7), 0.5, seed, 0.5)
        if seed % 2 == 1:
            rec = S.transform_scene(rec, random_rotation(rng), rng.uniform(-1, 1, 3) * 10.0,
                                    0.3 + 2.0 * abs(rng.uniform(-1, 1)))
        worst = max(worst, O.nullspace_residual(rec, engine.gauge_nullspace(rec)))
    assert worst < 1e-8


def test_criterion_5_sub_reconstruction_upper_bound(engine):  # acceptance.cpp:170-209
    rec = S.generate_random_scene(150, 800, 20.0 / 150.0, 5, 0.5)
    full = engine.compute_covariance(rec).camera_cov
    P = rec.cam_params
    min_ratio, checked = np.inf, 0
    for cams in R.plan_coverage(rec, 40, 0):
        m_ = np.isin(rec.obs_cam, cams)
        pts = np.nonzero(np.bincount(rec.obs_pt[m_], minlength=rec.num_points()) >= 2)[0].astype(np.int32)
        part = engine.compute_covariance(R.induced_scene(rec, cams, pts)).camera_cov
        for l, g in enumerate(cams):
            min_ratio = min(min_ratio, np.trace(part[l]) / np.trace(full[g]))
            checked += 1
    violations = 0
    for center in (0, 50, 100):
        small = R.extract_neighborhood(rec, center, 10)
        large = R.extract_neighborhood(rec, center, 40)
        violations += len(R.monotonicity_check(rec, small, large, engine=engine).violations)
    assert checked >= 150 and min_ratio >= 1.0 - 1e-8 and violations == 0


def test_criterion_6_error_decreases_with_window_size(engine):  # acceptance.cpp:211-235
    rec = S.generate_random_scene(40, 200, 0.2, 7, 0.5)
    sizes = [5, 10, 20, 40]
    rows = R.error_size_sweep(rec, sizes, 25, 123, engine=engine)
    medians = [np.median([r.err_relative for r in rows if r.k_bar == k]) for k in sizes]
    inversions = sum(1 for a, b in zip(medians, medians[1:]) if b > a)
    assert inversions <= 1


def test_criterion_7_scale(engine):  # acceptance.cpp:237-262 (limits: 120 s, 4 GiB host)
    rec = S.generate_random_scene(1000, 100000, 0.008, 3, 0.5)
    t0 = time.perf_counter()
    res = engine.compute_covariance(rec)
    elapsed = time.perf_counter() - t0
    assert elapsed < 120.0 and res.diagnostics.largest_dense_dim == 8 * 1000 + 7 and res.camera_cov.shape[0] == 1000


def test_criterion_8_determinism(engine):  # acceptance.cpp:264-293
    rec = S.generate_random_scene(150, 800, 20.0 / 150.0, 5, 0.5)
    a = engine.compute_covariance(rec, F.CovarianceOptions(threads=1)).camera_cov
    b = engine.compute_covariance(rec, F.CovarianceOptions(threads=1)).camera_cov
    c = engine.compute_covariance(rec, F.CovarianceOptions(threads=4)).camera_cov
    assert np.array_equal(a, b) and np.abs(a - c).max() <= 1e-12
