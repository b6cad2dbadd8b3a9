"""The reference's stage functions beyond compute_covariance, on the GPU:
invert_schur on arbitrary symmetric matrices (Jacobi eigendecomposition,
csrc/eigen.cu), full_covariance (covariance.hpp:115) and nullspace_residual
(nullspace.hpp:36).  The C++ header's versions of these and of
condition_columns / apply_conditioning / schur_reduce on caller-built systems
are exercised by tests/cpp/dropin_test.cpp (test_gpu_parity.py runs it)."""
import numpy as np
import pytest

from conftest import rel
from oracle import oracle as O
from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import synthetic as S


@pytest.mark.gpu
@pytest.mark.parametrize("n,neg", [(1, 0), (2, 1), (7, 3), (55, 7), (300, 7), (501, 40)])
def test_invert_schur_symmetric_indefinite(engine, n, neg):
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = rng.uniform(0.5, 20.0, n)
    lam[:neg] *= -1
    z = (q * lam) @ q.T
    z = 0.5 * (z + z.T)
    zi, (mn, mx), (pos, ng) = engine.invert_schur(z)
    assert (pos, ng) == (n - neg, neg)
    assert np.array_equal(zi, zi.T)
    assert np.abs(z @ zi - np.eye(n)).max() < 1e-10
    assert mn == pytest.approx(np.abs(lam).min(), rel=1e-10) and mx == pytest.approx(np.abs(lam).max(), rel=1e-10)


@pytest.mark.gpu
def test_invert_schur_rejects_singular_and_non_square(engine):
    with pytest.raises(F.Error) as e:
        engine.invert_schur(np.zeros((2, 3)))
    assert e.value.kind == F.ErrorKind.dimension
    z = np.diag([1.0, 2.0, 0.0])
    with pytest.raises(F.Error) as e:
        engine.invert_schur(z)
    assert e.value.kind == F.ErrorKind.degenerate and e.value.stage == "factorization"


@pytest.mark.gpu
@pytest.mark.parametrize("make", [lambda: S.generate_cube_scene(2, 0.5),
                                  lambda: S.generate_random_scene(12, 90, 0.4, 9, 0.5),
                                  lambda: S.generate_random_scene(10, 80, 0.5, 3, 0.5, 9)],
                         ids=["cube", "random12", "random10_p9"])
def test_full_covariance_matches_the_pipeline_blocks(engine, make):  # test_covariance.cpp:42-68
    rec = make()
    P, n, m = rec.cam_params, rec.num_cameras(), rec.num_points()
    sigma = engine.full_covariance(rec)
    assert sigma.shape == (rec.num_parameters(),) * 2 and np.array_equal(sigma, sigma.T)
    res = engine.compute_covariance(rec, F.CovarianceOptions(point_covariances=True, camera_cross_covariances=True))
    for i in range(n):
        assert rel(res.camera_cov[i], sigma[P * i:P * i + P, P * i:P * i + P]) < 1e-8
    for j in range(m):
        b = P * n + 3 * j
        assert rel(res.point_cov[j], sigma[b:b + 3, b:b + 3]) < 1e-8
    assert rel(res.camera_matrix, sigma[:P * n, :P * n]) < 1e-8
    # annihilates the gauge (test_covariance.cpp:70-78)
    H = O.nullspace(rec)[0]
    assert np.abs(H.T @ sigma).max() / (np.abs(H).max() * np.abs(sigma).max()) < 1e-6


@pytest.mark.gpu
def test_full_covariance_guard_and_invalid_scene(engine):  # test_covariance.cpp:120-135
    rec = S.generate_cube_scene(1, 0.0)
    with pytest.raises(F.Error) as e:
        engine.full_covariance(rec, 50)
    assert e.value.kind == F.ErrorKind.size_guard and "guard is 50" in str(e.value)
    bad = rec.copy()
    bad.cams[1, 6] = -1.0
    with pytest.raises(F.Error) as e:
        engine.full_covariance(bad)
    assert e.value.kind == F.ErrorKind.invariant and e.value.stage == "validate"


@pytest.mark.gpu
@pytest.mark.parametrize("make", [lambda: S.generate_cube_scene(1, 0.0), lambda: S.generate_cube_scene(2, 0.5),
                                  lambda: S.generate_random_scene(12, 90, 0.4, 5, 0.5)])
def test_nullspace_residual_on_the_gpu(engine, make):  # test_nullspace.cpp:53-69
    rec = make()
    H = O.nullspace(rec)[0]
    r = engine.nullspace_residual(rec, H)
    assert r < 1e-10
    assert r == pytest.approx(O.nullspace_residual(rec, H), rel=1e-6, abs=1e-16)
    H2 = H.copy()
    H2[0, 0] += 1.0
    assert engine.nullspace_residual(rec, H2) > 1e-4

