"""Pins of the CPU restatement (oracle/) against the reference's own
known-answer and property tests.  The reference ships
no golden vectors, so these are the pins; each test cites the reference test
it ports.  CPU only."""
import numpy as np
import pytest

from conftest import disconnected_scene, rel
from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S
from paper_1808_02414_b200.rotation import random_rotation, rotation_matrix as np_rotation, skew

pytestmark = pytest.mark.filterwarnings("ignore")


# ---- projection (tests/test_projection.cpp) ------------------------------------
def test_projection_known_answer():  # test_projection.cpp:31-46
    cam = np.array([0, 0, 0, 0, 0, 0, 2.0, 0.1])
    u = O.project(cam, np.array([0.2, -0.4, 2.0]))
    assert u[0] == pytest.approx(0.201, rel=1e-12) and u[1] == pytest.approx(-0.402, rel=1e-12)
    cam[7] = 0.0
    u = O.project(cam, np.array([0.2, -0.4, 2.0]))
    assert u[0] == pytest.approx(0.2, rel=1e-12) and u[1] == pytest.approx(-0.4, rel=1e-12)


def test_points_behind_camera_are_rejected():  # test_projection.cpp:48-61
    cam = np.array([0, 0, 0, 0, 0, 0, 100.0, 0.0])
    for z in (0.0, 1e-10, -2.0):
        for fn in (O.project, O.observation_jacobian):
            with pytest.raises(O.OracleFailure) as e:
                fn(cam, np.array([0.1, 0.1, z]))
            assert e.value.kind_name == "degenerate" and e.value.stage == "projection"
            assert "behind camera" in str(e.value)
    O.project(cam, np.array([0.1, 0.1, 1e-8]))


def _random_pair(rng, P):
    while True:
        axis = rng.uniform(-1, 1, 3)
        if np.linalg.norm(axis) < 1e-3:
            continue
        r = axis / np.linalg.norm(axis) * abs(rng.uniform(-1, 1)) * 3.0
        C = rng.uniform(-1, 1, 3) * 5.0
        intr = [rng.uniform(50, 200), rng.uniform(-0.3, 0.3)] + ([rng.uniform(-0.1, 0.1)] if P == 9 else [])
        cam = np.concatenate([r, C, intr])
        X = rng.uniform(-1, 1, 3) * 5.0
        v = np_rotation(r) @ (X - C)
        if v[2] < 0.5 or abs(v[0] / v[2]) > 1.5 or abs(v[1] / v[2]) > 1.5:
            continue
        return cam, X


@pytest.mark.parametrize("P", [8, 9])
def test_analytic_jacobian_matches_finite_differences(P):  # test_projection.cpp:63-72, acceptance criterion 3
    rng = np.random.default_rng(123 + P)
    worst = 0.0
    for _ in range(200):
        cam, X = _random_pair(rng, P)
        jc, jp = O.observation_jacobian(cam, X)
        x = np.concatenate([cam, X])
        num = np.empty((2, P + 3))
        for p in range(P + 3):
            h = 1e-6 * max(1.0, abs(x[p]))
            hi, lo = x.copy(), x.copy()
            hi[p] += h
            lo[p] -= h
            num[:, p] = (O.project(hi[:P], hi[P:]) - O.project(lo[:P], lo[P:])) / (2 * h)
        ana = np.hstack([jc, jp])
        worst = max(worst, np.abs(ana - num).max() / max(1.0, np.abs(num).max()))
    assert worst < 1e-5


def test_center_and_point_derivatives_are_exact_negatives():  # test_projection.cpp:74-81
    rng = np.random.default_rng(321)
    for _ in range(50):
        cam, X = _random_pair(rng, 8)
        jc, jp = O.observation_jacobian(cam, X)
        assert np.array_equal(jc[:, 3:6], -jp)


def test_failures_name_the_observation():  # test_projection.cpp:103-110
    rec = S.generate_cube_scene(4, 0.0)
    rec.pts[5] = rec.cams[0, 3:6]
    with pytest.raises(O.OracleFailure) as e:
        O.jacobian(rec)
    assert e.value.stage == "jacobian" and "observation 5" in str(e.value)


# ---- rotation (tests/test_rotation.cpp) ----------------------------------------
def test_rotation_is_orthonormal():  # test_rotation.cpp:35-44
    rng = np.random.default_rng(101)
    for angle in (0.0, 1e-12, 1e-9, 1e-8, 1e-4, 0.5, 2.0, 3.1, np.pi):
        v = rng.uniform(-1, 1, 3)
        R = O.rotation_matrix(v / np.linalg.norm(v) * angle)
        assert np.abs(R.T @ R - np.eye(3)).max() < 1e-13
        assert np.linalg.det(R) == pytest.approx(1.0, rel=1e-12)


def test_series_branch_joins_closed_form():  # test_rotation.cpp:62-70
    axis = np.array([0.3, -0.5, 0.8])
    axis /= np.linalg.norm(axis)
    for angle in (0.99e-8, 1.01e-8):
        r = axis * angle
        assert np.abs(O.rotation_matrix(r) - (np.eye(3) + skew(r))).max() < 1e-15


def test_rotate_point_derivative_matches_fd():  # test_rotation.cpp:72-88
    rng = np.random.default_rng(7)
    for angle in (0.0, 1e-9, 1e-7, 0.2, 1.3, 2.8):
        for _ in range(10):
            v = rng.uniform(-1, 1, 3)
            r = v / np.linalg.norm(v) * angle
            w = rng.uniform(-5, 5, 3)
            ana = O.rotate_point_derivative(r, w)
            num = np.empty((3, 3))
            for p in range(3):
                h = 1e-6 * max(1.0, abs(r[p]))
                hi, lo = r.copy(), r.copy()
                hi[p] += h
                lo[p] -= h
                num[:, p] = (O.rotation_matrix(hi) @ w - O.rotation_matrix(lo) @ w) / (2 * h)
            assert np.abs(ana - num).max() / max(1.0, np.abs(num).max()) < 1e-5


def test_deterministic_sincos_is_accurate():
    xs = np.concatenate([np.linspace(0, np.pi, 2001), [1e-9, 0.7853981633974483, 2.356194490192345]])
    for x in xs:
        s, c = O.sincos(x)
        assert abs(s - np.sin(x)) <= 2.3e-16 and abs(c - np.cos(x)) <= 2.3e-16


# ---- synthetic scenes (tests/test_synthetic.cpp) ---------------------------------
def test_cube_scene_has_the_fixed_shape():  # test_synthetic.cpp:14-29
    rec = S.generate_cube_scene(1, 0.0)
    assert (rec.num_cameras(), rec.num_points(), rec.num_observations()) == (6, 15, 60)
    for i in range(6):
        assert np.linalg.norm(rec.cams[i, 3:6]) == pytest.approx(10.0)
        assert rec.cams[i, 6] == 100.0 + 5.0 * i
    for t in range(60):
        assert rec.obs_cam[t] == t // 10 and rec.obs_pt[t] == (2 * rec.obs_cam[t] + t % 10) % 15


# ---- Fisher blocks (tests/test_fisher.cpp) ---------------------------------------
def _dense_from_blocks(rec, D, A, Cp):
    n, m, P = rec.num_cameras(), rec.num_points(), rec.cam_params
    M = np.zeros((P * n + 3 * m,) * 2)
    for i in range(n):
        M[P * i:P * i + P, P * i:P * i + P] = D[i]
    for j in range(m):
        M[P * n + 3 * j:P * n + 3 * j + 3, P * n + 3 * j:P * n + 3 * j + 3] = A[j]
    for t in range(rec.num_observations()):
        ci, pj = rec.obs_cam[t], rec.obs_pt[t]
        M[P * ci:P * ci + P, P * n + 3 * pj:P * n + 3 * pj + 3] += Cp[t]
        M[P * n + 3 * pj:P * n + 3 * pj + 3, P * ci:P * ci + P] += Cp[t].T
    return M


def _dense_jacobian(rec):
    jc, jp = O.jacobian(rec)
    n, P = rec.num_cameras(), rec.cam_params
    J = np.zeros((2 * rec.num_observations(), rec.num_parameters()))
    for t in range(rec.num_observations()):
        ci, pj = rec.obs_cam[t], rec.obs_pt[t]
        J[2 * t:2 * t + 2, P * ci:P * ci + P] = jc[t]
        J[2 * t:2 * t + 2, P * n + 3 * pj:P * n + 3 * pj + 3] = jp[t]
    return J


@pytest.mark.parametrize("scene", ["cube0", "cube05", "ring"])
def test_block_fisher_matches_dense_product(scene):  # test_fisher.cpp:42-52
    rec = {"cube0": lambda: S.generate_cube_scene(1, 0.0), "cube05": lambda: S.generate_cube_scene(1, 0.5),
           "ring": lambda: S.generate_random_scene(7, 50, 0.5, 4, 0.7)}[scene]()
    D, A, Cp, *_ = O.fisher(rec)
    J = _dense_jacobian(rec)
    W = np.zeros((J.shape[0],) * 2)
    for t in range(rec.num_observations()):
        W[2 * t:2 * t + 2, 2 * t:2 * t + 2] = np.linalg.inv(rec.obs_sigma[t])
    assert rel(_dense_from_blocks(rec, D, A, Cp), J.T @ W @ J) < 1e-13


def test_sigma_scaling_scales_blocks_bitwise():  # test_fisher.cpp:54-68
    rec = S.generate_cube_scene(2, 0.5)
    loose = rec.copy()
    loose.obs_sigma *= 4.0
    D, A, Cp, *_ = O.fisher(rec)
    D4, A4, Cp4, *_ = O.fisher(loose)
    assert np.array_equal(D4, 0.25 * D) and np.array_equal(A4, 0.25 * A) and np.array_equal(Cp4, 0.25 * Cp)


def test_non_spd_sigma_is_reported_by_index():  # test_fisher.cpp:70-89
    rec = S.generate_cube_scene(3, 0.5)
    rec.obs_sigma[7] = [[1.0, 2.0], [2.0, 1.0]]
    with pytest.raises(O.OracleFailure) as e:
        O.fisher(rec)
    assert e.value.kind_name == "degenerate" and e.value.stage == "fisher" and "observation 7" in str(e.value)


def test_conditioning_normalises_diagonals_and_border():  # test_fisher.cpp:128-150
    rec = S.generate_cube_scene(4, 0.5)
    D, A, Cp, sa, sb, flagged = O.fisher(rec)
    assert flagged == []
    n, P = rec.num_cameras(), rec.cam_params
    for i in range(n):
        assert np.array_equal(sa[P * i:P * i + P], 1.0 / np.sqrt(np.diag(D[i])))
        assert np.allclose(np.diag(sa[P * i:P * i + P, None] * D[i] * sa[None, P * i:P * i + P]), 1.0, rtol=1e-12)
    for j in range(rec.num_points()):
        s = sa[P * n + 3 * j:P * n + 3 * j + 3]
        assert np.allclose(np.diag(s[:, None] * A[j] * s[None, :]), 1.0, rtol=1e-12)
    H, _ = O.nullspace(rec)
    Hs = sa[:, None] * H * sb[None, :]
    assert np.allclose(np.linalg.norm(Hs, axis=0), 1.0, rtol=1e-12)


# ---- nullspace (tests/test_nullspace.cpp) ------------------------------------------
def test_closed_form_rows():  # test_nullspace.cpp:28-51
    rec = S.generate_cube_scene(1, 0.5)
    H, _ = O.nullspace(rec)
    n, P = rec.num_cameras(), rec.cam_params
    for i in range(n):
        C = rec.cams[i, 3:6]
        assert np.array_equal(H[P * i + 3:P * i + 6, 0:3], np.eye(3))
        assert np.array_equal(H[P * i + 3:P * i + 6, 3:6], skew(C))
        assert np.array_equal(H[P * i + 3:P * i + 6, 6], C)
        assert not H[P * i + 6:P * i + P].any()
        assert not H[P * i:P * i + 3, 0:3].any() and not H[P * i:P * i + 3, 6].any()
    for j in range(rec.num_points()):
        X = rec.pts[j]
        r0 = P * n + 3 * j
        assert np.array_equal(H[r0:r0 + 3, 0:3], np.eye(3))
        assert np.array_equal(H[r0:r0 + 3, 3:6], skew(X))
        assert np.array_equal(H[r0:r0 + 3, 6], X)


@pytest.mark.parametrize("P", [8, 9])
def test_jh_vanishes(P):  # test_nullspace.cpp:53-61, acceptance criterion 2
    for rec in (S.generate_cube_scene(1, 0.0, P), S.generate_cube_scene(2, 0.5, P),
                S.generate_random_scene(12, 90, 0.4, 5, 0.5, P)):
        _, res = O.nullspace(rec)
        assert res < 1e-10


def test_residual_detects_corruption():  # test_nullspace.cpp:63-69
    rec = S.generate_cube_scene(1, 0.5)
    H, _ = O.nullspace(rec)
    H[0, 0] += 1.0
    assert O.nullspace_residual(rec, H) > 1e-4


def test_basis_has_full_column_rank():  # test_nullspace.cpp:71-78
    rec = S.generate_random_scene(8, 60, 0.5, 3, 0.5)
    H, _ = O.nullspace(rec)
    sv = np.linalg.svd(H / np.linalg.norm(H, axis=0), compute_uv=False)
    assert sv[6] / sv[0] > 1e-8


def test_residual_survives_similarity_transform():  # test_nullspace.cpp:144-151
    rng = np.random.default_rng(9)
    rec = S.generate_random_scene(9, 70, 0.4, 8, 0.5)
    moved = S.transform_scene(rec, random_rotation(rng), np.array([3.0, -1.0, 2.0]), 0.6)
    assert O.nullspace(moved)[1] < 1e-8


# ---- Schur reduction (tests/test_schur.cpp) -----------------------------------------
def _conditioned(rec):
    D, A, Cp, sa, sb, _ = O.fisher(rec)
    H, _ = O.nullspace(rec)
    return D, A, Cp, sa, sb, H


def test_schur_matches_dense_elimination():  # test_schur.cpp:57-64
    rec = S.generate_cube_scene(1, 0.5)
    D, A, Cp, sa, sb, H = _conditioned(rec)
    n, m, P = rec.num_cameras(), rec.num_points(), rec.cam_params
    M = _dense_from_blocks(rec, D, A, Cp)
    Ms = sa[:, None] * M * sa[None, :]
    Hs = sa[:, None] * H * sb[None, :]
    Nc = P * n
    Dp = np.zeros((Nc + 7, Nc + 7))
    Dp[:Nc, :Nc] = Ms[:Nc, :Nc]
    Dp[:Nc, Nc:] = Hs[:Nc]
    Dp[Nc:, :Nc] = Hs[:Nc].T
    Cc = np.hstack([Ms[Nc:, :Nc], Hs[Nc:]])
    ref = Dp - Cc.T @ np.linalg.solve(Ms[Nc:, Nc:], Cc)
    z = O.schur(rec)
    assert rel(z, ref) < 1e-10
    assert np.array_equal(z, z.T)  # test_schur.cpp:66-70


def test_disconnected_components_never_couple():  # test_schur.cpp:72-80
    rec = disconnected_scene(3, 0.5)
    z = O.schur(rec)
    assert not z[:48, 48:96].any()


def test_inversion_records_inertia():  # test_schur.cpp:115-129
    rec = S.generate_cube_scene(7, 0.5)
    z = O.schur(rec)
    zi, d = O.invert_schur(z)
    assert np.abs(z @ zi - np.eye(z.shape[0])).max() < 1e-8
    assert np.array_equal(zi, zi.T)
    assert (d.inertia_positive, d.inertia_negative) == (48, 7)
    assert d.min_pivot > 0 and d.max_pivot >= d.min_pivot


def test_small_hand_checked_factorizations():  # test_schur.cpp:131-150
    zi, d = O.invert_schur(np.diag([2.0, 3.0]))
    assert zi[0, 0] == pytest.approx(0.5, rel=1e-14) and zi[1, 1] == pytest.approx(1 / 3, rel=1e-14)
    assert (d.inertia_positive, d.inertia_negative) == (2, 0)
    assert d.min_pivot == pytest.approx(2.0) and d.max_pivot == pytest.approx(3.0)
    sw = np.array([[0.0, 1.0], [1.0, 0.0]])
    zi, d = O.invert_schur(sw)
    assert np.abs(zi - sw).max() < 1e-14 and (d.inertia_positive, d.inertia_negative) == (1, 1)


# ---- pipeline (tests/test_covariance.cpp, test_oracle.cpp) ---------------------------
def test_pipeline_diagnostics_on_a_good_scene():  # test_covariance.cpp:16-40
    cov, d, flagged, _ = O.compute_covariance(S.generate_cube_scene(1, 0.5))
    assert cov.shape == (6, 8, 8) and flagged == []
    assert d.scale_min > 0 and d.scale_max >= d.scale_min and d.negative_eigenvalue_warnings == 0
    assert (d.inertia_positive, d.inertia_negative, d.largest_dense_dim) == (48, 7, 55)
    assert d.min_pivot > 1e-12 * d.max_pivot
    for c in cov:
        assert np.abs(c - c.T).max() <= 1e-14 * np.abs(c).max() and np.diag(c).min() > 0


@pytest.mark.parametrize("scene", ["cube", "ring"])
def test_pipeline_matches_the_dense_pseudoinverse(scene):  # test_oracle.cpp:90-101, acceptance 1
    rec = S.generate_cube_scene(7, 0.5) if scene == "cube" else S.generate_random_scene(10, 80, 0.4, 6, 0.5)
    cov, *_ = O.compute_covariance(rec)
    gt, sigma, sv, gap = O.pseudoinverse(rec)
    assert O.error_metric(gt, cov, rec.cams)[0] < 1e-4
    assert max(rel(a, b) for a, b in zip(cov, gt)) < 1e-6


def test_pseudoinverse_identities_and_gap():  # test_oracle.cpp:27-51
    rec = S.generate_cube_scene(3, 0.5)
    M = O.dense_fisher(rec)
    _, sigma, sv, gap = O.pseudoinverse(rec)
    assert len(sv) == 93 and np.all(np.diff(sv) <= 0) and gap > 1e6
    assert rel(M @ sigma @ M, M) < 1e-6 and rel(sigma @ M @ sigma, sigma) < 1e-6
    assert np.trace(M @ sigma) == pytest.approx(93 - 7, rel=1e-9)
    H, _ = O.nullspace(rec)
    assert np.abs(H.T @ sigma).max() / (np.abs(H).max() * np.abs(sigma).max()) < 1e-8


def test_disconnected_scene_fails_in_factorization():  # test_covariance.cpp:80-90
    with pytest.raises(O.OracleFailure) as e:
        O.compute_covariance(disconnected_scene(4, 0.5))
    assert e.value.kind_name == "degenerate" and e.value.stage == "factorization"
    assert "disconnected" in str(e.value)


def test_relabelling_points_does_not_change_cameras():  # test_covariance.cpp:92-104
    rec = S.generate_cube_scene(5, 0.5)
    m = rec.num_points()
    perm = (7 * np.arange(m) + 3) % m
    moved = rec.copy()
    moved.pts[perm] = rec.pts
    moved.obs_pt = perm[rec.obs_pt].astype(np.int32)
    a, *_ = O.compute_covariance(rec)
    b, *_ = O.compute_covariance(moved)
    assert max(rel(x, y) for x, y in zip(a, b)) < 1e-10


def test_intrinsics_invariant_under_similarity():  # test_covariance.cpp:106-118
    rng = np.random.default_rng(11)
    rec = S.generate_random_scene(10, 80, 0.4, 7, 0.5)
    moved = S.transform_scene(rec, random_rotation(rng), np.array([2.0, 5.0, -1.0]), 0.6)
    a, *_ = O.compute_covariance(rec)
    b, *_ = O.compute_covariance(moved)
    for x, y in zip(a, b):
        assert rel(x[6:8, 6:8], y[6:8, 6:8]) < 1e-6


def test_results_are_identical_for_any_thread_count():  # test_covariance.cpp:137-156
    rec = S.generate_random_scene(12, 90, 0.4, 9, 0.5)
    a, *_ = O.compute_covariance(rec, threads=1)
    b, *_ = O.compute_covariance(rec, threads=1)
    c, *_ = O.compute_covariance(rec, threads=4)
    assert np.array_equal(a, b) and np.array_equal(a, c)


@pytest.mark.parametrize("P", [8, 9])
def test_cholesky_route_equals_bordered_ldlt(P):  # SURVEY.md appendix A, route A
    rec = S.generate_random_scene(12, 150, 0.34, 3, 0.5, P)
    cov, *_ = O.compute_covariance(rec)
    z = O.schur(rec)
    _, _, _, sa, _, _ = O.fisher(rec)
    chol = O.cholesky_route(z, rec.num_cameras(), P, sa[:P * rec.num_cameras()])
    assert max(rel(a, b) for a, b in zip(chol, cov)) < 1e-10


# ---- validation messages (src/scene.cpp:19-78) ---------------------------------------
@pytest.mark.parametrize("mutate,fragment", [
    (lambda r: r.cams.__setitem__((2, 0), np.nan), "camera 2 has non-finite parameters"),
    (lambda r: r.cams.__setitem__((1, 6), -1.0), "camera 1 has non-positive focal length"),
    (lambda r: r.pts.__setitem__((4, 1), np.inf), "point 4 has non-finite coordinates"),
    (lambda r: r.obs_cam.__setitem__(3, 99), "observation 3 camera index out of range"),
    (lambda r: r.obs_pt.__setitem__(5, -1), "observation 5 point index out of range"),
    (lambda r: r.obs_sigma.__setitem__((6, 0, 1), 0.3), "observation 6 covariance not symmetric"),
    (lambda r: r.obs_sigma.__setitem__(8, -np.eye(2)), "observation 8 covariance not positive definite"),
    (lambda r: r.obs_pt.__setitem__(1, r.obs_pt[0]), "duplicate (camera, point) observation pair"),
])
def test_validation_messages(mutate, fragment):  # tests/test_scene.cpp
    rec = S.generate_cube_scene(1, 0.5)
    mutate(rec)
    with pytest.raises(O.OracleFailure) as e:
        O.validate(rec)
    assert e.value.stage == "validate" and e.value.kind_name == "invariant" and fragment in str(e.value)


def test_count_floors():
    rec = S.generate_cube_scene(1, 0.5)
    keep = rec.obs_cam != 2
    keep[np.flatnonzero(rec.obs_cam == 2)[:3]] = True  # camera 2 keeps 3 observations
    sub = rec.copy()
    for k in ("obs_cam", "obs_pt", "obs_u", "obs_sigma"):
        setattr(sub, k, getattr(rec, k)[keep])
    with pytest.raises(O.OracleFailure) as e:
        O.validate(sub)
    assert "camera 2 observes 3 points, need at least 4" in str(e.value)


def test_point_and_cross_covariances_match_the_materialized_covariance():  # test_covariance.cpp:42-68
    rec = S.generate_cube_scene(2, 0.5)
    cov, pc, cm, _ = O.compute_covariance_full(rec)
    _, sigma, _, _ = O.pseudoinverse(rec)
    n, P, m = rec.cams.shape[0], rec.cams.shape[1], rec.pts.shape[0]
    assert sigma.shape[0] == P * n + 3 * m
    for i in range(n):
        assert rel(cov[i], sigma[P * i:P * i + P, P * i:P * i + P]) < 1e-8
    assert pc.shape == (m, 3, 3)
    for j in range(m):
        r0 = P * n + 3 * j
        assert rel(pc[j], sigma[r0:r0 + 3, r0:r0 + 3]) < 1e-8
    assert cm.shape == (P * n, P * n)
    for i in range(n):
        assert np.array_equal(cm[P * i:P * i + P, P * i:P * i + P], cov[i])
        for l in range(n):
            assert rel(cm[P * i:P * i + P, P * l:P * l + P], sigma[P * i:P * i + P, P * l:P * l + P]) < 1e-8


@pytest.mark.parametrize("make", [lambda: S.generate_cube_scene(1, 0.5),
                                  lambda: S.generate_random_scene(12, 150, 0.3, 5, 0.5)], ids=["cube", "random12"])
def test_restatement_matches_the_long_double_bordered_inverse(make):
    # the reference route (dsytrf + dsytrs2 on the bordered Schur matrix) and
    # a long-double LU solve of the unreduced bordered Fisher matrix agree to
    # FP64 rounding: the two formulations of src/covariance.cpp:137-279 are
    # the same inverse, and the long-double solve is the truth the GPU's
    # double-double refinement is checked against (test_gpu_truth.py)
    rec = make()
    exact = O.exact_camera_blocks(rec, 5000)
    ref = O.compute_covariance(rec)[0]
    worst = max(np.linalg.norm(a - b) / np.linalg.norm(b) for a, b in zip(ref, exact))
    assert worst <= 1e-11
