"""Parity against the exact inverse of the bordered Fisher system.

The reference's camera covariance is the camera block of K^-1,
K = [[M, H], [H^T, 0]] (src/covariance.cpp:33-279, src/nullspace.cpp:14-62).
The FP64 values of M's blocks (D, A, couplings) and of H are bit-identical
between the GPU and the CPU restatement (test_gpu_parity.py), so taking them
as exact data defines one target for every route.  The GPU computes it by
iterative refinement with double-double residuals
(sfmcov_cuda_refine_covariance); on small scenes that truth is checked against
an independent long-double LU solve of K on the CPU (oracle/).  Then the FP64
product pipeline is held to <= 1e-9 per camera block (north_star) against it
on every BASELINE config and on the reference's README scale point (P = 8,
1000 cameras, 100k points, N = 8007: proj/README.md:21-23,
tests/acceptance.cpp:237-262) -- including configs 4 and 5, where no CPU
inverse is affordable.  profiles/r02_truth_parity.txt records the same
numbers with the reference route (the restatement's dsytrf + dsytrs2) beside
them.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1808_02414_b200 import synthetic as S

ITERS = 3


def rel_blocks(a, b):
    return np.linalg.norm((a - b).reshape(len(a), -1), axis=1) / np.linalg.norm(b.reshape(len(b), -1), axis=1)


def refine_all(engine, rec, cams=None):
    cams = np.arange(rec.num_cameras(), dtype=np.int32) if cams is None else cams
    truth, base, hist = engine.refine_covariance(rec, cams, ITERS)
    # converged: the last step changes no block by more than a few ulps
    assert hist[0] == pytest.approx(1.0) and hist[-1] <= 1e-14, hist
    return truth, base


@pytest.mark.gpu
@pytest.mark.parametrize("make", [lambda: S.generate_cube_scene(1, 0.5),
                                  lambda: S.generate_random_scene(12, 150, 0.3, 5, 0.5),
                                  lambda: S.generate_random_scene(20, 300, 0.3, 11, 0.5, 9)],
                         ids=["cube", "random12", "random20_p9"])
def test_refined_truth_matches_the_long_double_solve(engine, make):
    rec = make()
    truth, base = refine_all(engine, rec)
    exact = O.exact_camera_blocks(rec, 5000)
    assert rel_blocks(truth, exact).max() <= 1e-14
    assert rel_blocks(base, exact).max() <= 1e-9
    # the restatement of the reference route, for scale (~1e-13 here)
    assert rel_blocks(O.compute_covariance(rec)[0], exact).max() <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("config", [1, 2, 3])
def test_configs_within_1e9_of_the_exact_inverse(engine, config):
    rec = S.generate_config(config)
    truth, base = refine_all(engine, rec)
    err = rel_blocks(base, truth)
    assert err.max() <= 1e-9, (err.max(), int(err.argmax()))


@pytest.mark.gpu
def test_readme_scale_point_p8(engine):
    # 1000 cameras (P = 8), 100k points, visibility 0.008 -> N = 8007, the
    # scene behind the reference's only published number
    rec = S.generate_random_scene(1000, 100000, 0.008, 3, 0.5)
    assert rec.cam_params == 8 and rec.num_cameras() == 1000
    truth, base = refine_all(engine, rec)
    err = rel_blocks(base, truth)
    assert err.max() <= 1e-9, (err.max(), int(err.argmax()))


@pytest.mark.gpu
def test_config4_every_camera_within_1e9(engine):
    # Z 27000^2; the reference's own route (dsytrf + dsytrs2 on the
    # restatement's Z_p) is off by up to 1.3e-8 here (83 blocks > 1e-9,
    # profiles/r02_truth_parity.txt): the bar is met by the GPU, not by it
    rec = S.generate_config(4)
    truth, base = refine_all(engine, rec)
    err = rel_blocks(base, truth)
    assert err.max() <= 1e-9, (err.max(), int(err.argmax()))


@pytest.mark.gpu
def test_config5_sampled_cameras_within_1e9(engine):
    # Z 90000^2 (65 GB): 48 seeded random cameras
    rec = S.generate_config(5)
    cams = np.sort(np.random.default_rng(0).choice(rec.num_cameras(), 48, replace=False)).astype(np.int32)
    truth, base = refine_all(engine, rec, cams)
    err = rel_blocks(base, truth)
    assert err.max() <= 1e-9, (err.max(), int(cams[err.argmax()]))


@pytest.mark.gpu
@pytest.mark.parametrize("args", [(200, 5000, 0.1, 21, 0.5, 9), (300, 20000, 0.05, 22, 0.5, 8),
                                  (150, 3000, 0.2, 23, 2.0, 8)],
                         ids=["random200_p9", "random300_p8", "random150_noisy"])
def test_random_scenes_within_1e9_of_the_exact_inverse(engine, args):
    # beyond the BASELINE configs: the reference generator's random scenes
    # (src/synthetic.cpp:52-110) at a few sizes, densities and noise levels
    rec = S.generate_random_scene(*args)
    truth, base = refine_all(engine, rec)
    err = rel_blocks(base, truth)
    assert err.max() <= 1e-9, (err.max(), int(err.argmax()))
