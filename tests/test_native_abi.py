"""The drop-in C ABI library loads and exports every symbol
include/sfmcov_b200.h declares; it has no CPU path; the scene generators are
deterministic and satisfy the reference's scene invariants.  CPU only (no
compute calls into the CUDA library)."""
import ctypes as C
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1808_02414_b200 import _native as N
from paper_1808_02414_b200 import synthetic as S

HEADER = (ROOT / "include" / "sfmcov_b200.h").read_text()


def declared_functions():
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    return sorted(set(re.findall(r"\b(sfmcov_(?:cuda|synth|nccl|plan|view|extract|scene|covio)_\w+)\s*\(", body)))


def test_header_declares_the_entry_points():
    names = declared_functions()
    for must in ("sfmcov_cuda_compute_covariance", "sfmcov_cuda_compute_covariance_device", "sfmcov_cuda_jacobian",
                 "sfmcov_cuda_nullspace", "sfmcov_cuda_fisher", "sfmcov_cuda_schur", "sfmcov_cuda_create"):
        assert must in names


def test_cuda_library_exports_every_declared_symbol():
    lib = C.CDLL(str(N.LIB_PATH))
    synth = C.CDLL(str(N.SYNTH_PATH))
    missing = [n for n in declared_functions()
               if not hasattr(synth if n.startswith(("sfmcov_synth", "sfmcov_scene", "sfmcov_covio")) else lib, n)]
    assert missing == []
    # and the Python binding table covers them all
    assert set(declared_functions()) == set(N.CUDA_SYMBOLS) | set(N.SYNTH_SYMBOLS)


def test_library_is_built_for_sm_100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1808_02414_b200 import sfmcov as F
    with pytest.raises(F.Error) as e:
        F.Engine(0)
    assert e.value.kind == F.ErrorKind.device


def _invariants(rec):
    t = rec.num_observations()
    assert np.bincount(rec.obs_cam, minlength=rec.num_cameras()).min() >= 4
    assert np.bincount(rec.obs_pt, minlength=rec.num_points()).min() >= 2
    keys = rec.obs_cam.astype(np.int64) << 32 | rec.obs_pt.astype(np.int64)
    assert np.unique(keys).size == t


def test_generators_are_deterministic():
    a = S.generate_random_scene(8, 50, 0.4, 9, 0.5)
    b = S.generate_random_scene(8, 50, 0.4, 9, 0.5)
    assert np.array_equal(a.obs_u, b.obs_u) and np.array_equal(a.cams, b.cams)
    c = S.generate_random_scene(8, 50, 0.4, 10, 0.5)
    assert not np.array_equal(a.obs_u[0], c.obs_u[0])


def test_noise_sets_covariance():  # test_synthetic.cpp:46-56
    noisy = S.generate_cube_scene(5, 0.5)
    assert np.array_equal(noisy.obs_sigma, np.broadcast_to(0.25 * np.eye(2), noisy.obs_sigma.shape))
    clean = S.generate_cube_scene(5, 0.0)
    assert np.array_equal(clean.obs_sigma, np.broadcast_to(np.eye(2), clean.obs_sigma.shape))


@pytest.mark.parametrize("cfg", [1, 2])
def test_baseline_config_scenes(cfg):
    rec = S.generate_config(cfg)
    n, m = {1: (10, 1000), 2: (100, 20000)}[cfg]
    assert rec.cam_params == 9 and rec.num_cameras() == n and rec.num_points() == m
    assert np.all(rec.cams[:, 6] == 1000.0) and not rec.cams[:, 7:].any()
    _invariants(rec)
    k = np.bincount(rec.obs_pt)
    if cfg == 1:
        assert k.min() >= 2 and k.max() <= 10
    else:
        assert k.min() >= 2 and k.max() <= 20 and 3.5 < k.mean() < 4.5  # geometric, mean 4
    again = S.generate_config(cfg)
    assert np.array_equal(again.obs_u, rec.obs_u)


def test_random_scenes_satisfy_invariants():  # test_synthetic.cpp:71-83
    for seed in (1, 2, 3, 4, 5):
        _invariants(S.generate_random_scene(4 + seed * 3, 30 + 10 * seed, 0.5, seed, 0.5))


def test_generator_preconditions():  # test_synthetic.cpp:85-91
    from paper_1808_02414_b200.sfmcov import Error
    for args in ((1, 30, 0.5, 1, 0.0), (5, 7, 0.5, 1, 0.0), (5, 30, 0.0, 1, 0.0), (5, 30, 1.5, 1, 0.0)):
        with pytest.raises(Error):
            S.generate_random_scene(*args)


def test_error_metric_matches_the_restatement():  # oracle.cpp:74-110 (host-only)
    from oracle import oracle as O
    from paper_1808_02414_b200 import sfmcov as F
    rng = np.random.default_rng(3)
    rec = S.generate_random_scene(12, 90, 0.4, 9, 0.5)
    gt = rng.standard_normal((12, 8, 8))
    est = gt + 1e-6 * rng.standard_normal((12, 8, 8))
    r = F.error_metric(gt, est, rec)
    mean, median, per, zero = O.error_metric(gt, est, rec.cams)
    assert np.allclose(r.per_camera, per, rtol=1e-14) and abs(r.mean - mean) < 1e-15 and r.median == median
    assert r.zero_components == zero
