"""Golden fixtures (tests/golden/make_golden.py): the seeded generators and
the CPU restatement reproduce them exactly.  CPU only."""
from pathlib import Path

import numpy as np
import pytest

from conftest import rel
from oracle import oracle as O
from paper_1808_02414_b200.sfmcov import Reconstruction

GOLDEN = Path(__file__).resolve().parent / "golden"
FIXTURES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load(name):
    g = dict(np.load(GOLDEN / f"{name}.npz"))
    rec = Reconstruction(g["cams"], g["pts"], g["obs_cam"], g["obs_pt"], g["obs_u"], g["obs_sigma"])
    return rec, g


@pytest.mark.parametrize("name", FIXTURES)
def test_generator_reproduces_fixture(name):
    import sys
    sys.path.insert(0, str(GOLDEN))
    from make_golden import SCENES
    rec, g = load(name)
    fresh = SCENES[name]()
    for k in ("cams", "pts", "obs_cam", "obs_pt", "obs_u", "obs_sigma"):
        assert np.array_equal(getattr(fresh, k), g[k]), k


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_reproduces_fixture(name):
    rec, g = load(name)
    jc, jp = O.jacobian(rec)
    assert np.array_equal(jc, g["jc"]) and np.array_equal(jp, g["jp"])
    H, _ = O.nullspace(rec)
    assert np.array_equal(H, g["H"])
    D, A, Cp, sa, sb, _ = O.fisher(rec)
    assert np.array_equal(D, g["D"]) and np.array_equal(A, g["A"]) and np.array_equal(sa, g["s_a"])
    assert np.array_equal(O.schur(rec), g["z_p"])
    cov, d, _, _ = O.compute_covariance(rec)
    assert max(rel(a, b) for a, b in zip(cov, g["cov"])) < 1e-13
    assert [d.inertia_positive, d.inertia_negative] == list(g["inertia"])
