import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def _ensure_built():
    libs = [ROOT / "paper_1808_02414_b200" / "libsfmcov_b200.so", ROOT / "paper_1808_02414_b200" / "libsfmcov_synth.so",
            ROOT / "oracle" / "liboracle_sfmcov.so"]
    if not all(p.exists() for p in libs):
        subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.build()"], cwd=ROOT, check=True)


_ensure_built()


@pytest.fixture(scope="session")
def engine():
    from paper_1808_02414_b200 import sfmcov as F
    eng = F.Engine(0)
    yield eng
    eng.close()


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / n) if n > 0 else float(np.linalg.norm(a - b))


def disconnected_scene(seed, noise):
    """Two cube scenes 100 apart sharing nothing: a 14-dim gauge
    (tests/support.hpp:106-122)."""
    from paper_1808_02414_b200 import synthetic as S
    from paper_1808_02414_b200.sfmcov import Reconstruction
    a = S.generate_cube_scene(seed, noise)
    b = S.transform_scene(S.generate_cube_scene(seed + 1, noise), np.eye(3), np.array([100.0, 0, 0]), 1.0)
    return Reconstruction(np.vstack([a.cams, b.cams]), np.vstack([a.pts, b.pts]),
                          np.concatenate([a.obs_cam, b.obs_cam + a.num_cameras()]),
                          np.concatenate([a.obs_pt, b.obs_pt + a.num_points()]),
                          np.vstack([a.obs_u, b.obs_u]), np.concatenate([a.obs_sigma, b.obs_sigma]))
