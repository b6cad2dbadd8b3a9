"""Generates the committed golden fixtures (tests/golden/*.npz) from the CPU
restatement (oracle/) on small seeded scenes.  Run from the repo root:
    python tests/golden/make_golden.py
The fixtures pin the oracle and the scene generators against regressions and
give the GPU parity tests inputs/outputs that do not depend on re-running the
oracle.  (The reference ships no golden vectors of its own.)"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_1808_02414_b200 import synthetic as S  # noqa: E402

SCENES = {
    "cube_p8": lambda: S.generate_cube_scene(1, 0.5),
    "ring_p8": lambda: S.generate_random_scene(12, 90, 0.4, 9, 0.5),
    "ring_p9": lambda: S.generate_random_scene(10, 80, 0.4, 6, 0.5, 9),
    "config1_p9": lambda: S.generate_config(1),
}


def make(name, rec):
    jc, jp = O.jacobian(rec)
    H, res = O.nullspace(rec)
    D, A, Cp, sa, sb, flagged = O.fisher(rec)
    z = O.schur(rec)
    cov, d, _, _ = O.compute_covariance(rec)
    out = dict(cams=rec.cams, pts=rec.pts, obs_cam=rec.obs_cam, obs_pt=rec.obs_pt, obs_u=rec.obs_u,
               obs_sigma=rec.obs_sigma, jc=jc, jp=jp, H=H, D=D, A=A, s_a=sa, s_b=sb, z_p=z, cov=cov,
               inertia=np.array([d.inertia_positive, d.inertia_negative]), dense_dim=np.array([d.largest_dense_dim]))
    np.savez_compressed(ROOT / "tests" / "golden" / f"{name}.npz", **out)


if __name__ == "__main__":
    for name, fn in SCENES.items():
        make(name, fn())
        print("wrote", name)
