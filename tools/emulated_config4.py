"""Accuracy of the multi-GPU code path (emulated ranks) at config 4 against
the exact inverse (double-double refinement) on the cameras where it departs
most from the single-GPU result.  usage: python tools/emulated_config4.py [R ...]"""
import os, sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_1808_02414_b200 import sfmcov as F, synthetic as S


def rel(a, b):
    return np.linalg.norm((a - b).reshape(len(a), -1), axis=1) / np.linalg.norm(b.reshape(len(b), -1), axis=1)


rec = S.generate_config(4)
eng = F.Engine(0)
one = eng.compute_covariance(rec).camera_cov
Rs = [int(a) for a in sys.argv[1:]] or [2, 8]
many = {R: eng.compute_covariance_emulated(rec, R).camera_cov for R in Rs}
worst = set()
for R in Rs:
    worst |= set(np.argsort(-rel(many[R], one))[:12].tolist())
cams = np.array(sorted(worst), dtype=np.int32)
truth, base, hist = eng.refine_covariance(rec, cams, 3)
print("cameras", len(cams), "single vs truth max", rel(one[cams], truth).max(), flush=True)
for R in Rs:
    print(f"R={R}: vs single max {rel(many[R], one).max():.3e}; vs truth max {rel(many[R][cams], truth).max():.3e}",
          flush=True)
