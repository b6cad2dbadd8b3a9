"""Per-camera error of the FP64 pipeline (and of the restatement's reference
route) against the exact inverse of the bordered Fisher system, computed by
the GPU's double-double refinement (sfmcov_cuda_refine_covariance).

usage: python tools/truth_gpu.py SCENE [SCENE ...] [--restatement] [--sample K] [--iters I]
SCENE: cube | small | c1..c5 | readme (the reference README scale point, P=8)
Writes gpurun_out/truth_<scene>.npz and prints one summary line per scene.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np

from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import synthetic as S


def scene(name):
    if name == "cube":
        return S.generate_cube_scene(1, 0.5)
    if name == "small":
        return S.generate_random_scene(12, 150, 0.3, 5, 0.5)
    if name == "readme":  # proj/README.md:21-23, tests/acceptance.cpp:237-262
        return S.generate_random_scene(1000, 100000, 0.008, 3, 0.5)
    return S.generate_config(int(name[1:]))


def rel(a, b):
    return np.linalg.norm((a - b).reshape(len(a), -1), axis=1) / np.linalg.norm(b.reshape(len(b), -1), axis=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("scenes", nargs="+")
    ap.add_argument("--restatement", action="store_true")
    ap.add_argument("--sample", type=int, default=0)
    ap.add_argument("--iters", type=int, default=4)
    a = ap.parse_args()
    eng = F.Engine(0)
    os.makedirs("gpurun_out", exist_ok=True)
    for name in a.scenes:
        rec = scene(name)
        n = rec.num_cameras()
        cams = np.arange(n, dtype=np.int32)
        if a.sample and a.sample < n:
            cams = np.sort(np.random.default_rng(0).choice(n, a.sample, replace=False)).astype(np.int32)
        t0 = time.time()
        truth, base, hist = eng.refine_covariance(rec, cams, a.iters)
        t_ref = time.time() - t0
        e_gpu = rel(base, truth)
        line = (f"{name}: n={n} P={rec.cam_params} cams={len(cams)} refine {t_ref:.1f}s hist "
                + " ".join(f"{h:.1e}" for h in hist)
                + f" | gpu vs truth max {e_gpu.max():.3e} median {np.median(e_gpu):.3e} >1e-9: {(e_gpu > 1e-9).sum()}")
        out = {"cams": cams, "truth": truth, "gpu": base, "hist": hist}
        if name in ("cube", "small"):
            from oracle import oracle as O
            ex = O.exact_camera_blocks(rec, 5000)[cams]
            line += f" | truth vs CPU long double {rel(truth, ex).max():.3e}"
        if a.restatement:
            from oracle import oracle as O
            t1 = time.time()
            ref = O.compute_covariance(rec)[0][cams]
            e_ref = rel(ref, truth)
            line += (f" | restatement (dsytrf route) vs truth max {e_ref.max():.3e} median {np.median(e_ref):.3e} "
                     f">1e-9: {(e_ref > 1e-9).sum()} ({time.time() - t1:.0f}s)")
            out["restatement"] = ref
        np.savez(f"gpurun_out/truth_{name}.npz", **out)
        print(line, flush=True)


if __name__ == "__main__":
    main()
