"""Parity evidence at the BASELINE sizes the pytest suite cannot afford.

config 4 (Z 27000^2): the GPU camera blocks against the CPU restatement
    (oracle/, all host cores), relative Frobenius error per camera block.
config 5 (Z 90000^2, 65 GB): no CPU run is affordable (~1e15 flops on the
    host); the single-GPU result is checked against the emulated 2-rank path
    (different Schur reduction split, different dense update grouping) and
    for symmetry / positive definiteness / finiteness of every block.

usage: python tools/parity_big.py 4|5 [out.txt]
"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np

from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import synthetic as S


def rel_blocks(a, b):
    num = np.linalg.norm((a - b).reshape(len(a), -1), axis=1)
    den = np.linalg.norm(b.reshape(len(b), -1), axis=1)
    return num / den


def block_properties(c):
    sym = max(np.abs(b - b.T).max() / np.abs(b).max() for b in c)
    # scale-free: smallest eigenvalue of the block's correlation matrix
    min_eig = min(np.linalg.eigvalsh((0.5 * (b + b.T)) / np.sqrt(np.outer(np.diag(b), np.diag(b)))).min() for b in c)
    return bool(np.isfinite(c).all()), float(sym), float(min_eig)


def main():
    cfg = int(sys.argv[1])
    out = open(sys.argv[2], "w") if len(sys.argv) > 2 else sys.stdout

    def say(*a):
        print(*a, file=out, flush=True)
        if out is not sys.stdout:
            print(*a, flush=True)

    t0 = time.time()
    rec = S.generate_config(cfg)
    say(f"config {cfg}: cameras {rec.num_cameras()} points {rec.num_points()} observations {len(rec.obs_cam)} "
        f"(generated in {time.time() - t0:.1f} s), host cores {os.cpu_count()}")
    eng = F.Engine(0)
    t0 = time.time()
    gpu = eng.compute_covariance(rec).camera_cov
    say(f"gpu compute_covariance {time.time() - t0:.2f} s")
    fin, sym, mine = block_properties(gpu)
    say(f"gpu blocks: finite {fin}, max asymmetry {sym:.2e}, min correlation-matrix eigenvalue {mine:.3e}")
    if cfg == 4:
        from oracle import oracle as O
        cores = os.cpu_count() or 1
        O.lib().oracle_blas_threads(cores)
        t0 = time.time()
        ref, _, _, times = O.compute_covariance(rec, threads=cores)
        say(f"cpu restatement ({cores} threads) {time.time() - t0:.1f} s; stages "
            + ", ".join(f"{k} {v:.2f}" for k, v in times.items()))
        r = rel_blocks(gpu, ref)
        say(f"gpu vs restatement, relative Frobenius per camera block: max {r.max():.3e} median {np.median(r):.3e} "
            f"(camera {int(r.argmax())}); bound 1e-9: {'PASS' if r.max() <= 1e-9 else 'FAIL'}")
    else:
        t0 = time.time()
        emu = eng.compute_covariance_emulated(rec, 2).camera_cov
        say(f"gpu emulated 2 ranks {time.time() - t0:.2f} s")
        r = rel_blocks(emu, gpu)
        say(f"emulated 2-rank vs single GPU, relative Frobenius per camera block: max {r.max():.3e} "
            f"median {np.median(r):.3e}; bound 1e-9: {'PASS' if r.max() <= 1e-9 else 'FAIL'}")


if __name__ == "__main__":
    main()
