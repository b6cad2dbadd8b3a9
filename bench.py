#!/usr/bin/env python
"""Benchmark of the B200 camera-covariance hot path (BASELINE.json metric).

One step = one full ``compute_covariance`` of the BASELINE config scene
(default: config 3 — 1000 cameras (P = 9), 200k points, ~1.5M observations,
Z 9000 x 9000): validation, observation index, Jacobian, nullspace, Fisher
blocks, conditioning, Schur reduction, gauge-fixed Cholesky inversion,
per-camera blocks.

* ``value``      device-resident inputs, CUDA events on the library stream.
* ``e2e``        the public C-ABI host call (sfmcov_cuda_compute_covariance)
                 with pinned host scene buffers: H2D of the scene, the whole
                 pipeline and D2H of the camera blocks, host wall clock.
* ``roofline``   the dense FP64 factorisation stage (DMMA GEMM + panel
                 kernels), algorithmic flops N^3/3 (POTRF) + N^3/3 (TRTRI).
* ``cpu_baseline`` / ``--impl reference``: the CPU restatement of the
                 reference path (oracle/, kind "port") on the host cores.

Multi-GPU (torchrun, one process per GPU): by default the sharded pipeline
(csrc/dist.cu) — the camera-pair-sorted observation-pair work split over the
ranks with an NCCL all-reduce of the camera-pair blocks, and the dense
inversion as a 1D block-cyclic fused Cholesky / inverse sweep with an NCCL
panel broadcast per step — on the same scene (strong scaling), timed with
CUDA events as the max over ranks.  ``--mode replicas`` runs independent
single-GPU replicas instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# DRAM bytes (read + write) of one dense sweep, summed over its launches in an
# ncu launch list of this bench command (per config; profiles/ names the file)
SWEEP_DRAM_BYTES = {3: (62780.3e6 / 7, "profiles/r02_launches_bench_config3.txt (sweep DRAM over 7 runs / 7)")}
FP64_PEAK_TFLOPS = 37.1  # measured DMMA throughput on this pool, m8n8k4 and m16n8k16 alike (profiles/r01_fp64_peak_probe.txt)
FP64_PEAK_SOURCE = "measured: tools/probe/fp64_probe.cu DMMA loop 37.1 TF/s, profiles/r01_fp64_peak_probe.txt (cuBLAS DGEMM 16384^3: 36.0; MEASURED_PEAKS.json has no FP64 entry)"


def measured_hbm():
    try:
        return float(json.load(open(ROOT / "MEASURED_PEAKS.json"))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def dist_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def scene_bytes(rec):
    """Bytes the host API copies to the device per call: every scene array but
    the pixels u, which the library only validates (finite) and does so on the
    host while the rest uploads."""
    return (rec.cams.nbytes + rec.pts.nbytes + rec.obs_cam.nbytes + rec.obs_pt.nbytes +
            (rec.obs_sigma.nbytes if rec.obs_sigma is not None else 0))


def panel_width(Npad: int) -> int:
    """Dense panel width of the single-GPU sweep (csrc/capi.cu panel_blocks)."""
    K = Npad // 128
    g = K // 24
    if K >= 60 and g < 4:
        g = 4
    return 128 * min(16, max(3, g))


def workload_name(cfg, rec):
    n, m, t, P = rec.num_cameras(), rec.num_points(), rec.num_observations(), rec.cam_params
    return (f"config{cfg}: {n} cameras (P={P}), {m} points, {t} observations; "
            f"Z {P * n}x{P * n} FP64")


TRS_SAMPLE = 32  # the reference-configuration CPU run samples dsytrs2 at 1/32 and 2/32 of the columns


def cpu_identity():
    """Host CPU model and the OpenBLAS kernel set the restatement runs on."""
    from oracle import oracle as O
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "openblas_corename": O.blas_corename(),
            "OPENBLAS_CORETYPE": os.environ.get("OPENBLAS_CORETYPE")}


def run_cpu(rec, threads: int, blas_threads: int):
    """One full compute_covariance of the CPU restatement (oracle/)."""
    from oracle import oracle as O
    O.lib().oracle_blas_threads(blas_threads)
    t0 = time.perf_counter()
    _, _, _, times = O.compute_covariance(rec, threads=threads)
    return time.perf_counter() - t0, times


def run_cpu_reference(rec, cores: int):
    """The reference's own configuration (src/threading.cpp:14-22, 54-57):
    Jacobian / Fisher / point loops on every core, the serial Schur loop,
    dsytrf + dsytrs2 on ONE BLAS thread.  Bounded sample: dsytrs2 solves
    1/TRS_SAMPLE and then 2/TRS_SAMPLE of the identity's columns and the
    affine fit of the two times gives the full solve (oracle/sfmcov_oracle.cpp,
    g_trs_sample); every other stage runs in full.  Returns (seconds for the
    full workload, stage times with the dsytrs2 samples)."""
    import ctypes as C
    from oracle import oracle as O
    O.lib().oracle_blas_threads(1)
    O.lib().oracle_trs_sample(TRS_SAMPLE)
    try:
        t0 = time.perf_counter()
        _, _, _, times = O.compute_covariance(rec, threads=cores)
        wall = time.perf_counter() - t0
    finally:
        O.lib().oracle_trs_sample(1)
    cols, secs = (C.c_int64 * 2)(), (C.c_double * 2)()
    O.lib().oracle_trs_sample_info(cols, secs)
    times = dict(times)
    sampled = secs[0] + secs[1]
    times["dsytrs2_samples"] = {"columns": [cols[0], cols[1]], "seconds": [secs[0], secs[1]]}
    value = wall - sampled + times["dsytrs2"]  # the two sampled solves replaced by the fitted full solve
    times["total"] = value
    return value, times


def reference_sample_text(cfg, cores):
    return (f"config {cfg} compute_covariance of the CPU restatement (oracle/) in the reference's configuration: "
            f"parallel loops on {cores} threads, serial Schur loop, dsytrf + dsytrs2 on 1 OpenBLAS thread "
            f"(src/threading.cpp:54-57); every stage in full except dsytrs2, timed on 1/{TRS_SAMPLE} and "
            f"2/{TRS_SAMPLE} of the identity's columns and extrapolated to all columns by the affine fit "
            f"(fixed + per-column cost; within 4 % of a full solve at config 3)")


def reference_arm(args, world, rank):
    """--impl reference: the CPU restatement of the reference path on the host
    cores in the reference's own threading (oracle/, kind "port"; the
    reference itself cannot be built here: no Eigen, no lapacke.h)."""
    if rank != 0:
        return
    from paper_1808_02414_b200 import synthetic as S
    cores = os.cpu_count() or 1
    rec = S.generate_config(args.config)
    warm = S.generate_config(1)  # warm-up: the code paths and BLAS on the tiny config
    for _ in range(args.warmup):
        run_cpu_reference(warm, cores)
    ts, stages = [], None
    for _ in range(args.steps):
        dt, stages = run_cpu_reference(rec, cores)
        ts.append(dt)
    v = float(np.mean(ts))
    line = {
        "impl": "reference", "metric": "end-to-end camera-covariance s", "value": v, "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * v,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, rec), "config_index": args.config, "parallelism": "cpu",
                   "warmup_steps": "config 1 (tiny), same code path"},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port",
                         "sample": reference_sample_text(args.config, cores), "stages_s": stages,
                         "host": cpu_identity()},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-blas-threads", type=int, default=0)
    ap.add_argument("--mode", default="sharded", choices=["sharded", "replicas"],
                    help="multi-GPU mode (N > 1): one scene sharded over the ranks, or one replica per rank")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the sharded code path even on one GPU (a one-rank group)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local = dist_setup()
    if args.impl == "reference":
        reference_arm(args, world, rank)
        barrier(world)
        return

    import torch
    from paper_1808_02414_b200 import _native as N
    from paper_1808_02414_b200 import sfmcov as F
    from paper_1808_02414_b200 import synthetic as S

    torch.cuda.set_device(local)
    rec = S.generate_config(args.config)
    eng = F.Engine(local)
    lib = N.cuda_lib()
    sharded = args.mode == "sharded" and (world > 1 or args.force_sharded)
    if sharded:
        from paper_1808_02414_b200 import multi as M
        M.attach(eng, rank, world, device=torch.device("cuda", local))
    dev_fn = lib.sfmcov_cuda_compute_covariance_sharded_device if sharded else lib.sfmcov_cuda_compute_covariance_device
    host_fn = lib.sfmcov_cuda_compute_covariance_sharded if sharded else lib.sfmcov_cuda_compute_covariance
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))

    # device-resident scene
    dev = torch.device("cuda", local)
    tens = {k: torch.from_numpy(getattr(rec, k)).to(dev) for k in ("cams", "pts", "obs_cam", "obs_pt", "obs_u", "obs_sigma")}
    P, n = rec.cam_params, rec.num_cameras()
    d_cov = torch.empty((n, P, P), dtype=torch.float64, device=dev)
    sc = N.Scene()
    sc.n_cams, sc.n_pts, sc.n_obs, sc.cam_params = n, rec.num_points(), rec.num_observations(), P
    sc.cams, sc.pts = tens["cams"].data_ptr(), tens["pts"].data_ptr()
    sc.obs_cam, sc.obs_pt = tens["obs_cam"].data_ptr(), tens["obs_pt"].data_ptr()
    sc.obs_u, sc.obs_sigma = tens["obs_u"].data_ptr(), tens["obs_sigma"].data_ptr()
    torch.cuda.synchronize()
    opts = N.Options(0, 0, 0, 0)
    diag = N.Diagnostics()
    err = N.ErrorStruct()
    import ctypes as C

    def device_step():
        code = dev_fn(eng.handle, C.byref(sc), C.byref(opts), d_cov.data_ptr(), C.byref(diag), C.byref(err))
        if code:
            raise RuntimeError(err.message.decode())

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MiB > L2

    eng.set_profiling(True)
    for _ in range(args.warmup):
        device_step()
    barrier(world)
    torch.cuda.synchronize()
    times, stage_acc = [], {}
    launches = 0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)  # L2 flush between timed steps (outside the events)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                device_step()
                e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            for k, v in eng.stage_times().items():
                stage_acc[k] = stage_acc.get(k, 0.0) + v
            cts = eng.counts()
            launches += cts["kernel_launches"]
    torch.cuda.synchronize()
    barrier(world)
    ms = dist_max(float(np.mean(times)), world)
    counts = eng.counts()
    stages = {k: v / args.steps for k, v in stage_acc.items()}

    # ---- e2e through the public host C ABI with pinned host buffers -------------
    pinned = {}
    for k in ("cams", "pts", "obs_cam", "obs_pt", "obs_u", "obs_sigma"):
        a = getattr(rec, k)
        t = torch.from_numpy(a).pin_memory()
        pinned[k] = t
    host_cov = torch.empty((n, P, P), dtype=torch.float64).pin_memory()
    hs = N.Scene()
    hs.n_cams, hs.n_pts, hs.n_obs, hs.cam_params = n, rec.num_points(), rec.num_observations(), P
    hs.cams, hs.pts = pinned["cams"].data_ptr(), pinned["pts"].data_ptr()
    hs.obs_cam, hs.obs_pt = pinned["obs_cam"].data_ptr(), pinned["obs_pt"].data_ptr()
    hs.obs_u, hs.obs_sigma = pinned["obs_u"].data_ptr(), pinned["obs_sigma"].data_ptr()
    eng.set_profiling(False)

    def host_step():
        code = host_fn(eng.handle, C.byref(hs), C.byref(opts), host_cov.data_ptr(), C.byref(diag), C.byref(err))
        if code:
            raise RuntimeError(err.message.decode())

    for _ in range(2):
        host_step()
    barrier(world)
    e2e = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host_step()
        e2e.append(time.perf_counter() - t0)
    e2e_s = dist_max(float(np.mean(e2e)), world)

    # ---- roofline: dense FP64 factorisation stage ---------------------------------
    N_ = counts["N"]
    Npad = counts["Npad"]
    dense_ms = stages.get("cholesky", 0.0) + stages.get("trtri", 0.0)
    flops = 2.0 * Npad ** 3 / 3.0
    algo_flops = 2.0 * N_ ** 3 / 3.0
    achieved = algo_flops / (dense_ms * 1e-3) / 1e12 if dense_ms > 0 else None
    peak = FP64_PEAK_TFLOPS * (world if sharded else 1)  # the sharded sweep runs on all ranks
    hbm, hbm_src = measured_hbm()
    # Schur stage accounting
    pairs, nnz = counts["obs_pairs"], counts["nnz_blocks"]
    t_obs, m_pts = counts["n_obs"], counts["n_pts"]
    b_schur = t_obs * (2 * (P + 3) * 8 + 4) + m_pts * (3 * 8 + 4) + nnz * P * P * 8 + (P * n * 7 + 49) * 8
    f_schur = 6 * P * P * pairs
    schur_ms = stages.get("schur_point_prep", 0) + stages.get("pair_sort", 0) + stages.get("schur_pair_reduce", 0)
    t_hbm, t_fp64 = b_schur / (hbm * 1e9), f_schur / (FP64_PEAK_TFLOPS * 1e12)
    t_star = max(t_hbm, t_fp64)
    # Jacobian stage bytes and the dense-Z fill, reported separately
    has_sigma = rec.obs_sigma is not None
    b_jac = t_obs * (4 + 4 + 24 * has_sigma) + m_pts * 24 + n * P * 8 + t_obs * 2 * (P + 3) * 8
    jac_ms = stages.get("jacobian", 0.0)
    fill_ms = stages.get("dense_fill", 0.0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        dt, cst = run_cpu_reference(rec, cores)
        cpu = {"value": dt, "unit": "s", "cores": cores, "kind": "port",
               "sample": reference_sample_text(args.config, cores), "stages_s": cst, "host": cpu_identity()}
        # the best this host does with the restatement: every core in BLAS too
        # (not the reference's configuration; reported beside it, labelled)
        dtb, cstb = run_cpu(rec, cores, cores)
        cpu["cpu_best"] = {"value": dtb, "unit": "s", "cores": cores,
                           "sample": f"one full config {args.config} compute_covariance, parallel loops and "
                                     f"dsytrf + dsytrs2 on {cores} OpenBLAS threads (all columns)",
                           "stages_s": cstb}

    if rank == 0:
        out = {
            "metric": "end-to-end camera-covariance s",
            "value": ms * 1e-3,
            "unit": "s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": False,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded BASELINE.json config generator; the paper's datasets are not available)",
            "config": {
                "workload": workload_name(args.config, rec),
                "config_index": args.config,
                "parallelism": (f"sharded{world}: stage A replicated, observation-pair chunks + NCCL reduce-scatter of camera-pair blocks to their column owners; "
                                f"1D block-cyclic Cholesky/inverse sweep with NCCL panel broadcast") if sharded
                               else ("replicas" if world > 1 else "single"),
                "l2": "256 MiB write between timed steps; working set (Z 660 MB) > L2",
                "obs_pairs": pairs, "nnz_camera_blocks": nnz,
                "nnz_block_fraction": nnz / (n * (n + 1) / 2),
            },
            "e2e": {"value": e2e_s, "unit": "s",
                    "h2d_bytes_per_step": scene_bytes(rec), "d2h_bytes_per_step": int(n * P * P * 8),
                    "timing": ("host wall clock around sfmcov_cuda_compute_covariance" + ("_sharded" if sharded else "")
                               + " (pinned host buffers), max over ranks")},
            "gpu_launches": launches,
            "roofline": {
                "kernel": "dense FP64 Cholesky + triangular inverse (k_gemm DMMA m16n8k16 + k_potrf_diag)",
                "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if achieved else None,
                "traffic": SWEEP_DRAM_BYTES.get(args.config, (None, None))[0],
                "traffic_source": SWEEP_DRAM_BYTES.get(args.config, (None, None))[1],
                "algorithmic_bytes": 8.0 * N_ * N_,
                "traffic_model": 16.0 * Npad ** 3 / (3.0 * panel_width(Npad)) + 8.0 * Npad * Npad,
                "traffic_note": ("algorithmic_bytes: the compulsory N^2/2 doubles of Z read and of X = L^-1 written; "
                                 "traffic: DRAM read+write summed over one sweep's launches in the ncu launch list "
                                 "(traffic_source; null for configs without one); traffic_model: the right-looking "
                                 "sweep streams the trailing lower triangle once per W-column panel for the "
                                 "Cholesky and once for the inverse, 16 N^3 / (3 W) B, W = panel width"),
                "peak_source": FP64_PEAK_SOURCE,
                "algorithmic_flops": algo_flops, "executed_flops_padded": flops,
                "stage_ms": dense_ms,
            },
            "jacobian_stage": {"GB_per_s": b_jac / (jac_ms * 1e-3) / 1e9 if jac_ms else None, "bytes": b_jac,
                               "stage_ms": jac_ms, "hbm_frac": (b_jac / (hbm * 1e9)) / (jac_ms * 1e-3) if jac_ms else None},
            "dense_fill": {"GB_per_s": Npad * Npad * 4 / (fill_ms * 1e-3) / 1e9 if fill_ms else None,
                           "note": "lower triangle of the padded Z written once (N^2/2 x 8 B)", "stage_ms": fill_ms},
            "schur": {
                "hbm_frac": (t_hbm * 1e3) / schur_ms if schur_ms else None,
                "fp64_frac": (t_fp64 * 1e3) / schur_ms if schur_ms else None,
                "binding": "fp64" if t_fp64 >= t_hbm else "hbm",
                "obs_pairs_per_s": pairs / (schur_ms * 1e-3) if schur_ms else None,
                "GB_per_s": b_schur / (schur_ms * 1e-3) / 1e9 if schur_ms else None,
                "roofline_time_ms": t_star * 1e3, "frac": (t_star * 1e3) / schur_ms if schur_ms else None,
                "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src, "bytes": b_schur, "flops": f_schur,
                "stage_ms": schur_ms,
                "stage_note": ("point prep + pair-list wait + pair reduction; the pair reduction of the block "
                               "columns beyond the first panel runs on a second stream beside the first panel's "
                               "factorisation and is counted here in full (its time also lies inside the "
                               "cholesky stage, which the roofline above therefore understates)"),
            },
            "inversion": {"TFLOP_per_s": achieved, "frac_fp64": achieved / peak if achieved else None},
            "stages_ms": stages,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    barrier(world)


if __name__ == "__main__":
    main()
