"""Sub-reconstruction covariances (reference include/sfmcov/subrec.hpp):
view graph, greedy neighborhoods, seeded coverings and the per-camera
aggregation of many independent sub-scene covariances, batched on the GPU.
Thin wrappers over the C ABI (csrc/subrec.cpp)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .sfmcov import Engine, Error, Reconstruction, _raise, default_engine


@dataclass
class ViewGraph:
    n_cams: int
    edges: List[List[Tuple[int, int]]]  # per camera: (neighbor, weight), ascending neighbor


@dataclass
class SubScene:
    cameras: np.ndarray  # ascending global ids
    points: np.ndarray
    scene: Reconstruction
    component_truncated: bool


@dataclass
class AggregatedCovariance:
    target_size: int
    cov: np.ndarray       # (n, P, P): the kept block per camera
    trace: np.ndarray     # (n,)
    subset_id: np.ndarray  # (n,)


@dataclass
class MonotonicityReport:
    violations: List[Tuple[int, float, float]]  # (camera, trace_small, trace_large)
    cameras_checked: int


def build_view_graph(rec: Reconstruction, min_covis: int = 1, engine: Optional[Engine] = None) -> ViewGraph:
    """build_view_graph (src/subrec.cpp:90-116); with an engine, counted on
    the device from the covariance pipeline's sorted pair list."""
    n, t = rec.num_cameras(), rec.num_observations()
    cap = max(1, 2 * t * 20)
    off = np.zeros(n + 1, np.int64)
    nbr = np.zeros(cap, np.int32)
    w = np.zeros(cap, np.int32)
    cnt = C.c_int64()
    err = N.ErrorStruct()
    sc = rec.c_struct()
    if engine is not None:
        _raise(N.cuda_lib().sfmcov_cuda_view_graph(engine.handle, C.byref(sc), min_covis, off.ctypes.data,
                                                   nbr.ctypes.data, w.ctypes.data, cap, C.byref(cnt), C.byref(err)),
               err)
    else:
        _raise(N.cuda_lib().sfmcov_view_graph(C.byref(sc), min_covis, off.ctypes.data, nbr.ctypes.data,
                                              w.ctypes.data, cap, C.byref(cnt), C.byref(err)), err)
    if cnt.value > cap:
        raise Error(5, "subrec", "view graph larger than the buffer")
    return ViewGraph(n, [[(int(nbr[k]), int(w[k])) for k in range(off[i], off[i + 1])] for i in range(n)])


def induced_scene(rec: Reconstruction, cameras: np.ndarray, points: np.ndarray) -> Reconstruction:
    """The sub-reconstruction on the given (already filtered) camera / point ids."""
    cl = -np.ones(rec.num_cameras(), np.int64)
    pl = -np.ones(rec.num_points(), np.int64)
    cl[cameras] = np.arange(len(cameras))
    pl[points] = np.arange(len(points))
    keep = (cl[rec.obs_cam] >= 0) & (pl[rec.obs_pt] >= 0)
    return Reconstruction(rec.cams[cameras].copy(), rec.pts[points].copy(), cl[rec.obs_cam[keep]].astype(np.int32),
                          pl[rec.obs_pt[keep]].astype(np.int32),
                          None if rec.obs_u is None else rec.obs_u[keep].copy(),
                          None if rec.obs_sigma is None else rec.obs_sigma[keep].copy())


def extract_neighborhood(rec: Reconstruction, center: int, k_bar: int) -> SubScene:
    n, m = rec.num_cameras(), rec.num_points()
    cams = np.zeros(max(1, n), np.int32)
    pts = np.zeros(max(1, m), np.int32)
    nc, npt, tr = C.c_int64(), C.c_int64(), C.c_int32()
    err = N.ErrorStruct()
    sc = rec.c_struct()
    _raise(N.cuda_lib().sfmcov_extract_neighborhood(C.byref(sc), center, k_bar, cams.ctypes.data, C.byref(nc),
                                                    pts.ctypes.data, C.byref(npt), C.byref(tr), C.byref(err)), err)
    cams, pts = cams[:nc.value].copy(), pts[:npt.value].copy()
    return SubScene(cams, pts, induced_scene(rec, cams, pts), bool(tr.value))


def plan_coverage(rec: Reconstruction, k_bar: int, seed: int) -> List[np.ndarray]:
    n = rec.num_cameras()
    cap_s, cap_c = max(1, n), max(1, n * n)
    off = np.zeros(cap_s + 1, np.int64)
    cams = np.zeros(cap_c, np.int32)
    ns = C.c_int64()
    err = N.ErrorStruct()
    sc = rec.c_struct()
    _raise(N.cuda_lib().sfmcov_plan_coverage(C.byref(sc), k_bar, seed, off.ctypes.data, cap_s, cams.ctypes.data,
                                             cap_c, C.byref(ns), C.byref(err)), err)
    return [cams[off[i]:off[i + 1]].copy() for i in range(ns.value)]


def approximate_covariances(rec: Reconstruction, k_bar: int, n_decompositions: int, seed: int, workers: int = 4,
                            engine: Optional[Engine] = None) -> AggregatedCovariance:
    engine = engine or default_engine()
    n, P = rec.num_cameras(), rec.cam_params
    cov = np.zeros((max(1, n), P, P))
    tr = np.zeros(max(1, n))
    sid = -np.ones(max(1, n), np.int32)
    err = N.ErrorStruct()
    sc = rec.c_struct()
    _raise(N.cuda_lib().sfmcov_cuda_approximate_covariances(engine.handle, C.byref(sc), k_bar, n_decompositions, seed,
                                                            workers, cov.ctypes.data, tr.ctypes.data, sid.ctypes.data,
                                                            C.byref(err)), err)
    return AggregatedCovariance(k_bar, cov[:n], tr[:n], sid[:n])


@dataclass
class ShardResult:
    """One rank's part of a sharded approximate_covariances call."""
    cov: np.ndarray        # (n, P, P): the smallest-trace block among this rank's subsets (zeros where none)
    trace: np.ndarray      # (n,): its trace (+inf where none)
    subset_id: np.ndarray  # (n,): its subset id (-1 where none)
    code: int = 0          # 0, or the error kind of this rank's first failing step
    failed_key: int = -1   # the failure's place in the reference's order (-1: before any covering)
    stage: str = ""
    message: str = ""


def approximate_covariances_shard(rec: Reconstruction, k_bar: int, n_decompositions: int, seed: int, nranks: int,
                                  rank: int, workers: int = 4, engine: Optional[Engine] = None) -> ShardResult:
    """This rank's share of approximate_covariances (subset i of covering d
    goes to rank (i * n_decompositions + d) mod nranks); errors are returned,
    not raised, so that merge_shards reports the first failing subset of all
    ranks as the single call does."""
    engine = engine or default_engine()
    n, P = rec.num_cameras(), rec.cam_params
    cov = np.zeros((max(1, n), P, P))
    tr = np.zeros(max(1, n))
    sid = -np.ones(max(1, n), np.int32)
    failed = C.c_int64(-1)
    err = N.ErrorStruct()
    sc = rec.c_struct()
    code = N.cuda_lib().sfmcov_cuda_approximate_covariances_shard(
        engine.handle, C.byref(sc), k_bar, n_decompositions, seed, workers, nranks, rank, cov.ctypes.data,
        tr.ctypes.data, sid.ctypes.data, C.byref(failed), C.byref(err))
    msg = err.message.decode(errors="replace") if code else ""
    stage = err.stage.decode(errors="replace") if code else ""
    return ShardResult(cov[:n], tr[:n], sid[:n], int(code), int(failed.value), stage, msg)


def merge_shards(parts: List[ShardResult], k_bar: int) -> AggregatedCovariance:
    """The single-call result from the ranks' partial aggregates: per camera
    the smallest (trace, subset id) -- the reference keeps a camera's block
    from the earliest subset with the smallest trace.  Errors: the one with
    the smallest failed_key over all ranks -- the reference draws covering d,
    then computes its subsets, covering after covering, and stops at the
    first failure (an error before any covering, key -1, is the same on
    every rank)."""
    failed = [p for p in parts if p.code]
    if failed:
        first = min(failed, key=lambda p: p.failed_key)  # -1 (before any covering) first: the same on every rank
        raise Error(first.code, first.stage, first.message)
    tr = np.stack([p.trace for p in parts])            # (R, n)
    sid = np.stack([p.subset_id for p in parts]).astype(np.int64)
    big = np.iinfo(np.int64).max
    key_sid = np.where(sid >= 0, sid, big)
    order = np.lexsort((key_sid, tr), axis=0)[0]       # per camera: the rank with the smallest (trace, sid)
    cams = np.arange(tr.shape[1])
    best_sid = sid[order, cams]
    if np.any(best_sid < 0):
        i = int(np.nonzero(best_sid < 0)[0][0])
        raise Error(3, "subrec", f"subrec: camera {i} was not covered by any subset")
    cov = np.stack([p.cov for p in parts])[order, cams]
    return AggregatedCovariance(k_bar, cov, tr[order, cams], best_sid.astype(np.int32))


def approximate_covariances_distributed(rec: Reconstruction, k_bar: int, n_decompositions: int, seed: int,
                                        workers: int = 4, engine: Optional[Engine] = None,
                                        group=None) -> AggregatedCovariance:
    """approximate_covariances over the ranks of a torch.distributed group
    (one process per GPU): each rank computes its share, the partial
    aggregates are all-gathered (tiny: n x (P^2 + 2) values per rank) and
    merged; every rank returns the single-call result."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    part = approximate_covariances_shard(rec, k_bar, n_decompositions, seed, world, rank, workers, engine)
    return gather_and_merge(part, k_bar, group)


def gather_and_merge(part: ShardResult, k_bar: int, group=None) -> AggregatedCovariance:
    """All-gather every rank's ShardResult over a torch.distributed group
    (any backend: the payload goes through all_gather_object) and merge."""
    import torch.distributed as dist
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, part, group=group)
    return merge_shards(parts, k_bar)


def shard_owner(subset_index: int, decomposition: int, n_decompositions: int, nranks: int) -> int:
    """The rank that computes subset `subset_index` of covering
    `decomposition` (csrc/subrec.cpp, pipelined_covariances)."""
    return (subset_index * n_decompositions + decomposition) % nranks


@dataclass
class SweepRow:
    k_bar: int
    subset_id: int
    camera_id: int
    err_relative: float
    err_absolute: float
    trace: float


def error_size_sweep(rec: Reconstruction, sizes: List[int], subsets_per_size: int, seed: int, workers: int = 4,
                     engine: Optional[Engine] = None) -> List[SweepRow]:
    """Per window size, seeded random centers; every subset camera's block
    against the full-scene block (src/subrec.cpp:258-297)."""
    engine = engine or default_engine()
    sz = np.ascontiguousarray(sizes, np.int32)
    cap = max(1, int(sum(int(k) for k in sizes) * subsets_per_size))
    ints = np.zeros((cap, 3), np.int32)
    vals = np.zeros((cap, 3))
    nrows = C.c_int64()
    err = N.ErrorStruct()
    sc = rec.c_struct()
    _raise(N.cuda_lib().sfmcov_cuda_error_size_sweep(engine.handle, C.byref(sc), sz.ctypes.data, len(sz),
                                                     subsets_per_size, seed, workers, ints.ctypes.data,
                                                     vals.ctypes.data, cap, C.byref(nrows), C.byref(err)), err)
    k = min(nrows.value, cap)
    return [SweepRow(int(ints[i, 0]), int(ints[i, 1]), int(ints[i, 2]), float(vals[i, 0]), float(vals[i, 1]),
                     float(vals[i, 2])) for i in range(k)]


def write_sweep_csv(rows: List[SweepRow], path: str) -> None:
    """The reference's CSV layout (src/subrec.cpp:299-312), %.17g numbers."""
    try:
        with open(path, "w") as f:
            f.write("kbar,subset_id,camera_id,err_relative,err_absolute,trace\n")
            for r in rows:
                f.write(f"{r.k_bar},{r.subset_id},{r.camera_id},{r.err_relative:.17g},{r.err_absolute:.17g},"
                        f"{r.trace:.17g}\n")
    except OSError as e:
        raise Error(1, "subrec", f"cannot open '{path}' for writing") from e


def monotonicity_check(rec: Reconstruction, small: SubScene, large: SubScene, rel_tol: float = 1e-8,
                       engine: Optional[Engine] = None) -> MonotonicityReport:
    engine = engine or default_engine()
    sc_ = np.ascontiguousarray(small.cameras, np.int32)
    lc = np.ascontiguousarray(large.cameras, np.int32)
    k = max(1, len(sc_))
    vc, ts, tl = np.zeros(k, np.int32), np.zeros(k), np.zeros(k)
    nv, checked = C.c_int64(), C.c_int64()
    err = N.ErrorStruct()
    sc = rec.c_struct()
    _raise(N.cuda_lib().sfmcov_cuda_monotonicity_check(engine.handle, C.byref(sc), sc_.ctypes.data, len(sc_),
                                                       lc.ctypes.data, len(lc), rel_tol, vc.ctypes.data, ts.ctypes.data,
                                                       tl.ctypes.data, C.byref(nv), C.byref(checked), C.byref(err)), err)
    return MonotonicityReport([(int(vc[i]), float(ts[i]), float(tl[i])) for i in range(nv.value)], checked.value)
