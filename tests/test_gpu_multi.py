"""GPU tests of the multi-GPU code path (csrc/dist.cu): the pair-chunk
sharded Schur assembly, the 1D block-cyclic fused Cholesky / inverse sweep and
the output all-reduces, with R ranks emulated on the one GPU of the test box
(in-process panel copies in place of ncclBroadcast; the rest of the code is
the path a multi-process NCCL run takes).  Bars as for the single-GPU path:
camera blocks within 1e-9 of the CPU restatement."""
import numpy as np
import pytest

from conftest import disconnected_scene, rel
from oracle import oracle as O
from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import synthetic as S

pytestmark = pytest.mark.gpu
COV_TOL = 1e-9

SCENES = {
    "cube_p8": lambda: S.generate_cube_scene(1, 0.5),
    "ring_p9": lambda: S.generate_random_scene(16, 200, 0.3, 4, 0.7, 9),
    "ring64_p8": lambda: S.generate_random_scene(64, 200, 0.40625, 13, 0.5),
    "config1": lambda: S.generate_config(1),
    "config2": lambda: S.generate_config(2),
}


def worst_block(a, b):
    return max(rel(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("ranks", [1, 2, 3, 5])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_emulated_ranks_match_restatement(engine, name, ranks):
    rec = SCENES[name]()
    cov, d, flagged, _ = O.compute_covariance(rec)
    res = engine.compute_covariance_emulated(rec, ranks)
    assert worst_block(res.camera_cov, cov) <= COV_TOL
    g = res.diagnostics
    assert (g.inertia_positive, g.inertia_negative) == (d.inertia_positive, d.inertia_negative)
    assert g.negative_eigenvalue_warnings == d.negative_eigenvalue_warnings == 0
    assert g.flagged_columns == flagged
    for c in res.camera_cov:
        assert np.abs(c - c.T).max() <= 1e-14 * np.abs(c).max() and np.diag(c).min() > 0


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_config3_emulated_matches_single_gpu(engine, ranks):
    rec = S.generate_config(3)
    one = engine.compute_covariance(rec)
    many = engine.compute_covariance_emulated(rec, ranks)
    assert worst_block(many.camera_cov, one.camera_cov) <= COV_TOL  # two FP64 orderings; same bar as parity
    assert many.diagnostics.min_pivot == pytest.approx(one.diagnostics.min_pivot, rel=1e-9)
    assert many.diagnostics.max_pivot == pytest.approx(one.diagnostics.max_pivot, rel=1e-9)


def test_emulated_result_is_independent_of_rank_count_up_to_rounding(engine):
    rec = S.generate_config(2)
    base = engine.compute_covariance_emulated(rec, 1).camera_cov
    for r in (2, 3, 4, 6):
        assert worst_block(engine.compute_covariance_emulated(rec, r).camera_cov, base) <= 1e-10
    again = engine.compute_covariance_emulated(rec, 3).camera_cov
    assert np.array_equal(again, engine.compute_covariance_emulated(rec, 3).camera_cov)  # run to run bitwise


def test_single_rank_sharded_api_equals_emulated(engine):
    rec = S.generate_config(1)
    engine.comm_init(bytes(128), 1, 0)
    a = engine.compute_covariance_sharded(rec).camera_cov
    b = engine.compute_covariance_emulated(rec, 1).camera_cov
    assert np.array_equal(a, b)


def test_emulated_disconnected_scene_fails_in_factorization(engine):
    with pytest.raises(F.Error) as e:
        engine.compute_covariance_emulated(disconnected_scene(4, 0.5), 2)
    assert e.value.kind == F.ErrorKind.degenerate and e.value.stage == "factorization"


def _behind_camera(rec):
    rec.pts[5] = rec.cams[0, 3:6]
    return rec


def _two_behind(rec):  # failing observations in points owned by different ranks
    rec.pts[5] = rec.cams[0, 3:6]
    rec.pts[12] = rec.cams[2, 3:6]
    return rec


def _singular_point(rec):  # test_schur.cpp:82-93 (as in test_gpu_parity.py)
    m = rec.num_points()
    rec.cams = np.vstack([rec.cams, rec.cams[0]])
    rec.cams[6, 7] = 0.0
    rec.pts = np.vstack([rec.pts, np.array([rec.cams[0, 3:6] * 0.5])])
    rec.obs_cam = np.concatenate([rec.obs_cam, [0, 6, 6, 6, 6]]).astype(np.int32)
    rec.obs_pt = np.concatenate([rec.obs_pt, [m, m, 0, 1, 2]]).astype(np.int32)
    rec.obs_u = np.vstack([rec.obs_u, np.zeros((5, 2))])
    rec.obs_sigma = np.concatenate([rec.obs_sigma, np.broadcast_to(np.eye(2), (5, 2, 2))])
    return rec


@pytest.fixture(params=[False, True], ids=["replicated_a", "sharded_a"])
def stage_a(engine, request):
    """Run a test with both multi-GPU stage-A modes."""
    engine.set_sharded_stage_a(request.param)
    yield request.param
    engine.set_sharded_stage_a(False)


@pytest.mark.parametrize("ranks", [2, 3])
@pytest.mark.parametrize("mutate", [_behind_camera, _two_behind, _singular_point,
                                    lambda r: (r.cams.__setitem__((1, 6), -1.0), r)[1]],
                         ids=["behind_camera", "two_behind", "singular_point", "validation"])
def test_multi_gpu_path_reports_the_single_gpu_error(engine, stage_a, mutate, ranks):
    """Errors are reported with the global observation / point ids, first
    failing index over all ranks, exactly as the single-GPU pipeline words
    them -- also when a rank finds them inside its own point shard."""
    rec = mutate(S.generate_cube_scene(4, 0.5))
    with pytest.raises(F.Error) as e1:
        engine.compute_covariance(rec)
    with pytest.raises(F.Error) as e2:
        engine.compute_covariance_emulated(rec, ranks)
    assert (e2.value.kind, e2.value.stage, str(e2.value)) == (e1.value.kind, e1.value.stage, str(e1.value))


@pytest.mark.parametrize("ranks", [2, 5])
def test_multi_gpu_path_diagnostics(engine, stage_a, ranks):
    rec = S.generate_config(2)
    one = engine.compute_covariance(rec).diagnostics
    many = engine.compute_covariance_emulated(rec, ranks).diagnostics
    assert many.scale_max == pytest.approx(one.scale_max, rel=1e-12)
    assert many.scale_min == pytest.approx(one.scale_min, rel=1e-12)
    assert many.flagged_columns == one.flagged_columns
    assert (many.inertia_positive, many.inertia_negative) == (one.inertia_positive, one.inertia_negative)


def test_replicated_and_sharded_stage_a_agree_on_a_well_conditioned_scene(engine):
    rec = S.generate_config(2)
    rep = engine.compute_covariance_emulated(rec, 3).camera_cov
    engine.set_sharded_stage_a(True)
    try:
        shard = engine.compute_covariance_emulated(rec, 3).camera_cov
    finally:
        engine.set_sharded_stage_a(False)
    assert worst_block(shard, rep) <= 1e-10


def test_config4_multi_gpu_path_within_1e9_of_the_exact_inverse(engine):
    """The default (replicated stage A) multi-GPU path at config 4 against the
    exact inverse on the cameras where it departs most from one GPU: within
    the north_star's 1e-9 (measured 2.3e-10 / 8.2e-10 / 5.0e-10 at R = 2 / 4 /
    8; the point-sharded stage A reaches 1.2e-8 here)."""
    rec = S.generate_config(4)
    one = engine.compute_covariance(rec).camera_cov
    many = {R: engine.compute_covariance_emulated(rec, R).camera_cov for R in (2, 8)}
    worst = set()
    for R, c in many.items():
        e = np.linalg.norm((c - one).reshape(len(one), -1), axis=1) / np.linalg.norm(one.reshape(len(one), -1), axis=1)
        worst |= set(np.argsort(-e)[:12].tolist())
    cams = np.array(sorted(worst), dtype=np.int32)
    truth, _, hist = engine.refine_covariance(rec, cams, 3)
    assert hist[-1] <= 1e-14
    for R, c in many.items():
        assert max(rel(a, b) for a, b in zip(c[cams], truth)) <= 1e-9, R


def test_emulated_rank_bounds(engine):
    with pytest.raises(F.Error):
        engine.compute_covariance_emulated(S.generate_cube_scene(1, 0.5), 0)


# ---- two processes, two GPUs, NCCL (skipped on a one-GPU box) ----------------------
def _nccl_worker(rank, world, port, configs, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_1808_02414_b200 import multi as M
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        eng = F.Engine(rank)
        M.attach(eng, rank, world, device=torch.device("cuda", rank))
        out = {}
        for c in configs:
            rec = S.generate_config(c)
            a = eng.compute_covariance_sharded(rec).camera_cov
            b = eng.compute_covariance_sharded(rec).camera_cov
            out[c] = (a, bool(np.array_equal(a, b)))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_process_nccl_matches_single_gpu(engine):
    """The real NCCL data plane (panel broadcasts, pair-block and output
    all-reduces) across two processes on two GPUs: the sharded result is
    within 1e-10 of the single-GPU pipeline and bitwise repeatable."""
    import socket

    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (the round-end box has one)")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    configs = [2, 3]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, configs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for c in configs:
        single = engine.compute_covariance(S.generate_config(c)).camera_cov
        for r in range(2):
            blocks, repeat = res[r][c]
            assert repeat
            assert worst_block(blocks, single) <= 1e-10
        assert np.array_equal(res[0][c][0], res[1][c][0])  # every rank returns every block
