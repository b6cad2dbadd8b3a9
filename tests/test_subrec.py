"""Sub-reconstructions (reference include/sfmcov/subrec.hpp; tests ported
from tests/test_subrec.cpp).  Planner checks run on CPU; the batched GPU
covariances are checked against the CPU restatement per sub-scene."""
import numpy as np
import pytest

from conftest import rel
from oracle import oracle as O
from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import subrec as R
from paper_1808_02414_b200 import synthetic as S


def covis_count(rec, a, b):  # test_subrec.cpp:23-33
    pa = set(rec.obs_pt[rec.obs_cam == a].tolist())
    pb = set(rec.obs_pt[rec.obs_cam == b].tolist())
    return len(pa & pb)


def connected(graph, cams):  # test_subrec.cpp:41-55
    inside = set(int(c) for c in cams)
    seen, stack = {int(cams[0])}, [int(cams[0])]
    while stack:
        c = stack.pop()
        for nb, _ in graph.edges[c]:
            if nb in inside and nb not in seen:
                seen.add(nb)
                stack.append(nb)
    return len(seen) == len(cams)


def points_of(rec, cams):
    m = np.isin(rec.obs_cam, cams)
    cnt = np.bincount(rec.obs_pt[m], minlength=rec.num_points())
    return np.nonzero(cnt >= 2)[0].astype(np.int32)


def test_view_graph_counts_co_observed_points():  # test_subrec.cpp:64-87
    rec = S.generate_random_scene(20, 150, 0.3, 5, 0.5)
    g = R.build_view_graph(rec)
    assert g.n_cams == 20
    for a in range(20):
        nbrs = [b for b, _ in g.edges[a]]
        assert nbrs == sorted(nbrs)
        for b in range(20):
            if a == b:
                continue
            w = dict(g.edges[a]).get(b, 0)
            assert w == covis_count(rec, a, b)
    strict = R.build_view_graph(rec, min_covis=5)
    for a in range(20):
        assert all(w >= 5 for _, w in strict.edges[a])


def test_components_stay_separate():  # test_subrec.cpp:89-96
    from conftest import disconnected_scene
    rec = disconnected_scene(4, 0.5)
    g = R.build_view_graph(rec)
    n = rec.num_cameras()
    half = n // 2
    for a in range(half):
        assert all(b < half for b, _ in g.edges[a])


def test_window_as_large_as_the_scene_reproduces_it():  # test_subrec.cpp:98-112
    rec = S.generate_cube_scene(3, 0.5)
    for k_bar in (6, 100):
        sub = R.extract_neighborhood(rec, 0, k_bar)
        assert sub.component_truncated == (k_bar > 6)
        assert len(sub.cameras) == 6 and len(sub.points) == 15
        assert sub.scene.num_observations() == rec.num_observations()
        assert np.array_equal(sub.scene.obs_cam, rec.obs_cam) and np.array_equal(sub.scene.obs_u, rec.obs_u)


def test_bad_window_arguments_are_rejected():  # test_subrec.cpp:114-123 (planner part)
    rec = S.generate_cube_scene(4, 0.5)
    for center, k in ((0, 1), (6, 5), (-1, 5)):
        with pytest.raises(F.Error):
            R.extract_neighborhood(rec, center, k)


def test_neighborhoods_grow_connected_sets():  # test_subrec.cpp:125-139
    rec = S.generate_random_scene(40, 200, 0.2, 7, 0.5)
    g = R.build_view_graph(rec)
    for center in (0, 13, 20, 39):
        sub = R.extract_neighborhood(rec, center, 5)
        assert not sub.component_truncated and len(sub.cameras) == 5
        assert center in sub.cameras and np.all(np.diff(sub.cameras) > 0)
        assert connected(g, sub.cameras)
        assert sub.scene.num_cameras() == 5
        assert np.all(np.bincount(sub.scene.obs_cam, minlength=5) >= 4)  # the induced filter's fixpoint
        assert np.all(np.bincount(sub.scene.obs_pt) >= 2)


def test_growing_the_window_keeps_earlier_cameras():  # test_subrec.cpp:141-155 (nesting part)
    rec = S.generate_random_scene(40, 200, 0.2, 7, 0.5)
    small = R.extract_neighborhood(rec, 20, 8)
    large = R.extract_neighborhood(rec, 20, 20)
    assert np.all(np.isin(small.cameras, large.cameras))


def test_coverage_covers_every_camera_deterministically():  # plan_coverage, src/subrec.cpp:154-181
    rec = S.generate_random_scene(40, 200, 0.2, 7, 0.5)
    a = R.plan_coverage(rec, 10, 9)
    b = R.plan_coverage(rec, 10, 9)
    assert len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b))
    assert set(np.concatenate(a).tolist()) == set(range(40))
    assert any(not np.array_equal(x, y) for x, y in zip(a, R.plan_coverage(rec, 10, 10)))


def reference_neighborhood(rec, graph, center, k_bar):
    """extract_neighborhood restated literally (src/subrec.cpp:118-152 and
    the induced filter's rounds of simultaneous removals, :24-86)."""
    n = rec.num_cameras()
    weight = np.zeros(n, np.int64)
    chosen, inside = [center], np.zeros(n, bool)
    inside[center] = True
    for nb, w in graph.edges[center]:
        weight[nb] += w
    while len(chosen) < k_bar:
        best, best_w = -1, 0
        for i in range(n):
            if not inside[i] and weight[i] > best_w:
                best, best_w = i, weight[i]
        if best < 0:
            break
        chosen.append(best)
        inside[best] = True
        for nb, w in graph.edges[best]:
            if not inside[nb]:
                weight[nb] += w
    cam_in = set(chosen)
    while True:
        m = np.isin(rec.obs_cam, sorted(cam_in))
        pc = np.bincount(rec.obs_pt[m], minlength=rec.num_points())
        drop = {c for c in cam_in if np.sum(pc[rec.obs_pt[rec.obs_cam == c]] >= 2) < 4}
        if not drop:
            return np.array(sorted(cam_in), np.int32)
        cam_in -= drop


def sparse_structure(seed, n=14, m=45):
    """A scene whose planner-relevant part (which camera sees which point) is
    random and sparse: 2-4 observers per point, so small subsets keep few
    points seen twice and the induced filter removes cameras, often in
    cascades.  The geometry is irrelevant to planning (no validation here)."""
    rng = np.random.default_rng(seed)
    oc, op = [], []
    for j in range(m):
        for c in sorted(rng.choice(n, size=int(rng.integers(2, 5)), replace=False)):
            oc.append(c)
            op.append(j)
    return F.Reconstruction(cams=np.zeros((n, 8)), pts=np.zeros((m, 3)), obs_cam=np.array(oc), obs_pt=np.array(op))


def cascade_structure():
    """Cameras H, A, B, C, D, E (0..5): A has 3 points seen twice, B, C, D 4
    each, chained by one point apiece (A-B, B-C, C-D), E shares 5 with H.
    The filter removes A, which costs B a point, which costs C one, ... down
    to {H, E}: each round of the reference removes exactly one camera."""
    H, A, B, C, D, E = range(6)
    obs = []
    j = 0
    def point(*cams):
        nonlocal j
        obs.extend((c, j) for c in cams)
        j += 1
    for cam, k in ((A, 2), (B, 2), (C, 2), (D, 3), (E, 5)):
        for _ in range(k):
            point(H, cam)
    point(A, B)
    point(B, C)
    point(C, D)
    oc, op = zip(*obs)
    return F.Reconstruction(cams=np.zeros((6, 8)), pts=np.zeros((j, 3)), obs_cam=np.array(oc), obs_pt=np.array(op))


def test_induced_filter_cascade():
    rec = cascade_structure()
    g = R.build_view_graph(rec)
    want = reference_neighborhood(rec, g, 0, 6)
    assert want.tolist() == [0, 5]
    assert R.extract_neighborhood(rec, 0, 6).cameras.tolist() == [0, 5]


def test_induced_filter_matches_the_reference_rounds():
    removed = cascades = 0
    for seed in range(12):
        rec = sparse_structure(seed)
        g = R.build_view_graph(rec)
        for k_bar in (3, 4, 5, 7, 10):
            for center in range(rec.num_cameras()):
                want = reference_neighborhood(rec, g, center, k_bar)
                try:
                    got = R.extract_neighborhood(rec, center, k_bar).cameras
                except F.Error:
                    got = np.zeros(0, np.int32)  # the filter emptied the subset
                assert np.array_equal(got, want), (seed, k_bar, center, got, want)
                removed += k_bar - len(want)
                cascades += len(want) == 0
    assert removed > 0 and cascades > 0  # the cases exercise removals, down to empty subsets


# ---- GPU --------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("scene,min_covis", [("config1", 1), ("config2", 1), ("config2", 5), ("random", 1),
                                             ("config3", 3)])
def test_device_view_graph_equals_the_host_graph(engine, scene, min_covis):
    rec = {"config1": lambda: S.generate_config(1), "config2": lambda: S.generate_config(2),
           "config3": lambda: S.generate_config(3),
           "random": lambda: S.generate_random_scene(40, 200, 0.2, 7, 0.5)}[scene]()
    host = R.build_view_graph(rec, min_covis)
    dev = R.build_view_graph(rec, min_covis, engine=engine)
    assert dev.n_cams == host.n_cams and dev.edges == host.edges


@pytest.mark.gpu
def test_bad_aggregation_arguments_are_rejected(engine):  # test_subrec.cpp:119-121
    rec = S.generate_cube_scene(4, 0.5)
    with pytest.raises(F.Error):
        R.approximate_covariances(rec, 1, 3, 0, engine=engine)
    with pytest.raises(F.Error):
        R.approximate_covariances(rec, 6, 0, 0, engine=engine)


@pytest.mark.gpu
def test_invalid_full_scene_fails_validation_before_planning(engine):  # src/subrec.cpp:191, 262
    # a duplicate (camera, point) pair: the reference's rec.validate() rejects
    # the whole scene before any subset is planned, with its own message
    rec = S.generate_random_scene(20, 150, 0.3, 5, 0.5)
    rec.obs_pt[1] = rec.obs_pt[0]
    rec.obs_cam[1] = rec.obs_cam[0]
    for call in (lambda: R.approximate_covariances(rec, 6, 1, 0, engine=engine),
                 lambda: R.error_size_sweep(rec, [6], 1, 0, engine=engine)):
        with pytest.raises(F.Error) as e:
            call()
        assert e.value.kind == F.ErrorKind.invariant and e.value.stage == "validate"
        assert "duplicate" in str(e.value)


@pytest.mark.gpu
def test_monotonicity_and_nesting(engine):  # test_subrec.cpp:141-169
    rec = S.generate_random_scene(40, 200, 0.2, 7, 0.5)
    small = R.extract_neighborhood(rec, 20, 8)
    large = R.extract_neighborhood(rec, 20, 20)
    rep = R.monotonicity_check(rec, small, large, engine=engine)
    assert rep.cameras_checked == len(small.cameras) and rep.violations == []
    assert R.monotonicity_check(rec, small, small, engine=engine).violations == []
    a = R.extract_neighborhood(rec, 0, 10)
    b = R.extract_neighborhood(rec, 20, 10)
    with pytest.raises(F.Error) as e:
        R.monotonicity_check(rec, a, b, engine=engine)
    assert e.value.kind == F.ErrorKind.invariant and "not nested" in str(e.value)


@pytest.mark.gpu
def test_full_size_aggregation_reproduces_the_full_covariance_exactly(engine):  # test_subrec.cpp:171-184
    rec = S.generate_cube_scene(5, 0.5)
    agg = R.approximate_covariances(rec, 6, 1, 3, engine=engine)
    full = engine.compute_covariance(rec)
    assert agg.target_size == 6 and agg.cov.shape[0] == 6
    for i in range(6):
        assert np.array_equal(agg.cov[i], full.camera_cov[i])
        assert agg.trace[i] == sum(full.camera_cov[i][p, p] for p in range(8))
        assert agg.subset_id[i] == 0


@pytest.mark.gpu
def test_extra_decompositions_only_lower_the_trace(engine):  # test_subrec.cpp:186-195
    rec = S.generate_random_scene(40, 200, 0.2, 7, 0.5)
    one = R.approximate_covariances(rec, 10, 1, 9, engine=engine)
    three = R.approximate_covariances(rec, 10, 3, 9, engine=engine)
    for i in range(40):
        assert three.trace[i] <= one.trace[i] and three.subset_id[i] >= 0
        assert three.trace[i] == sum(three.cov[i][p, p] for p in range(8))


@pytest.mark.gpu
def test_failures_name_the_subset_and_decomposition(engine):  # test_subrec.cpp:197-208
    rec = S.generate_cube_scene(6, 0.5)
    rec.pts[14] = rec.cams[3, 3:6]
    with pytest.raises(F.Error) as e:
        R.approximate_covariances(rec, 6, 1, 0, engine=engine)
    assert e.value.kind == F.ErrorKind.degenerate and e.value.stage == "subrec"
    assert "subset 0 (decomposition 0)" in str(e.value)


@pytest.mark.gpu
@pytest.mark.parametrize("workers", [1, 4])
def test_kept_blocks_match_the_restatement_per_subset(engine, workers):
    rec = S.generate_config(2)  # 100 cameras, windows of 20
    k_bar, decos, seed = 20, 2, 5
    agg = R.approximate_covariances(rec, k_bar, decos, seed, workers=workers, engine=engine)
    subsets = [c for d in range(decos) for c in R.plan_coverage(rec, k_bar, seed + d)]
    P = rec.cam_params
    cache = {}
    for g in range(rec.num_cameras()):
        sid = int(agg.subset_id[g])
        if sid not in cache:
            cams = subsets[sid]
            sub = R.induced_scene(rec, cams, points_of(rec, cams))
            cache[sid] = (cams, O.compute_covariance(sub)[0])
        cams, cov = cache[sid]
        l = int(np.searchsorted(cams, g))
        assert rel(agg.cov[g], cov[l]) <= 1e-9
    # batching (workers) does not change any result bit
    again = R.approximate_covariances(rec, k_bar, decos, seed, workers=1, engine=engine)
    assert np.array_equal(again.cov, agg.cov) and np.array_equal(again.subset_id, agg.subset_id)


@pytest.mark.gpu
def test_error_size_sweep_shrinks_with_larger_windows(engine):  # test_subrec.cpp:210-230
    rec = S.generate_random_scene(40, 200, 0.2, 7, 0.5)
    rows = R.error_size_sweep(rec, [5, 20], 6, 123, engine=engine)
    assert rows
    for r in rows:
        assert r.k_bar in (5, 20) and 0 <= r.subset_id < 6 and 0 <= r.camera_id < 40
        assert r.err_absolute >= 0 and r.err_relative >= 0 and r.trace > 0
    rel5 = [r.err_relative for r in rows if r.k_bar == 5]
    rel20 = [r.err_relative for r in rows if r.k_bar == 20]
    assert rel5 and rel20 and np.median(rel5) > np.median(rel20)


@pytest.mark.gpu
def test_sweep_rows_survive_a_csv_round_trip(engine, tmp_path):  # test_subrec.cpp:232-257
    rec = S.generate_cube_scene(7, 0.5)
    rows = R.error_size_sweep(rec, [4], 2, 11, engine=engine)
    p = tmp_path / "sweep.csv"
    R.write_sweep_csv(rows, str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "kbar,subset_id,camera_id,err_relative,err_absolute,trace"
    back = [l.split(",") for l in lines[1:] if l]
    assert len(back) == len(rows)
    for r, f in zip(rows, back):
        assert (int(f[0]), int(f[1]), int(f[2])) == (r.k_bar, r.subset_id, r.camera_id)
        assert (float(f[3]), float(f[4]), float(f[5])) == (r.err_relative, r.err_absolute, r.trace)


@pytest.mark.gpu
def test_batched_and_one_by_one_paths_agree(engine, tmp_path):
    """The batched sub-scene pipeline (one launch per stage over the
    concatenated sub-scenes, csrc/batch.cu) against the one-sub-scene-at-a-time
    path (SFMCOV_SUBREC_BATCH=0, in a subprocess): same winning subsets, blocks
    equal to FP64 rounding (the per-scene gauge sums run in another order)."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import sys, numpy as np; sys.path.insert(0, '.');"
            "from paper_1808_02414_b200 import sfmcov as F, synthetic as S, subrec as R;"
            "a = R.approximate_covariances(S.generate_config(2), 12, 2, 5, engine=F.Engine(0));"
            "np.savez(sys.argv[1], cov=a.cov, sid=a.subset_id)")
    out = str(tmp_path / "one.npz")
    subprocess.run([sys.executable, "-c", code, out], cwd=ROOT, env=dict(os.environ, SFMCOV_SUBREC_BATCH="0"),
                   check=True, timeout=600)
    one = np.load(out)
    batched = R.approximate_covariances(S.generate_config(2), 12, 2, 5, engine=engine)
    assert np.array_equal(batched.subset_id, one["sid"])
    worst = max(rel(a, b) for a, b in zip(batched.cov, one["cov"]))
    assert worst <= 1e-10


@pytest.mark.gpu
def test_concurrent_calls_on_one_handle(engine):
    """Two threads sharing one handle (the C++ header keeps one per device):
    each approximate_covariances call holds the handle for its whole pipeline
    (its chunks reuse the scene its validation uploaded), so the results equal
    the sequential ones bitwise."""
    import threading
    a, b = S.generate_config(2), S.generate_random_scene(40, 200, 0.2, 7, 0.5)
    want = [R.approximate_covariances(a, 12, 2, 5, engine=engine), R.approximate_covariances(b, 8, 2, 3, engine=engine)]
    got = [None, None]

    def run(i):
        got[i] = (R.approximate_covariances(a, 12, 2, 5, engine=engine) if i == 0 else
                  R.approximate_covariances(b, 8, 2, 3, engine=engine))

    for _ in range(3):
        th = [threading.Thread(target=run, args=(i,)) for i in (0, 1)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for w, g in zip(want, got):
            assert np.array_equal(w.subset_id, g.subset_id)
            assert np.array_equal(w.cov, g.cov)


@pytest.mark.gpu
def test_pipeline_chunking_does_not_change_results(engine, tmp_path):
    """The pipelined call packs sub-scenes into device chunks in arrival
    order; chunks of one sub-scene each (SFMCOV_SUBREC_MIN_CHUNK=1, in a
    subprocess) must give bitwise the same blocks and winning subsets."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import sys, numpy as np; sys.path.insert(0, '.');"
            "from paper_1808_02414_b200 import sfmcov as F, synthetic as S, subrec as R;"
            "a = R.approximate_covariances(S.generate_config(2), 12, 3, 9, engine=F.Engine(0));"
            "np.savez(sys.argv[1], cov=a.cov, sid=a.subset_id)")
    out = str(tmp_path / "tiny.npz")
    subprocess.run([sys.executable, "-c", code, out], cwd=ROOT, env=dict(os.environ, SFMCOV_SUBREC_MIN_CHUNK="1"),
                   check=True, timeout=600)
    tiny = np.load(out)
    ref = R.approximate_covariances(S.generate_config(2), 12, 3, 9, engine=engine)
    assert np.array_equal(ref.subset_id, tiny["sid"])
    assert np.array_equal(ref.cov, tiny["cov"])


def _emulated_subsets(seed, n=40, P=8, covers=3):
    """Random coverings (subset -> cameras, blocks) with deliberate trace ties."""
    rng = np.random.default_rng(seed)
    subs = []  # (decomposition, index within it, cams, blocks, traces)
    for d in range(covers):
        perm = rng.permutation(n)
        for i, cams in enumerate(np.array_split(perm, int(rng.integers(3, 7)))):
            cams = np.sort(np.concatenate([cams, rng.choice(n, 3)]))
            cams = np.unique(cams)
            blocks = rng.standard_normal((len(cams), P, P))
            tr = np.round(rng.uniform(1, 3, len(cams)), 1)  # coarse: many ties between subsets
            for b, t in zip(blocks, tr):
                b[np.diag_indices(P)] += (t - np.trace(b)) / P
            subs.append((d, i, cams, blocks, np.array([np.trace(b) for b in blocks])))
    return subs


def _emulated_aggregate(subs, n, P, owned=None):
    """csrc/subrec.cpp approximate_impl's aggregation over the given subsets
    (all, or one rank's), the partial form of a sharded call."""
    cov, tr, sid = np.zeros((n, P, P)), np.full(n, np.inf), -np.ones(n, np.int32)
    for s, (_, _, cams, blocks, trs) in enumerate(subs):
        if owned is not None and not owned[s]:
            continue
        for c, b, t in zip(cams, blocks, trs):
            if sid[c] < 0 or t < tr[c]:
                cov[c], tr[c], sid[c] = b, t, s
    return R.ShardResult(cov, tr, sid)


@pytest.mark.parametrize("nranks", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_merged_shards_equal_the_single_aggregation(nranks, seed):
    n, P, covers = 40, 8, 3
    subs = _emulated_subsets(seed, n, P, covers)
    want = _emulated_aggregate(subs, n, P)
    parts = [_emulated_aggregate(subs, n, P, [R.shard_owner(i, d, covers, nranks) == r for d, i, *_ in subs])
             for r in range(nranks)]
    got = R.merge_shards(parts, 10)
    assert np.array_equal(got.subset_id, want.subset_id)
    assert np.array_equal(got.trace, want.trace) and np.array_equal(got.cov, want.cov)


def test_shard_owner_spreads_every_covering():
    # consecutive subsets of one covering land on different ranks, and the
    # coverings are offset so small coverings do not all start on rank 0
    assert [R.shard_owner(i, 0, 3, 4) for i in range(4)] == [0, 3, 2, 1]
    assert [R.shard_owner(0, d, 3, 4) for d in range(3)] == [0, 1, 2]


def test_merge_reports_the_first_failure_in_reference_order_and_uncovered_cameras():
    n, P = 6, 8
    ok = R.ShardResult(np.zeros((n, P, P)), np.ones(n), np.arange(n, dtype=np.int32))
    key = lambda d, phase, i: (d << 33) | (phase << 32) | i  # csrc/subrec.cpp FirstFailure
    comp = R.ShardResult(ok.cov, ok.trace, ok.subset_id, 4, key(0, 1, 3), "subrec", "subrec: subset 3 (decomposition 0): y")
    draw1 = R.ShardResult(ok.cov, ok.trace, ok.subset_id, 4, key(1, 0, 0), "subrec", "subrec: camera 2 cannot anchor")
    comp1 = R.ShardResult(ok.cov, ok.trace, ok.subset_id, 4, key(1, 1, 0), "subrec", "subrec: subset 9 (decomposition 1): x")
    draw0 = R.ShardResult(ok.cov, ok.trace, ok.subset_id, 4, key(0, 0, 7), "subrec", "subrec: camera 5 cannot anchor")
    # covering 0's subsets are computed before covering 1 is drawn ...
    with pytest.raises(F.Error) as e:
        R.merge_shards([ok, comp1, draw1, comp], 6)
    assert e.value.kind == F.ErrorKind.degenerate and "subset 3 (decomposition 0)" in str(e.value)
    # ... and all of covering 0 is drawn before its first subset is computed
    with pytest.raises(F.Error) as e:
        R.merge_shards([comp, draw0], 6)
    assert "camera 5 cannot anchor" in str(e.value)
    early = R.ShardResult(ok.cov, ok.trace, ok.subset_id, 3, -1, "validate", "validate: bad scene")
    with pytest.raises(F.Error) as e:
        R.merge_shards([early, early], 6)
    assert e.value.stage == "validate"
    hole = R.ShardResult(ok.cov, np.where(np.arange(n) == 4, np.inf, 1.0), np.where(np.arange(n) == 4, -1, 0))
    with pytest.raises(F.Error) as e:
        R.merge_shards([hole, hole], 6)
    assert e.value.kind == F.ErrorKind.invariant and "camera 4 was not covered" in str(e.value)


def _gloo_merge_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        subs = _emulated_subsets(11)
        part = _emulated_aggregate(subs, 40, 8, [R.shard_owner(i, d, 3, world) == rank for d, i, *_ in subs])
        got = R.gather_and_merge(part, 10)
        q.put((rank, got.cov, got.trace, got.subset_id))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world2_gloo_shard_gather_and_merge():
    """The torch.distributed gather + merge of sharded sub-reconstructions
    on a world_size-2 gloo group: every rank gets the single-call result."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_merge_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    want = _emulated_aggregate(_emulated_subsets(11), 40, 8)
    for _, cov, tr, sid in res:
        assert np.array_equal(sid, want.subset_id) and np.array_equal(cov, want.cov) and np.array_equal(tr, want.trace)


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_calls_merge_to_the_single_call(engine, nranks):
    """Each rank's share run in turn on one engine (the per-rank work is
    independent), merged: bitwise the single call's blocks and subsets."""
    rec = S.generate_config(2)
    want = R.approximate_covariances(rec, 12, 3, 9, engine=engine)
    parts = [R.approximate_covariances_shard(rec, 12, 3, 9, nranks, r, engine=engine) for r in range(nranks)]
    assert all(p.code == 0 for p in parts)
    assert sum(int((p.subset_id >= 0).sum()) for p in parts) >= rec.num_cameras()
    got = R.merge_shards(parts, 12)
    assert np.array_equal(got.subset_id, want.subset_id)
    assert np.array_equal(got.cov, want.cov) and np.array_equal(got.trace, want.trace)


def _broken_cube():
    rec = S.generate_cube_scene(6, 0.5)
    rec.pts[14] = rec.cams[3, 3:6]  # a point at a camera centre: that sub-scene is degenerate
    return rec


@pytest.mark.gpu
@pytest.mark.parametrize("make,k_bar,decos,nranks", [
    (_broken_cube, 6, 2, 2), (_broken_cube, 6, 3, 3), (_broken_cube, 3, 3, 2),
    (lambda: S.generate_cube_scene(6, 0.5), 2, 3, 2), (lambda: S.generate_config(2), 2, 2, 4)])
def test_sharded_failure_is_the_single_calls_failure(engine, make, k_bar, decos, nranks):
    rec = make()
    try:
        R.approximate_covariances(rec, k_bar, decos, 0, engine=engine)
        single = None
    except F.Error as e:
        single = e
    parts = [R.approximate_covariances_shard(rec, k_bar, decos, 0, nranks, r, engine=engine) for r in range(nranks)]
    if single is None:
        assert all(p.code == 0 for p in parts)
        return
    with pytest.raises(F.Error) as merged:
        R.merge_shards(parts, k_bar)
    assert str(merged.value) == str(single) and merged.value.kind == single.kind
