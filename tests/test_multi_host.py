"""Host logic of the multi-GPU path on CPU: the partition plans of the
distributed pipeline (csrc/dist.cu) and the launcher plumbing of
paper_1808_02414_b200/multi.py across a world_size-2 gloo group.  No GPU
compute calls."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_02414_b200 import multi as M
from paper_1808_02414_b200 import sfmcov as F


@pytest.mark.parametrize("P", [8, 9])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 13, 100, 1000, 3000])
def test_dense_plan_partitions_columns_and_cameras(n, world, P):
    assert M.check_partition(n, P, world)
    npad, _, _ = F.plan_dense(n, P, world, 0)
    cpb = 128 // P
    assert npad == -(-n // cpb) * 128  # camera-aligned layout: no camera straddles a 128-block


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("nchunks", [0, 1, 7, 1000, 56253])
def test_chunk_plan_partitions_pairs(nchunks, world):
    ranges = [F.plan_chunks(nchunks, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == nchunks
    for (b0, e0), (b1, _) in zip(ranges, ranges[1:]):
        assert e0 == b1 and b0 <= e0
    sizes = [e - b for b, e in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_plan_rejects_bad_arguments():
    with pytest.raises(F.Error):
        F.plan_dense(10, 7, 2, 0)
    with pytest.raises(F.Error):
        F.plan_chunks(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = M.exchange_unique_id(rank)
        _, cols, owned = F.plan_dense(1000, 9, world, rank)
        b, e = F.plan_chunks(56253, world, rank)
        t = M.max_over_ranks(float(rank + 1), world)
        q.put((rank, uid, cols, owned.tolist(), (b, e), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world2_gloo_launcher_logic():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    uids = {r[1] for r in res}
    assert len(uids) == 1 and len(next(iter(uids))) == 128 and any(next(iter(uids)))  # same, non-empty id
    owned = np.array([r[3] for r in res])
    assert np.all(owned.sum(0) == 1)                      # every camera block on exactly one rank
    npad, _, _ = F.plan_dense(1000, 9, world, 0)
    assert sum(r[2] for r in res) == npad                 # local columns tile the matrix
    assert res[0][4][0] == 0 and res[0][4][1] == res[1][4][0] and res[1][4][1] == 56253
    assert all(r[5] == 2.0 for r in res)                  # max over ranks
