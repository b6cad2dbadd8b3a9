"""Host-side plumbing of the multi-GPU path (one process per GPU).

The compute and the collectives of the distributed pipeline live in the CUDA
library (csrc/dist.cu: NCCL broadcast of each factored panel, all-reduce of
the camera-pair blocks and of the outputs).  This module holds what the
launcher does around it: hand every rank the NCCL unique id, attach the
engine, and the max-over-ranks timing reduction.  It runs with any
torch.distributed backend (gloo on CPU for the tests, nccl on the GPU box).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import sfmcov as F


def exchange_unique_id(rank: int, device=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL id; every rank returns the same bytes."""
    buf = torch.zeros(128, dtype=torch.uint8, device=device or "cpu")
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(F.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def attach(engine: "F.Engine", rank: int, world: int, device=None) -> None:
    """Attach `engine` to rank `rank` of `world` (no communicator for world == 1)."""
    uid = exchange_unique_id(rank, device) if world > 1 else bytes(128)
    engine.comm_init(uid, world, rank)


def max_over_ranks(value: float, world: int, device=None) -> float:
    if world == 1:
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def check_partition(n_cams: int, cam_params: int, world: int, panel_blocks: int = 3):
    """Every camera block extracted by exactly one rank and the local columns
    summing to the padded dimension (the 1D block-cyclic plan of dist.cu)."""
    owned = np.zeros(n_cams, dtype=np.int64)
    cols = 0
    npad = None
    for r in range(world):
        npad, c, o = F.plan_dense(n_cams, cam_params, world, r, panel_blocks)
        owned += o
        cols += c
    return bool(np.all(owned == 1)) and cols == npad
