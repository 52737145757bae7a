"""Multi-GPU plumbing for libnj (one process per GPU, torch.distributed).

Host-side only: rank / world discovery, the row-balanced request split of the
request-sharded mode (no communication on the data path), the
vocab shard of the vocab-sharded mode (§8e.2, nj_shard_range) and the NCCL
bootstrap of libnj's own communicator (rank 0's nj_nccl_get_unique_id bytes
broadcast over the torch process group).  No verification arithmetic here.
"""
from __future__ import annotations

import os

import numpy as np


def env_world():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def split_requests(gamma, world: int, rank: int):
    """Contiguous request range [b0, b1) of `rank`, balanced by rows
    (N_g ~ N / G).  Every request lands on exactly one rank."""
    g = np.asarray(gamma, np.int64)
    rows = np.concatenate([[0], np.cumsum(g + 1)])
    N = int(rows[-1])
    cuts = [int(np.searchsorted(rows, N * r / world, side="left")) for r in range(world + 1)]
    cuts[0], cuts[-1] = 0, len(g)
    for r in range(1, world + 1):   # monotone
        cuts[r] = max(cuts[r], cuts[r - 1])
    return cuts[rank], cuts[rank + 1]


def vocab_shard(V: int, world: int, rank: int):
    """[v_begin, v_end) of `rank` in the vocab-sharded mode (nj_shard_range)."""
    from ._lib import shard_range
    return shard_range(V, world, rank)


def broadcast_bytes(data: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string from `src` (torch.distributed, any backend)."""
    import torch.distributed as dist
    box = [data]
    dist.broadcast_object_list(box, src=src, group=group)
    return box[0]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float (timing: max over ranks, never wall clock)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def nccl_comm_for_world(device: int):
    """libnj's own NCCL communicator over the current torch process group
    (rank 0's unique id broadcast through torch.distributed)."""
    import torch.distributed as dist

    from ._lib import NcclComm, nccl_unique_id
    ws, rank = dist.get_world_size(), dist.get_rank()
    uid = broadcast_bytes(nccl_unique_id() if rank == 0 else None)
    return NcclComm(ws, uid, rank, device)
