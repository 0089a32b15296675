"""Multi-process plumbing (one process per GPU, torch.distributed) for the sharded path.

Partition: Gaussians and all their optimizer state by contiguous id range, so
cull and both Adam passes are shard-local (no communication), and concatenating the per-shard
ascending id lists in shard order reproduces the global cull list bit-exactly. The image-parallel
exchange of splat records / screen-space gradients (two all-to-allv per view) lives in imgpar.py;
bench.py's N>1 default runs it (`--mode imgpar`), `--mode replicas` runs N independent engines
(weak-scaling replicas, no collective). Only the gloo path and N=1 NCCL have run so far; no
multi-GPU NCCL measurement exists.
"""
from __future__ import annotations

import os
from typing import List, Sequence, Tuple

import numpy as np


def world() -> Tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (single process: 0, 0, 1)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def id_range(n: int, rank: int, world_size: int) -> Tuple[int, int]:
    """Contiguous id range [lo, hi) of shard `rank`: sizes differ by at most one."""
    base, extra = divmod(n, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_seed(seed: int, rank: int) -> int:
    """Scene seed of a weak-scaling shard (independent object per rank)."""
    return seed + rank


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing (the contract's max-over-ranks) via all_reduce(MAX)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_ids(local_ids: np.ndarray, lo: int) -> np.ndarray:
    """Global ascending id list from per-shard local lists (local id + shard offset, shard order).
    Equal to the cull of the unsharded arena because the cull is per-row and ids ascend within
    and across shards."""
    import torch.distributed as dist

    glob = np.asarray(local_ids, np.int64) + lo
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return glob.astype(np.int32)
    parts: List[np.ndarray] = [None] * dist.get_world_size()  # type: ignore[list-item]
    dist.all_gather_object(parts, glob)
    return np.concatenate(parts).astype(np.int32)


def aggregate_throughput(units_per_rank: Sequence[float], ms_max: float) -> float:
    """Whole-job throughput: units all ranks processed / the max-over-ranks time."""
    return float(sum(units_per_rank)) / (ms_max / 1e3)
