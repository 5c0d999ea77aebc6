"""Multi-GPU host logic: the product is linear and column-independent in V, so N GPUs
run N independent RHS blocks of the same workload (weak scaling) with no data-path collective.

This module holds only the host-side bookkeeping of that scheme -- per-rank seeds, column
partitions, the max-over-ranks timing reduction and the whole-job throughput -- so it can be
tested on CPU with the ``gloo`` backend (tests/test_dist_cpu.py) and used unchanged by bench.py
under torchrun with ``nccl``.  No kernel arithmetic lives here.
"""
from __future__ import annotations

import os

RANK_SEED_STRIDE = 7919


def env_rank():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_seed(base_seed: int, rank: int) -> int:
    """Seed of rank ``rank``'s independent RHS block (rank 0 keeps the workload's own seed)."""
    return int(base_seed) + RANK_SEED_STRIDE * int(rank)


def column_partition(r_total: int, world: int, rank: int):
    """Contiguous [start, stop) of ``r_total`` columns owned by ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(int(r_total), int(world))
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the default process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_throughput(units_per_rank: float, world: int, max_ms_per_step: float) -> float:
    """Whole-job units/s: every rank processed ``units_per_rank`` in at most ``max_ms_per_step``."""
    return float(units_per_rank) * int(world) / (float(max_ms_per_step) * 1e-3)
