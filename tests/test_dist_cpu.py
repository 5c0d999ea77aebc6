"""world_size-2 ``gloo`` tests of the N > 1 host logic on CPU: per-rank seeds give
independent RHS blocks, column partitions tile the block, the timing reduction is the max over
ranks, and the whole-job throughput counts every rank's units."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads
from paper_2504_00480_b200 import dist as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, lr = D.env_rank()
        wl = workloads.CONFIGS["c3"]
        V = workloads.make_V(wl, n=64, seed=D.rank_seed(2000 + wl.index, r))
        # every rank's block must differ (independent problems)
        blocks = [torch.zeros(64, wl.r, dtype=torch.float64) for _ in range(w)]
        dist.all_gather(blocks, torch.from_numpy(V))
        distinct = all(not torch.equal(blocks[a], blocks[b]) for a in range(w) for b in range(a + 1, w))
        local_ms = 1.0 + 2.5 * r                    # rank 1 is the slow one
        mx = D.max_over_ranks(local_ms)
        parts = [D.column_partition(11, w, k) for k in range(w)]
        q.put((r, w, lr, distinct, mx, parts, D.weak_throughput(wl.units, w, mx)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    wl = workloads.CONFIGS["c3"]
    for k, (r, w, lr, distinct, mx, parts, thr) in enumerate(res):
        assert (r, w, lr) == (k, world, k)
        assert distinct
        assert mx == 1.0 + 2.5 * (world - 1)        # max over ranks, identical on every rank
        assert parts == [(0, 6), (6, 11)]
        assert thr == pytest.approx(wl.units * world / (mx * 1e-3))


def test_partition_and_seed_properties():
    for r_total in (1, 2, 11, 37):
        for world in (1, 2, 3, 8):
            parts = [D.column_partition(r_total, world, k) for k in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == r_total
            assert all(parts[k][1] == parts[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    assert D.rank_seed(2002, 0) == 2002 and len({D.rank_seed(2002, k) for k in range(64)}) == 64
    assert D.max_over_ranks(3.5) == 3.5            # no process group: identity
    with pytest.raises(ValueError):
        D.column_partition(4, 2, 2)
