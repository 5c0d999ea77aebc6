"""GPU parity of the point-sharded product through the C ABI.

The split entry points (akm_get_bounds / akm_set_bounds / akm_set_radius, akm_spread_grid,
akm_mvm_from_grid) let G shards of the rows each spread onto the same grids; summing the grids and
finishing on every shard must reproduce the single-plan product.  Two checks (and the window-sharded
plan at world 2 and 3, §8(e) item 3, at the end):
  * one process, two plans on cuda:0, grids summed by a device add (the library calls alone);
  * the ShardedPlan driver at world_size 2 over gloo, both ranks on cuda:0 (host-mediated all-reduce,
    no rank's kernels wait on another's: the NCCL/NVLink path differs only in the transport).
"""
import os
import socket

import numpy as np
import pytest

import workloads
from oracle import dense_apply
from oracle import fourier as F

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def akm():
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_2504_00480_b200 as mod
    return mod


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def _single(akm, X, wl, V, ops):
    dev = torch.device("cuda:0")
    plan = akm.Plan(0)
    plan.set_points(torch.from_numpy(X).to(dev), wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
    plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    Vd = torch.from_numpy(V).to(dev)
    outs = {op: torch.empty_like(Vd) for op in ops}
    plan.mvm_multi(Vd, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))
    torch.cuda.synchronize()
    info = plan.info()
    plan.close()
    return {k: v.cpu().numpy() for k, v in outs.items()}, info


@pytest.mark.parametrize("name,n,r,shards", [("c2", 6000, 2, 2), ("c4", 20000, 11, 3), ("c3", 8000, 3, 2),
                                              ("c1", 2000, 1, 4)])
def test_two_plans_sum_grids(akm, name, n, r, shards):
    wl = workloads.CONFIGS[name]
    X = workloads.make_X(wl, n=n)
    V = workloads.make_V(wl, n=n, r=r)
    ops = ("K", "dell", "dsf")
    dev = torch.device("cuda:0")
    plans, parts = [], []
    for k in range(shards):
        a = k * n // shards
        b = (k + 1) * n // shards
        p = akm.Plan(0)
        p.set_points(torch.from_numpy(np.ascontiguousarray(X[a:b])).to(dev), wl.windows, wl.family, wl.N,
                     wl.sigma_over, wl.m, wl.eps_B)
        plans.append(p)
        parts.append((a, b))
    bounds = [p.bounds() for p in plans]
    lo = np.min([b[0] for b in bounds], axis=0)
    hi = np.max([b[1] for b in bounds], axis=0)
    rad = np.max([p.set_bounds(lo, hi) for p in plans], axis=0)
    for p in plans:
        p.set_radius(rad)
        p.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    bins = [p.info()["bin"] for p in plans]
    if any(b != bins[0] for b in bins):
        for p in plans:
            p.set_bin_override(bins[0])
            p.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    size = plans[0].grid_size(r)
    assert all(p.grid_size(r) == size for p in plans)
    total = torch.zeros(size, dtype=torch.float64, device=dev)
    Vs = [torch.from_numpy(np.ascontiguousarray(V[a:b])).to(dev) for a, b in parts]
    for p, Vl in zip(plans, Vs):
        g = torch.empty(size, dtype=torch.float64, device=dev)
        p.spread_grid(Vl, g)
        total += g
    got = {op: np.zeros((n, r)) for op in ops}
    for p, Vl, (a, b) in zip(plans, Vs, parts):
        o = {op: torch.empty_like(Vl) for op in ops}
        p.mvm_from_grid(total, Vl, Y=o["K"], dY_ell=o["dell"], dY_sf=o["dsf"])
        torch.cuda.synchronize()
        for op in ops:
            got[op][a:b] = o[op].cpu().numpy()
    single, info = _single(akm, X, wl, V, ops)
    for p in plans:
        assert p.info()["c_w"] == pytest.approx(info["c_w"], rel=1e-15)
        p.close()
    for op in ops:
        assert rel(got[op], single[op]) <= 1e-12, (op, rel(got[op], single[op]))
    nd = F.additive_fastsum(X, wl.windows, wl.family, (wl.sigma_f, wl.ell, wl.sigma_eps), V, wl.N, wl.eps_B,
                            ops=ops, m=wl.m)
    tol = 1e-9 if wl.m == 6 else 1e-11
    for op in ops:
        assert rel(got[op], nd[op]) <= tol, (op, rel(got[op], nd[op]))


def test_shard_calls_validate(akm):
    wl = workloads.CONFIGS["c2"]
    X = workloads.make_X(wl, n=500)
    p = akm.Plan(0)
    p.set_points(X, wl.windows, wl.family)
    lo, hi = p.bounds()
    with pytest.raises(akm.AkmError):            # bounds must contain the plan's points
        p.set_bounds(lo + 0.01, hi)
    rad = p.set_bounds(lo - 0.1, hi + 0.1)
    with pytest.raises(akm.AkmError):            # radius below the plan's own
        p.set_radius(rad * 0.5)
    with pytest.raises(akm.AkmError):            # grid calls need theta
        p.grid_size(1)
    p.set_radius(rad * 1.5)
    p.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    assert p.info()["radius"] == pytest.approx(list(rad * 1.5))
    with pytest.raises(akm.AkmError):
        p.set_bin_override([5, 1, 1])
    p.set_bin_override([2, 2, 2])
    p.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    assert p.info()["bin"] == [2, 2, 2]
    p.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_00480_b200 import dist as D
        wl = workloads.CONFIGS["c2"]
        n, r = 5000, 2
        X = workloads.make_X(wl, n=n)
        V = workloads.make_V(wl, n=n, r=r)
        a, b = D.row_partition(n, world, rank)
        dev = torch.device("cuda:0")
        sp = D.ShardedPlan(torch.from_numpy(np.ascontiguousarray(X[a:b])).to(dev), wl.windows, wl.family, wl.N,
                           wl.sigma_over, wl.m, wl.eps_B, device=dev, comm_device=torch.device("cpu"))
        sp.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
        Vl = torch.from_numpy(np.ascontiguousarray(V[a:b])).to(dev)
        Y, dY = torch.empty_like(Vl), torch.empty_like(Vl)
        sp.mvm_multi(Vl, Y=Y, dY_ell=dY)
        torch.cuda.synchronize()
        q.put((rank, a, b, Y.cpu().numpy(), dY.cpu().numpy()))
        sp.close()
    finally:
        dist.destroy_process_group()


def test_sharded_plan_gloo_world2(akm):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = workloads.CONFIGS["c2"]
    n, r = 5000, 2
    X = workloads.make_X(wl, n=n)
    V = workloads.make_V(wl, n=n, r=r)
    Y, dY = np.zeros((n, r)), np.zeros((n, r))
    for _, a, b, y, dy in res:
        Y[a:b], dY[a:b] = y, dy
    single, _ = _single(akm, X, wl, V, ("K", "dell"))
    assert rel(Y, single["K"]) <= 1e-12 and rel(dY, single["dell"]) <= 1e-12
    de = dense_apply(X, wl.windows, wl.family, (wl.sigma_f, wl.ell, wl.sigma_eps), V, ops=("K", "dell"))
    assert rel(Y, de["K"]) <= 1e-6 and rel(dY, de["dell"]) <= 1e-6


def _obj_gloo_worker(rank, world, port, q, kpw):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2504_00480_b200 as akm
        from paper_2504_00480_b200 import dist as D
        wl = workloads.CONFIGS["c5"]
        n = 20000
        X = workloads.make_X(wl, n=n)
        V = workloads.make_V(wl, n=n)
        dev = torch.device("cuda:0")
        plan = akm.Plan(0)
        plan.set_points(torch.from_numpy(X).to(dev), wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
        if kpw:
            plan.set_preconditioner(kpw)
        plan.set_theta(0.5, 0.5, 1.0)   # CG converges in 50 iterations here (tests/test_gpu_objective.py)
        y = torch.from_numpy(np.ascontiguousarray(V[:, 0])).to(dev)
        Z = torch.from_numpy(np.ascontiguousarray(V[:, 1:])).to(dev)
        res = D.sharded_objective(plan, y, Z, 50, 30, comm_device=torch.device("cpu"), preconditioned=bool(kpw))
        single = (plan.objective if kpw else plan.objective_diag)(y, Z, 50, 30)
        plan.close()
        q.put((rank, res["Z"], res["quad"], res["slq"], single["Z"], single["quad"], single["slq"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kpw", [0, 60])
def test_probe_sharded_objective_gloo_world2(akm, kpw):
    """each rank runs a slice of the probes (rank 0 also CG) through the library;
    the combined Z~ equals the single-process Z~ (theta where 50 CG iterations converge: the two runs
    multiply differently sized blocks, so their products differ by rounding only)."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_obj_gloo_worker, args=(k, world, port, q, kpw)) for k in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, Zs, quad, slq, Z1, quad1, slq1 in res:
        assert Zs == pytest.approx(Z1, rel=1e-9)
        assert quad == pytest.approx(quad1, rel=1e-8)
        assert slq == pytest.approx(slq1, rel=1e-8)


def _grad_gloo_worker(rank, world, port, q, kpw):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2504_00480_b200 as akm
        from paper_2504_00480_b200 import dist as D
        wl = workloads.CONFIGS["c5"]
        n = 8000
        X = workloads.make_X(wl, n=n)
        V = workloads.make_V(wl, n=n)
        dev = torch.device("cuda:0")
        plan = akm.Plan(0)
        plan.set_points(torch.from_numpy(X).to(dev), wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
        if kpw:
            plan.set_preconditioner(kpw)
        th = (0.5, 0.5, 2.0)           # 50 CG iterations converge to rounding here (asserted below)
        plan.set_theta(*th)
        y = torch.from_numpy(np.ascontiguousarray(V[:, 0])).to(dev)
        Z = torch.from_numpy(np.ascontiguousarray(V[:, 1:])).to(dev)
        g = D.sharded_gradient(plan, y, Z, th, len(wl.windows), 50, comm_device=torch.device("cpu"),
                               preconditioned=bool(kpw))
        one = (plan.gradient if kpw else plan.gradient_diag)(y, Z, 50)
        single, last = one["grad"], one["cg_hist"][-1]
        plan.close()
        q.put((rank, g, single, last))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kpw", [0, 60])
def test_probe_sharded_gradient_gloo_world2(akm, kpw):
    """SURVEY.md §8(e) item 2 for the gradient: per-column raw terms (akm_gradient_columns) summed over
    the ranks reproduce the single-process gradient (diagonal M and AAFN)."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_gloo_worker, args=(k, world, port, q, kpw)) for k in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, g, single, last in res:
        assert last < 1e-11, last      # converged: the products' rounding does not move the solves
        for j in ("sf", "ell", "se"):
            assert g[j] == pytest.approx(single[j], rel=1e-9, abs=1e-9 * abs(single["se"])), j


# ---------------------------------------------------------------- window sharding (§8(e) item 3)
def _win_gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_00480_b200 import dist as D
        wl = workloads.CONFIGS["c4"]
        n, r = 20000, 3
        X = workloads.make_X(wl, n=n)
        V = workloads.make_V(wl, n=n, r=r)
        dev = torch.device("cuda:0")
        sp = D.WindowShardedPlan(torch.from_numpy(X).to(dev), wl.windows, wl.family, wl.N, wl.sigma_over, wl.m,
                                 wl.eps_B, device=dev, comm_device=torch.device("cpu"))
        sp.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
        Vd = torch.from_numpy(V).to(dev)
        Y, dY, dS = torch.empty_like(Vd), torch.empty_like(Vd), torch.empty_like(Vd)
        sp.mvm_multi(Vd, Y=Y, dY_ell=dY, dY_sf=dS)
        torch.cuda.synchronize()
        q.put((rank, (sp.w0, sp.w1), Y.cpu().numpy(), dY.cpu().numpy(), dS.cpu().numpy()))
        sp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_window_sharded_plan_gloo(akm, world):
    """c4's four windows over 2 ranks (2 + 2) and 3 ranks (2 + 1 + 1), both on cuda:0: every rank's
    all-reduced products equal the single plan's to rounding (the per-window frames are independent,
    reading R2; sigma_eps^2 V is added once)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_win_gloo_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = workloads.CONFIGS["c4"]
    X = workloads.make_X(wl, n=20000)
    V = workloads.make_V(wl, n=20000, r=3)
    single, _ = _single(akm, X, wl, V, ("K", "dell", "dsf"))
    assert [b for _, b, *_ in res][-1][1] == len(wl.windows)
    for _, _, Y, dY, dS in res:
        assert rel(Y, single["K"]) <= 1e-12 and rel(dY, single["dell"]) <= 1e-12 and rel(dS, single["dsf"]) <= 1e-12
