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


# ---------------------------------------------------------------- point-sharded product (§8(e) item 1)
class OracleShardBackend:
    """Test stand-in for the library behind ShardedPlan, built from the oracle's primitives: the
    'grid' of a shard is its inner sums a_k of eq. (3.3) per window (exact NDFT, real/imag pairs), so
    the sum over shards is the union's a_k exactly and the driver's frame agreement and all-reduce
    composition can be checked on CPU against the single-process oracle."""

    def __init__(self):
        from oracle import fourier as F
        self.F = F

    def set_points(self, X, windows, family, N, sigma_over, m, eps_B):
        self.X, self.windows, self.family, self.N, self.eps_B = np.asarray(X), windows, family, N, eps_B
        self.P = len(windows)
        self.lo = np.zeros((self.P, 3))
        self.hi = np.zeros((self.P, 3))
        for w, win in enumerate(windows):
            d = len(win)
            self.lo[w, 3 - d:] = self.X[:, list(win)].min(axis=0)
            self.hi[w, 3 - d:] = self.X[:, list(win)].max(axis=0)

    def bounds(self):
        return self.lo.copy(), self.hi.copy()

    def set_bounds(self, lo, hi):
        self.lo, self.hi = np.asarray(lo).reshape(self.P, 3), np.asarray(hi).reshape(self.P, 3)
        self.center = [0.5 * (self.lo[w, 3 - len(win):] + self.hi[w, 3 - len(win):]) for w, win in enumerate(self.windows)]
        self.R = np.array([np.sqrt(((self.X[:, list(win)] - self.center[w]) ** 2).sum(1)).max()
                           for w, win in enumerate(self.windows)])
        return self.R.copy()

    def set_radius(self, R):
        self.R = np.asarray(R, dtype=np.float64)

    def set_theta(self, sf, ell, se):
        F = self.F
        self.theta = (sf, ell, se)
        rho = 0.25 - self.eps_B / 2.0
        self.c, self.b = [], []
        for w, win in enumerate(self.windows):
            c = self.R[w] / rho if self.R[w] > 0 else 1.0
            if self.family == F.GAUSSIAN:
                c = max(c, ell * np.sqrt(2.0 * np.pi * self.N))
            self.c.append(c)
            d = len(win)
            self.b.append([F.fourier_coefficients(F.kernel_samples(self.family, ell / c, self.N, d, der))
                           for der in (False, True)])

    def info(self):
        return {"bin": [1] * self.P}

    def set_bin_override(self, bins):
        pass

    def _xs(self, w):
        return (self.X[:, list(self.windows[w])] - self.center[w]) / self.c[w]

    def grid_size(self, r):
        return sum(2 * self.N ** len(win) * r for win in self.windows)

    def spread_grid(self, V, grid):
        parts = []
        for w in range(self.P):
            a = self.F.ndft_adjoint(self._xs(w), V.numpy(), self.N)
            parts += [a.real.ravel(), a.imag.ravel()]
        grid.copy_(torch.from_numpy(np.concatenate(parts)))

    def mvm_from_grid(self, grid, V, Y, dY_ell, dY_sf):
        g = grid.numpy()
        Vn = V.numpy()
        r = Vn.shape[1]
        S, SD = np.zeros_like(Vn), np.zeros_like(Vn)
        off = 0
        for w, win in enumerate(self.windows):
            shape = (r,) + (self.N,) * len(win)
            size = int(np.prod(shape))
            a = g[off:off + size].reshape(shape) + 1j * g[off + size:off + 2 * size].reshape(shape)
            off += 2 * size
            xs = self._xs(w)
            S += np.real(self.F.ndft_forward(xs, self.b[w][0][None] * a))
            SD += np.real(self.F.ndft_forward(xs, self.b[w][1][None] * a)) / self.c[w]
        sf, ell, se = self.theta
        if Y is not None:
            Y.copy_(torch.from_numpy(sf * sf * S + se * se * Vn))
        if dY_ell is not None:
            dY_ell.copy_(torch.from_numpy(sf * sf * SD))
        if dY_sf is not None:
            dY_sf.copy_(torch.from_numpy(2.0 * sf * S))


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for name, n, r in (("c2", 900, 2), ("c3", 700, 3)):
            wl = workloads.CONFIGS[name]
            X = workloads.make_X(wl, n=n)
            V = workloads.make_V(wl, n=n, r=r)
            a, b = D.row_partition(n, world, rank)
            sp = D.ShardedPlan(X[a:b], wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B,
                               backend=OracleShardBackend())
            sp.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
            Vl = torch.from_numpy(np.ascontiguousarray(V[a:b]))
            Y, dY = torch.empty_like(Vl), torch.empty_like(Vl)
            sp.mvm_multi(Vl, Y=Y, dY_ell=dY)
            out[name] = (a, b, Y.numpy(), dY.numpy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_point_sharded_product():
    """world_size 2: each rank holds half the rows; the frame agreement (bounds MIN/MAX, radius MAX),
    one grid all-reduce and the per-rank finish reproduce the single-process truncated-Fourier product
    (eq. 3.3 on the union, scaling reading R2) to rounding, and the dense float64 oracle to the method
    tolerance."""
    from oracle import dense_apply
    from oracle import fourier as F
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name, n, r in (("c2", 900, 2), ("c3", 700, 3)):
        wl = workloads.CONFIGS[name]
        X = workloads.make_X(wl, n=n)
        V = workloads.make_V(wl, n=n, r=r)
        Y = np.zeros((n, r))
        dY = np.zeros((n, r))
        for k in range(world):
            a, b, y, dy = res[k][name]
            assert (a, b) == D.row_partition(n, world, k)
            Y[a:b], dY[a:b] = y, dy
        th = (wl.sigma_f, wl.ell, wl.sigma_eps)
        nd = F.additive_fastsum(X, wl.windows, wl.family, th, V, wl.N, wl.eps_B, ops=("K", "dell"))
        assert np.linalg.norm(Y - nd["K"]) <= 1e-12 * np.linalg.norm(nd["K"])
        assert np.linalg.norm(dY - nd["dell"]) <= 1e-12 * np.linalg.norm(nd["dell"])
        de = dense_apply(X, wl.windows, wl.family, th, V, ops=("K",))
        tol = 1e-6 if wl.family == 0 else 1e-3
        assert np.linalg.norm(Y - de["K"]) <= tol * np.linalg.norm(de["K"])


def test_row_partition():
    for n in (2, 7, 1000):
        for world in (1, 2, 8):
            if n < world:
                with pytest.raises(ValueError):
                    D.row_partition(n, world, 0)
                continue
            parts = [D.row_partition(n, world, k) for k in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n and all(b > a for a, b in parts)
    assert D.strong_throughput(1e6, 2.0) == pytest.approx(5e8)


# ---------------------------------------------------------------- probe-sharded objective (§8(e) item 2)
class OracleObjectivePlan:
    """Test stand-in for Plan.objective_diag: the oracle's CG + Lanczos driver on the dense K^."""

    def __init__(self, X, windows, family, theta):
        from oracle import aafn as A
        self.K = A.khat_dense(X, windows, family, theta)
        sf, _, se = theta
        self.c = sf * sf * len(windows) + se * se

    def objective_diag(self, y, Z, cg_iters, lanczos_steps):
        from oracle import krylov as KR
        o = KR.objective_diag(lambda B: self.K @ B, y.numpy(), Z.numpy(), self.c, cg_iters, lanczos_steps)
        return {"quad": o["quad"], "samples": o["samples"], "logdetM": o["logdetM"], "Z": o["Z"]}


def _obj_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = workloads.CONFIGS["c5"]
        n = 600
        X = workloads.make_X(wl, n=n)
        V = workloads.make_V(wl, n=n, r=8)
        plan = OracleObjectivePlan(X, wl.windows, wl.family, (1.0, 0.3, 0.3))
        res = D.sharded_objective(plan, torch.from_numpy(V[:, 0].copy()), torch.from_numpy(V[:, 1:].copy()), 40, 12)
        q.put((rank, res["Z"], res["quad"], res["slq"], res["probes"], res["columns"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_probe_sharded_objective(world):
    """The probe-sharded objective equals the single-process objective with all probes: the CG term
    from rank 0, the SLQ samples of every rank averaged over all n_z probes."""
    from oracle import aafn as A
    from oracle import krylov as KR
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_obj_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = workloads.CONFIGS["c5"]
    X = workloads.make_X(wl, n=600)
    V = workloads.make_V(wl, n=600, r=8)
    K = A.khat_dense(X, wl.windows, wl.family, (1.0, 0.3, 0.3))
    ref = KR.objective_diag(lambda B: K @ B, V[:, 0], V[:, 1:], 1.0**2 * 3 + 0.3**2, 40, 12)  # M = (sf^2 P + se^2) I
    for _, Zt, quad, slq, probes, cols in res:
        assert probes == 7
        assert Zt == pytest.approx(ref["Z"], rel=1e-10)
        assert quad == pytest.approx(ref["quad"], rel=1e-10)
        assert slq == pytest.approx(ref["slq"], rel=1e-10)
    assert [r[5] for r in res] == [D.column_partition(7, world, k) for k in range(world)]


class OracleGradientPlan:
    """Test stand-in for Plan.gradient_columns: oracle PCG (M = c I) and dense derivative products."""

    def __init__(self, X, windows, family, theta):
        from oracle import aafn as A
        from oracle import dense_apply
        self.K = A.khat_dense(X, windows, family, theta)
        self.X, self.windows, self.family, self.theta = X, windows, family, theta
        sf, _, se = theta
        self.c = sf * sf * len(windows) + se * se
        self.dense_apply = dense_apply

    def gradient_columns(self, y, Z, cg_iters, preconditioned=False):
        from oracle import krylov as KR
        y, Z = np.asarray(y), np.asarray(Z)
        minv = np.full(y.size, 1.0 / self.c)
        B = np.column_stack([y, Z])
        Xs = np.stack([KR.pcg(lambda V: self.K @ V, B[:, i], cg_iters, minv)[0] for i in range(B.shape[1])], axis=1)
        B2 = np.column_stack([Xs[:, 0], Z])
        o = self.dense_apply(self.X, self.windows, self.family, self.theta, B2, ops=("dsf", "dell", "dse"))
        dots = np.stack([(Xs * o[k]).sum(axis=0) for k in ("dsf", "dell", "dse")])
        return {"dots": dots, "sqnorms": (B * B).sum(axis=0)}


def _grad_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = workloads.CONFIGS["c5"]
        X = workloads.make_X(wl, n=400)
        V = workloads.make_V(wl, n=400, r=6)
        th = (0.9, 0.3, 0.4)
        plan = OracleGradientPlan(X, wl.windows, wl.family, th)
        g = D.sharded_gradient(plan, torch.from_numpy(V[:, 0].copy()), torch.from_numpy(V[:, 1:].copy()), th,
                               len(wl.windows), 60)
        q.put((rank, g))
    finally:
        dist.destroy_process_group()


def test_gloo_probe_sharded_gradient():
    """The probe-sharded gradient (raw per-column terms summed over ranks, then eq. (div) with M = c I)
    equals the single-process oracle gradient_diag."""
    from oracle import dense_apply
    from oracle import krylov as KR
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = workloads.CONFIGS["c5"]
    X = workloads.make_X(wl, n=400)
    V = workloads.make_V(wl, n=400, r=6)
    th = (0.9, 0.3, 0.4)
    from oracle import aafn as A
    K = A.khat_dense(X, wl.windows, wl.family, th)

    def dK(B):
        o = dense_apply(X, wl.windows, wl.family, th, np.ascontiguousarray(B), ops=("dell", "dsf", "dse"))
        return {"ell": o["dell"], "sf": o["dsf"], "se": o["dse"]}

    P = len(wl.windows)
    c = th[0] ** 2 * P + th[2] ** 2
    ref = KR.gradient_diag(lambda B: K @ B, dK, V[:, 0], V[:, 1:], c, {"sf": 2 * th[0] * P, "ell": 0.0, "se": 2 * th[2]},
                           60)["grad"]
    for _, g in res:
        assert g["probes"] == 5
        for j in ("sf", "ell", "se"):
            assert g[j] == pytest.approx(ref[j], rel=1e-10), j


# ---------------------------------------------------------------- window-sharded product (§8(e) item 3)
class OracleWindowBackend:
    """Test stand-in for the library behind WindowShardedPlan: the truncated-Fourier product (eq. 3.3,
    scaling reading R2) of the oracle over this rank's windows."""

    def set_points(self, X, windows, family, N, sigma_over, m, eps_B):
        self.X, self.windows, self.family, self.N, self.eps_B = np.asarray(X), windows, family, N, eps_B

    def set_theta(self, sf, ell, se):
        self.theta = (sf, ell, se)

    def mvm_multi(self, V, Y=None, dY_ell=None, dY_sf=None):
        from oracle import fourier as F
        out = F.additive_fastsum(self.X, self.windows, self.family, self.theta, V.numpy(), self.N, self.eps_B,
                                 ops=("K", "dell", "dsf"))
        for t, k in ((Y, "K"), (dY_ell, "dell"), (dY_sf, "dsf")):
            if t is not None:
                t.copy_(torch.from_numpy(out[k]))


def _window_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = workloads.CONFIGS["c2"]
        n, r = 400, 2
        X = workloads.make_X(wl, n=n)
        V = torch.from_numpy(np.ascontiguousarray(workloads.make_V(wl, n=n, r=r)))
        sp = D.WindowShardedPlan(X, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B,
                                 backend=OracleWindowBackend())
        sp.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
        Y, dY, dS = torch.empty_like(V), torch.empty_like(V), torch.empty_like(V)
        sp.mvm_multi(V, Y=Y, dY_ell=dY, dY_sf=dS)
        q.put((rank, (sp.w0, sp.w1), Y.numpy(), dY.numpy(), dS.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_window_sharded_product(world):
    """world 2 (windows 2 + 1) and world 4 (> W = 3: one rank holds no window): the sum over the ranks'
    window blocks (sigma_eps^2 V on rank 0 only) and one all-reduce per output reproduce the
    single-process oracle product on every rank, to rounding."""
    from oracle import fourier as F
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_window_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = workloads.CONFIGS["c2"]
    X = workloads.make_X(wl, n=400)
    V = workloads.make_V(wl, n=400, r=2)
    want = F.additive_fastsum(X, wl.windows, wl.family, (wl.sigma_f, wl.ell, wl.sigma_eps), V, wl.N, wl.eps_B,
                              ops=("K", "dell", "dsf"))
    blocks = [b for _, b, *_ in res]
    assert blocks[0][0] == 0 and blocks[-1][1] == len(wl.windows)
    assert all(blocks[k][1] == blocks[k + 1][0] for k in range(world - 1))
    if world > len(wl.windows):
        assert any(b == a for a, b in blocks)              # a rank without windows took part
    for _, _, Y, dY, dS in res:
        for got, key in ((Y, "K"), (dY, "dell"), (dS, "dsf")):
            assert np.abs(got - want[key]).max() <= 1e-12 * np.abs(want[key]).max(), key
