"""Multi-GPU layer.

**Point sharding** (``ShardedPlan``, §8(e) item 1).  The NFFT fast summation is a sum over points:
the inner sums a_k = sum_j v_j e^{-2 pi i k.x_j} of eq. (3.3) are linear in the point
set, and so are the oversampled grids the adjoint NFFT spreads them onto.  Each of G ranks (one
process per GPU) holds a disjoint row block of X and V; it

  1. agrees with the others on the union's window frame (bounding box -> centers, radius -> scale
     factors c_w, reading R2) with two tiny all-reduces at setup, so every rank builds the same
     grid boxes and multiplier tables;
  2. per product: spreads its own points onto full grids (``akm_spread_grid``), then ONE all-reduce
     (sum) of the grids -- W * r * prod(box) doubles, 8.6 MB at c4 -- over NCCL (NVLink/NVSwitch on a
     B200 node), then runs the small DFT / multiply / inverse DFT redundantly and interpolates at its
     own points (``akm_mvm_from_grid``).  No other exchange: the outputs stay row-sharded.

**Window sharding** (``WindowShardedPlan``, §8(e) item 3).  K-hat = sigma_f^2 sum_w K_w +
sigma_eps^2 I is a sum over the windows, each with its own frame (reading R2: c_w depends on that
window's points only).  Each rank holds all rows and a contiguous block of the windows, applies its
windows (rank 0 also the sigma_eps^2 V term), and ONE all-reduce (sum) of each n x r output combines
them.  At most W ranks do work (W <= 4 in BASELINE.json's configs).

**Probe (column) sharding** (``sharded_objective``, §8(e) item 2).  The CG column and every Lanczos
probe of the objective are independent recurrences: each rank holds the whole problem and runs a
slice of the probes (rank 0 also the CG column); one all-reduce of three scalars combines them.

Every step of the arithmetic runs in the library's kernels; this module only orders the calls and
issues the collectives (torch.distributed: ``nccl`` on GPUs, ``gloo`` in the CPU tests, where a
test backend stands in for the library).

Also here: the host bookkeeping bench.py uses under torchrun (row / column partitions, per-rank
seeds, the max-over-ranks timing and the whole-job throughput).
"""
from __future__ import annotations

import math
import os

import numpy as np

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


def row_partition(n: int, world: int, rank: int):
    """Contiguous [start, stop) of ``n`` rows owned by ``rank`` (sizes differ by <= 1; every rank
    needs at least one row for the point-sharded product)."""
    if n < world:
        raise ValueError(f"point sharding needs n >= world ({n} < {world})")
    return column_partition(n, world, rank)


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


def strong_throughput(units_total: float, max_ms_per_step: float) -> float:
    """Whole-job units/s of a fixed total problem split over the ranks (point sharding)."""
    return float(units_total) / (float(max_ms_per_step) * 1e-3)


class ShardedPlan:
    """Point-sharded additive-kernel product over the default process group (see module docstring).

    ``X_local`` / ``V_local`` are this rank's rows (``row_partition``); outputs are this rank's rows of
    K-hat V, dK-hat/d ell V, dK-hat/d sigma_f V.  ``backend`` defaults to the library's ``Plan`` on
    ``device``; the CPU tests pass an object with the same methods."""

    def __init__(self, X_local, windows, family=0, N=32, sigma_over=2.0, m=6, eps_B=1.0 / 16, *, device=None,
                 backend=None, comm_device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        if backend is None:
            from . import Plan
            backend = Plan(0 if device is None else int(torch.device(device).index or 0))
        self.backend = backend
        self.comm_device = comm_device if comm_device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu"))
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self._grid = None
        backend.set_points(X_local, windows, family, N, sigma_over, m, eps_B)
        lo, hi = backend.bounds()
        lo = self._reduce(lo, dist.ReduceOp.MIN)
        hi = self._reduce(hi, dist.ReduceOp.MAX)
        rad = backend.set_bounds(lo, hi)
        backend.set_radius(self._reduce(rad, dist.ReduceOp.MAX))

    def _reduce(self, arr, op):
        t = self.torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64), device=self.comm_device)
        self.dist.all_reduce(t, op=op)
        return t.cpu().numpy().reshape(np.shape(arr))

    def set_theta(self, sigma_f, ell, sigma_eps):
        """set_theta on every rank; the bin edges must agree (the grid boxes depend on them)."""
        self.backend.set_theta(sigma_f, ell, sigma_eps)
        bins = np.asarray(self.backend.info()["bin"], dtype=np.float64)
        first = bins.copy()
        t = self.torch.as_tensor(first, device=self.comm_device)
        self.dist.broadcast(t, src=0)
        first = t.cpu().numpy()
        if not np.array_equal(first, bins):
            self.backend.set_bin_override(first.astype(np.int32))
            self.backend.set_theta(sigma_f, ell, sigma_eps)
        return self

    def info(self):
        return self.backend.info()

    def grid_buffer(self, r, like):
        size = self.backend.grid_size(r)
        if self._grid is None or self._grid.numel() < size or self._grid.device != like.device:
            self._grid = self.torch.empty(size, dtype=self.torch.float64, device=like.device)
        return self._grid[:size]

    def mvm_multi(self, V_local, Y=None, dY_ell=None, dY_sf=None):
        """This rank's rows of the requested products: spread, all-reduce the grids, finish."""
        r = V_local.shape[1] if V_local.dim() == 2 else 1
        grid = self.grid_buffer(r, V_local)
        self.backend.spread_grid(V_local, grid)
        self.dist.all_reduce(grid)
        self.backend.mvm_from_grid(grid, V_local, Y, dY_ell, dY_sf)
        return Y, dY_ell, dY_sf

    def close(self):
        close = getattr(self.backend, "close", None)
        if close:
            close()


def window_partition(P: int, world: int, rank: int):
    """Contiguous [start, stop) of the ``P`` windows owned by ``rank`` (empty when world > P for the
    last ranks; rank 0 always holds one when P >= 1)."""
    return column_partition(P, world, rank)


class WindowShardedPlan:
    """Window-sharded additive-kernel product over the default process group (module docstring).

    Every rank passes ALL rows of ``X``; it builds a plan for its block of ``windows``
    (``window_partition``).  ``mvm_multi`` returns the full products on every rank: the local windows'
    sum (rank 0 adds sigma_eps^2 V), then one all-reduce per requested output.  ``backend`` defaults to
    the library's ``Plan`` on ``device``; the CPU tests pass an object with the same methods."""

    def __init__(self, X, windows, family=0, N=32, sigma_over=2.0, m=6, eps_B=1.0 / 16, *, device=None,
                 backend=None, comm_device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.w0, self.w1 = window_partition(len(windows), self.world, self.rank)
        self.windows = [tuple(w) for w in windows][self.w0:self.w1]
        self.comm_device = comm_device
        self.backend = None
        if self.windows:
            if backend is None:
                from . import Plan
                backend = Plan(0 if device is None else int(torch.device(device).index or 0))
            self.backend = backend
            backend.set_points(X, self.windows, family, N, sigma_over, m, eps_B)

    def set_theta(self, sigma_f, ell, sigma_eps):
        """theta on the local windows; the sigma_eps^2 I term belongs to rank 0 only."""
        if self.backend is not None:
            self.backend.set_theta(sigma_f, ell, sigma_eps if self.rank == 0 else 0.0)
        return self

    def info(self):
        return self.backend.info() if self.backend is not None else {"P": 0}

    def mvm_multi(self, V, Y=None, dY_ell=None, dY_sf=None):
        """The full products on every rank: the local windows' part, then one all-reduce per output."""
        outs = [t for t in (Y, dY_ell, dY_sf) if t is not None]
        if self.backend is not None:
            self.backend.mvm_multi(V, Y=Y, dY_ell=dY_ell, dY_sf=dY_sf)
        else:
            for t in outs:
                t.zero_()
        for t in outs:
            if self.comm_device is None or t.device == self.comm_device:
                self.dist.all_reduce(t)
            else:  # the collective's device differs from the output's (gloo on CPU for GPU outputs)
                c = t.to(self.comm_device)
                self.dist.all_reduce(c)
                t.copy_(c)
        return Y, dY_ell, dY_sf

    def close(self):
        close = getattr(self.backend, "close", None)
        if close:
            close()


def sharded_objective(plan, y, Z, cg_iters=50, lanczos_steps=30, comm_device=None, preconditioned=False):
    """Z~ (eq. 1.4) with the probe columns sharded over the ranks (the CG column
    and every Lanczos probe are independent recurrences, so no exchange is needed until the scalars).

    Every rank holds the whole problem (all n points) in ``plan``; the n_z probe columns of ``Z`` are
    split by ``column_partition``.  Rank 0 runs CG on y together with its probes; the other ranks run
    their probes with y = 0 (the library's CG column is then inactive) and no CG iterations.  One
    all-reduce of [y^T x, sum of SLQ samples, probe count] combines them:
        Z~ = 1/2 (y^T x + log det M + (1/n_z) sum_i samples_i + n log 2 pi).
    ``preconditioned`` uses ``plan.objective`` (the plan's preconditioner, e.g. AAFN) instead of
    ``plan.objective_diag``.  Returns the terms as a dict (like ``Plan.objective_diag``)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    n_z = Z.shape[1]
    c0, c1 = column_partition(n_z, world, rank)
    fn = plan.objective if preconditioned else plan.objective_diag
    quad, ssum, cnt, out = 0.0, 0.0, 0, None
    if c1 > c0:
        Zk = Z[:, c0:c1]
        Zk = Zk.contiguous() if hasattr(Zk, "contiguous") else np.ascontiguousarray(Zk)
        if rank == 0:
            out = fn(y, Zk, cg_iters, lanczos_steps)
            quad = out["quad"]
        else:
            y0 = torch.zeros_like(y) if hasattr(y, "new_zeros") else np.zeros_like(y)
            out = fn(y0, Zk, 0, lanczos_steps)
        ssum, cnt = float(sum(out["samples"])), c1 - c0
    dev = comm_device if comm_device is not None else (
        torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu"))
    t = torch.tensor([quad, ssum, float(cnt)], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    quad, ssum, cnt = (float(v) for v in t.cpu())
    n = y.shape[0]
    logdet = torch.tensor([out["logdetM"] if (out is not None and rank == 0) else 0.0], dtype=torch.float64, device=dev)
    dist.broadcast(logdet, src=0)
    logdet = float(logdet.item())
    slq = ssum / cnt
    res = {"Z": 0.5 * (quad + logdet + slq + n * math.log(2.0 * math.pi)), "quad": quad, "logdetM": logdet,
           "slq": slq, "probes": int(cnt), "local": out, "columns": (c0, c1)}
    return res


def sharded_gradient(plan, y, Z, theta, P, cg_iters=50, comm_device=None, preconditioned=False):
    """grad Z~ (eq. (div)) with the probe columns sharded over the ranks.

    Rank 0 solves for alpha = Khat^{-1} y with its probes, the other ranks their probes with y = 0;
    every rank returns its raw per-column terms (``Plan.gradient_columns``), one all-reduce sums them,
    and the components are assembled as akm_gradient_diag does (include/akm.h):
        grad_k = 1/2 ( -alpha^T dK_k alpha + n dc_k/c + (1/n_z) sum_i (z_i^T Khat^{-1} dK_k z_i - dc_k/c ||z_i||^2) ),
    c = sigma_f^2 P + sigma_eps^2, dc = (2 sigma_f P, 0, 2 sigma_eps); under AAFN (``preconditioned``) dc = 0.
    ``theta`` = (sigma_f, ell, sigma_eps) of the plan, ``P`` its window count.  Returns the gradient
    in the order (sigma_f, ell, sigma_eps)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    n_z = Z.shape[1]
    c0, c1 = column_partition(n_z, world, rank)
    acc = np.zeros(3 * 2 + 1)  # [alpha terms (3) | probe sums (3) | probe count]
    if c1 > c0:
        Zk = Z[:, c0:c1]
        Zk = Zk.contiguous() if hasattr(Zk, "contiguous") else np.ascontiguousarray(Zk)
        y_k = y if rank == 0 else (torch.zeros_like(y) if hasattr(y, "new_zeros") else np.zeros_like(y))
        out = plan.gradient_columns(y_k, Zk, cg_iters if rank == 0 else cg_iters, preconditioned)
        sf, _, se = theta
        c = sf * sf * P + se * se
        dc = np.zeros(3) if preconditioned else np.array([2.0 * sf * P, 0.0, 2.0 * se])
        dots, sq = out["dots"], out["sqnorms"]
        acc[0:3] = dots[:, 0] if rank == 0 else 0.0
        acc[3:6] = (dots[:, 1:] - (dc / c)[:, None] * sq[None, 1:]).sum(axis=1)
        acc[6] = c1 - c0
    dev = comm_device if comm_device is not None else (
        torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu"))
    t = torch.as_tensor(acc, dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    acc = t.cpu().numpy()
    sf, _, se = theta
    c = sf * sf * P + se * se
    dc = np.zeros(3) if preconditioned else np.array([2.0 * sf * P, 0.0, 2.0 * se])
    n = y.shape[0]
    g = 0.5 * (-acc[0:3] + n * dc / c + acc[3:6] / acc[6])
    return {"sf": float(g[0]), "ell": float(g[1]), "se": float(g[2]), "probes": int(acc[6])}
