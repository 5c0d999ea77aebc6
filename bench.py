#!/usr/bin/env python
"""bench.py -- batched additive-kernel MVM throughput on B200 (BASELINE.json metric).

One "step" is one pass of the hot path: a single
``akm_kernel_mvm_multi`` call through the C ABI producing every product the workload requests
(e.g. c2: K-hat v and dK-hat/d ell v), on inputs already resident in HBM.  set_points / set_theta
(S0/S1, once per X / theta) run before the timed region.

  value  = n * r * windows / (device time per step)            [pts/s, whole job over N GPUs]
  e2e    = the same through the C ABI with pinned HOST V and outputs (H2D + D2H inside the timing)
  roofline: the dominant kernel (from in-library CUDA events on the launching stream) against the
           FP64 FMA peak (the path is FP64-ALU bound)
  cpu_baseline: the float64 dense oracle (oracle/dense.c) on a bounded row sample, rank 0, N = 1

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]
Under torchrun (N > 1) the square products (c1-c4) are point-sharded: each rank owns a row block of
the same problem and every product does one NCCL all-reduce of the grids (strong scaling,
"scaling": "strong"); the Krylov drivers (c5, g5) and the cross product (x4) run one independent
replica per rank (weak scaling).  Rank 0 prints the max-over-ranks timing.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

PEAK_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2: SMs x FP64 FMA/clk/SM x 2 x max SM clock
MEASURED_FP64 = {"dfma_tflops": 34.1, "dmma_tflops": 37.1, "source": "profiles/r01_fp64_peaks.txt"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()

    @staticmethod
    def one_shot(gpu_index):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={ClockSampler.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20).stdout
            return [l.strip() for l in out.splitlines() if l.strip()]
        except Exception:
            return []

    def summary(self, extra_lines=()):
        rows = []
        for line in list(self.lines) + list(extra_lines):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[4:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, flags in rows:
            for nm, fl in zip(names, flags[1:5]):
                if fl.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


def algorithmic_counts(wl, info, r, ops, n_local=None):
    """FP64 flops of spreading / interpolation and minimal bytes of one step on this
    rank (n_local: its rows under point sharding).
    Cross products (extra n_src): the method spreads the sources and interpolates at the targets."""
    n, W = (wl.n if n_local is None else n_local), len(wl.windows)
    n_s = wl.extra.get("n_src", n)
    n_i = n - n_s if "n_src" in wl.extra else n
    d = [len(w) for w in wl.windows]
    taps = [(2 * wl.m) ** dw for dw in d]
    n_ops = len({"K" if o in ("K", "dsf") else o for o in ops})      # distinct operators interpolated
    spread_flops = sum(2.0 * n_s * r * t for t in taps)
    interp_flops = sum(2.0 * n_i * r * t * n_ops for t in taps)
    ntap = [int(np.prod(b)) for b in info["box"]]
    grid_bytes = sum(8.0 * nt * r * (2 + 2 * n_ops) for nt in ntap)
    bytes_ = 8.0 * (n_s + n_i) * sum(d) + 8.0 * n_s * r + 8.0 * n_i * r * len(ops) + grid_bytes
    return spread_flops, interp_flops, bytes_


def stage_bytes(wl, info, r, ops, n_local=None):
    """Algorithmic HBM bytes per MVM of each stage (BJ north_star: HBM GB/s of spreading, DFT and
    interpolation): what the stage must read and write at least, with every grid in HBM.
      spread: coordinates (d doubles per point-window) + permutation (int32) + V rows + grid write;
      fft:    grid read + H write (one grid per interpolated operator);
      interp: H read + coordinates + permutation + per-window partial outputs;
      epilogue: partials read + V (noise term) + outputs."""
    n, W = (wl.n if n_local is None else n_local), len(wl.windows)
    n_s = wl.extra.get("n_src", n)
    n_i = n - n_s if "n_src" in wl.extra else n
    d = [len(w) for w in wl.windows]
    n_ops = len({"K" if o in ("K", "dsf") else o for o in ops})
    ntap = [int(np.prod(b)) for b in info["box"]]
    grid = sum(8.0 * nt * r for nt in ntap)
    return {
        "spread": 8.0 * n_s * sum(d) + 4.0 * n_s * W + 8.0 * n_s * r + grid,
        "fft": grid + grid * n_ops,
        "interp": grid * n_ops + 8.0 * n_i * sum(d) + 4.0 * n_i * W + 8.0 * n_i * r * n_ops * W,
        "epilogue": 8.0 * n_i * r * n_ops * W + 8.0 * n_i * r + 8.0 * n_i * r * len(ops),
    }


def _oracle_inputs(wl):
    """(X, V, theta, candidate rows) for the CPU oracle legs.  Cross workloads: the dense products
    on the union with the targets' V rows zero are exactly the cross product at the target rows
    (tests/test_oracle_cross.py), so the targets' rows are sampled."""
    X = workloads.make_X(wl)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    if "n_src" in wl.extra:
        n_s = wl.extra["n_src"]
        V = np.vstack([workloads.make_V(wl, n=n_s), np.zeros((wl.n - n_s, wl.r))])
        rows_all = n_s + workloads.make_rows(wl, wl.n - n_s, n=wl.n - n_s)
    else:
        V = workloads.make_V(wl)
        rows_all = workloads.make_rows(wl, wl.n)
    return X, V, theta, rows_all


def _metric(wl):
    if "n_src" in wl.extra:
        return "cross K_{*X} V throughput (n_target*r*windows pts/s)"
    return "batched K-hat V throughput (n*r*windows pts/s)"


def run_reference(args, wl):
    """The reference arm: the CPU float64 dense oracle timed as it stands on bounded row samples."""
    from oracle import dense_apply
    X, V, theta, rows_all = _oracle_inputs(wl)
    n_rows = rows_all.shape[0]
    # calibrate the sample so that each step is ~1-3 s of CPU work
    t0 = time.perf_counter()
    dense_apply(X, wl.windows, wl.family, theta, V, rows=rows_all[:64], ops=wl.ops)
    per_row = (time.perf_counter() - t0) / 64
    # each step ~2 s of CPU work, and the whole --warmup + --steps run within ~2 minutes
    step_budget = min(2.0, 120.0 / max(1, args.warmup + args.steps))
    rows_per_step = int(min(n_rows, max(64, step_budget / max(per_row, 1e-9))))
    times = []
    for s in range(args.warmup + args.steps):
        rows = rows_all[(s * rows_per_step) % max(1, n_rows - rows_per_step + 1):][:rows_per_step]
        t0 = time.perf_counter()
        dense_apply(X, wl.windows, wl.family, theta, V, rows=rows, ops=wl.ops)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    full_equiv = t * n_rows / rows_per_step
    value = wl.units / full_equiv
    cores = os.cpu_count()
    sample = f"{rows_per_step} of {n_rows} rows per step (dense direct sums, all {wl.n} columns), extrapolated x{n_rows / rows_per_step:.1f}"
    line = {
        "impl": "reference", "metric": _metric(wl), "value": value,
        "unit": "pts/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": full_equiv * 1e3,
        "higher_is_better": True, "scaling": "none", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(wl),
        "cpu_baseline": {"value": value, "unit": "pts/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "pts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(wl, parallelism="1 GPU"):
    extra = {"n_src": wl.extra["n_src"], "n_target": wl.n - wl.extra["n_src"]} if "n_src" in wl.extra else {}
    return {"workload": wl.name, "description": wl.description, "n": wl.n, **extra, "r": wl.r, "windows": len(wl.windows),
            "d": [len(w) for w in wl.windows], "family": "gaussian" if wl.family == 0 else "matern12",
            "N": wl.N, "sigma_over": wl.sigma_over, "m": wl.m, "ops": list(wl.ops),
            "l2": "256 MiB written between timed steps (L2 flush)", "parallelism": parallelism}


def cpu_baseline(wl, budget_s=10.0):
    from oracle import dense_apply
    X, V, theta, rows_all = _oracle_inputs(wl)
    t0 = time.perf_counter()
    dense_apply(X, wl.windows, wl.family, theta, V, rows=rows_all[:32], ops=wl.ops)
    per_row = max((time.perf_counter() - t0) / 32, 1e-9)
    nrows = int(min(rows_all.shape[0], max(32, budget_s / per_row)))
    t0 = time.perf_counter()
    dense_apply(X, wl.windows, wl.family, theta, V, rows=rows_all[:nrows], ops=wl.ops)
    t = time.perf_counter() - t0
    value = nrows * wl.r * len(wl.windows) / t
    return {"value": value, "unit": "pts/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{nrows} seeded rows of {rows_all.shape[0]} (all {wl.n} columns) of the dense float64 products "
                      f"{list(wl.ops)}; "
                      f"{t:.1f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-launches", action="store_true", help="short run for ncu launch lists")
    args = ap.parse_args()
    wl = workloads.CONFIGS[args.config]

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, wl)
        return

    import torch
    import paper_2504_00480_b200 as akm
    from paper_2504_00480_b200 import dist as D   # host-side N > 1 logic only (no kernels)

    # AKM_BENCH_DEVICE / AKM_BENCH_BACKEND: exercise the N > 1 code path on a single GPU (every rank on
    # one device over gloo; a plumbing check only, never a timing)
    if os.environ.get("AKM_BENCH_DEVICE"):
        local = int(os.environ["AKM_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("AKM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    X = workloads.make_X(wl)
    cross = "n_src" in wl.extra              # f2: K_{*X} V from the first n_src rows to the rest
    n_src = wl.extra.get("n_src", wl.n)
    objective = "cg_iters" in wl.extra          # c5: one Z~ evaluation per step (S8)
    gradient = "grad_cg_iters" in wl.extra      # g5: one gradient of Z~ per step (f1)
    probe_sharded = world > 1 and (objective or gradient)  # c5 / c5a / g5: probe columns over the ranks (§8(e) 2)
    # N > 1: the square products are point-sharded (each rank owns a row block of the SAME problem,
    # one grid all-reduce per product: strong scaling); the Krylov drivers and the cross
    # product run as independent replicas (weak scaling)
    sharded = world > 1 and not (objective or gradient or cross)
    if sharded:
        row0, row1 = D.row_partition(wl.n, world, rank)
        V = workloads.make_V(wl)[row0:row1]
        Xd = torch.from_numpy(np.ascontiguousarray(X[row0:row1])).to(dev)
    else:
        row0, row1 = 0, wl.n
        # independent RHS block per rank (replicas); the probe-sharded objective shares one problem
        V = workloads.make_V(wl, n=n_src, seed=None if probe_sharded else D.rank_seed(2000 + wl.index, rank))
        Xd = torch.from_numpy(X).to(dev)
    V = np.ascontiguousarray(V)
    Vd = torch.from_numpy(V).to(dev)
    outs = {op: torch.empty_like(Vd) for op in wl.ops}
    if cross:
        outs = {"K": torch.empty((wl.n - n_src, wl.r), dtype=torch.float64, device=dev)}
    stream = torch.cuda.current_stream(dev)

    t0 = time.perf_counter()
    if sharded:
        sp = D.ShardedPlan(Xd, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B, device=dev)
        sp.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
        plan = sp.backend
    else:
        plan = akm.Plan(local)
        plan.set_points(Xd, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
        if "reg_p" in wl.extra:                 # f4: kappa_R with the near-field correction
            plan.set_regularization(wl.extra["reg_eps_I"], wl.extra["reg_p"])
        if "aafn_kpw" in wl.extra:              # f3: AAFN preconditioner
            plan.set_preconditioner(wl.extra["aafn_kpw"])
        plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    torch.cuda.synchronize(dev)
    set_theta_ms = (time.perf_counter() - t0) * 1e3   # set_points + the first set_theta (allocations)
    # a theta step as an optimizer takes it: ell moved by 1% (Gaussian windows re-bin: c_w follows
    # ell), median of 3, host wall clock around the synchronised call; theta restored afterwards
    setter = sp if sharded else plan
    warm = []
    for k in range(3):
        a = time.perf_counter()
        setter.set_theta(wl.sigma_f, wl.ell * (1.0 + 0.01 * (k + 1)), wl.sigma_eps)
        torch.cuda.synchronize(dev)
        warm.append((time.perf_counter() - a) * 1e3)
    setter.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    torch.cuda.synchronize(dev)
    set_theta_warm_ms = float(np.median(warm))
    info = plan.info()

    if objective:
        cg, lz = wl.extra["cg_iters"], wl.extra["lanczos_steps"]
        yd, Zd = Vd[:, 0].contiguous(), Vd[:, 1:].contiguous()
        products_per_step = max(cg, lz)
        last = {}

        if probe_sharded:
            def step():   # every rank: the whole problem, a slice of the probes (rank 0 also CG)
                if "aafn_kpw" in wl.extra:
                    plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
                res = D.sharded_objective(plan, yd, Zd, cg, lz, preconditioned="aafn_kpw" in wl.extra)
                loc = res["local"] or {}
                last["out"] = {**loc, "Z": res["Z"], "quad": res["quad"], "slq": res["slq"],
                               "product_columns": loc.get("product_columns", 0)}
        elif "aafn_kpw" in wl.extra:
            def step():   # theta -> AAFN factors -> Z~ (the factors depend on theta: rebuilt every step)
                plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
                last["out"] = plan.objective(yd, Zd, cg, lz)
        else:
            def step():
                last["out"] = plan.objective_diag(yd, Zd, cg, lz)
    elif gradient and probe_sharded:
        gcg = wl.extra["grad_cg_iters"]
        yd, Zd = Vd[:, 0].contiguous(), Vd[:, 1:].contiguous()
        products_per_step = gcg + 1
        last = {}

        def step():   # every rank: the whole problem, a slice of the probes (rank 0 also alpha)
            g = D.sharded_gradient(plan, yd, Zd, (wl.sigma_f, wl.ell, wl.sigma_eps), len(wl.windows), gcg)
            last["out"] = {"grad": {k: g[k] for k in ("sf", "ell", "se")}, "cg_hist": [float("nan")]}
    elif gradient:
        gcg = wl.extra["grad_cg_iters"]
        yd, Zd = Vd[:, 0].contiguous(), Vd[:, 1:].contiguous()
        products_per_step = gcg + 1
        last = {}

        def step():
            last["out"] = plan.gradient_diag(yd, Zd, gcg)
    elif cross:
        products_per_step = 1

        def step():
            plan.cross_mvm(n_src, Vd, outs["K"])
    elif sharded:
        products_per_step = 1

        def step():
            sp.mvm_multi(Vd, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))
    else:
        products_per_step = 1

        def step():
            plan.mvm_multi(Vd, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    if objective:   # after the Lanczos steps only the CG column is multiplied: count live columns only
        cols = float(last["out"]["product_columns"])
        if probe_sharded:   # the whole job's columns (every rank's slice)
            tcols = torch.tensor([cols], dtype=torch.float64, device=dev)
            dist.all_reduce(tcols)
            cols = float(tcols.item())
        products_per_step = cols / wl.r

    K = args.steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    plan.stage_times(reset=True)          # zero the launch counters: the timed region counts its own
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    for i in range(K):
        flush.fill_(float(i))
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    sampler.stop()
    tail = ClockSampler.one_shot(local)
    launches_timed = plan.stage_times(reset=True)["kernel_launches"]
    total_ms = D.max_over_ranks(sum(s.elapsed_time(e) for s, e in zip(starts, ends)), dev)
    ms_per_step = total_ms / K
    if sharded or probe_sharded:
        value = D.strong_throughput(wl.units * products_per_step, ms_per_step)
    else:
        value = D.weak_throughput(wl.units * products_per_step, world, ms_per_step)

    # ---------------- per-stage device times: a separate pass of the same steps with the library's
    # stage events on the launching stream (direct launches; the timed region above replays the
    # captured CUDA graph and records no stage events)
    plan.set_profiling(True)
    for i in range(K):
        flush.fill_(float(i))
        step()
    torch.cuda.synchronize(dev)
    plan.set_profiling(False)
    stages = plan.stage_times(reset=True)

    # ---------------- e2e: same call with pinned host V and outputs
    Vh = torch.from_numpy(V).pin_memory()
    Oh = {op: torch.empty(tuple(outs[op].shape) if cross else V.shape, dtype=torch.float64).pin_memory()
          for op in wl.ops}
    if objective or gradient:
        yh, Zh = Vh[:, 0].contiguous().pin_memory(), Vh[:, 1:].contiguous().pin_memory()

    def e2e_step():
        if probe_sharded and gradient:
            D.sharded_gradient(plan, yh, Zh, (wl.sigma_f, wl.ell, wl.sigma_eps), len(wl.windows), gcg)
        elif probe_sharded:
            if "aafn_kpw" in wl.extra:
                plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
            D.sharded_objective(plan, yh, Zh, cg, lz, preconditioned="aafn_kpw" in wl.extra)
        elif objective and "aafn_kpw" in wl.extra:
            plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
            plan.objective(yh, Zh, cg, lz, stream=stream.cuda_stream)
        elif objective:   # host y, Z in; the objective's terms come back to the host
            plan.objective_diag(yh, Zh, cg, lz, stream=stream.cuda_stream)
        elif gradient:  # host y, Z in; the three components come back to the host
            plan.gradient_diag(yh, Zh, gcg, stream=stream.cuda_stream)
        elif cross:
            plan.cross_mvm(n_src, Vh, Oh["K"], stream=stream.cuda_stream)
        elif sharded:   # the caller's copies around the sharded product (its entry points take device memory)
            Vd.copy_(Vh, non_blocking=True)
            sp.mvm_multi(Vd, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))
            for op in wl.ops:
                Oh[op].copy_(outs[op], non_blocking=True)
        else:
            plan.mvm_multi(Vh, Y=Oh.get("K"), dY_ell=Oh.get("dell"), dY_sf=Oh.get("dsf"), stream=stream.cuda_stream)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize(dev)
    e_s = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    e_e = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if dist:
        dist.barrier()
    for i in range(K):
        flush.fill_(float(i))
        e_s[i].record(stream)
        e2e_step()
        e_e[i].record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = D.max_over_ranks(sum(s.elapsed_time(e) for s, e in zip(e_s, e_e)), dev)
    e2e_sync_ms = e2e_ms
    # streaming host batches (akm_kernel_mvm_pipelined): the same K products from the same pinned
    # host blocks, every step's V copied in and outputs copied out, with batch k's copy-out and batch
    # k+1's copy-in overlapping the products; one device-timed region from before the first copy-in
    # (e0 has completed before the first call is issued) to the last copy-out (pipeline_wait)
    # (batches under the library's 4 MiB split threshold -- c1, c2 -- are host-bound through the Python
    # binding when nothing blocks: they keep the synchronous call's per-step device intervals)
    pipelined = not (objective or gradient or cross or sharded) and V.nbytes >= (4 << 20)
    if pipelined:
        def pipe_step():
            plan.mvm_pipelined(Vh, Y=Oh.get("K"), dY_ell=Oh.get("dell"), dY_sf=Oh.get("dsf"), stream=stream.cuda_stream)
        for _ in range(3):
            pipe_step()
        plan.pipeline_wait(stream=stream.cuda_stream)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        e0.record(stream)
        e0.synchronize()
        for i in range(K):
            flush.fill_(float(i))
            pipe_step()
        plan.pipeline_wait(stream=stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = D.max_over_ranks(e0.elapsed_time(e1), dev)
    if sharded or probe_sharded:
        e2e_value = D.strong_throughput(wl.units * products_per_step, e2e_ms / K)
    else:
        e2e_value = D.weak_throughput(wl.units * products_per_step, world, e2e_ms / K)
        e2e_sync_value = D.weak_throughput(wl.units * products_per_step, world, e2e_sync_ms / K)

    # ---------------- roofline of the dominant kernel
    spread_fl, interp_fl, alg_bytes = algorithmic_counts(wl, info, wl.r, wl.ops, n_local=row1 - row0)
    alg_bytes *= products_per_step
    cand = []
    if stages["spread_launches"]:
        cand.append(("spread", stages["spread_ms"], stages["spread_launches"], spread_fl))
    if stages["interp_launches"]:
        cand.append(("interp", stages["interp_ms"], stages["interp_launches"], interp_fl))
    name, st_ms, launches, flops = max(cand, key=lambda c: c[1])
    try:   # DRAM traffic of that kernel per launch, from the round's committed ncu capture
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["bytes_per_launch"][wl.name][name]
    except Exception:
        traffic = None
    per_launch_ms = st_ms / launches
    flops_per_launch = flops * products_per_step / (launches / K)
    achieved = flops_per_launch / (per_launch_ms * 1e-3) / 1e12
    peaks = _peaks()
    stage_total = stages["spread_ms"] + stages["fft_ms"] + stages["interp_ms"] + stages["epilogue_ms"]
    # per-stage HBM rate (algorithmic bytes / stage time) and, where the round's ncu capture has
    # this workload, the measured DRAM bytes of the stage's dominant kernel per launch
    sb = stage_bytes(wl, info, wl.r, wl.ops, n_local=row1 - row0)
    try:
        measured = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["bytes_per_launch"].get(wl.name, {})
    except Exception:
        measured = {}
    hbm_stages = {}
    for k in ("spread", "fft", "interp", "epilogue"):
        t = stages[k + "_ms"] / (K * products_per_step) * 1e-3  # seconds per MVM
        if t <= 0:
            continue
        e = {"algorithmic_bytes": sb[k], "gbs": sb[k] / t / 1e9, "frac": sb[k] / t / 1e9 / peaks.get("hbm_gbs", 6650.0)}
        if k in measured and stages.get(k + "_launches"):
            per_mvm = measured[k] * stages[k + "_launches"] / (K * products_per_step)
            e["dram_bytes_ncu"] = per_mvm
            e["dram_gbs_ncu"] = per_mvm / t / 1e9
        hbm_stages[k] = e
    clocks = sampler.summary(tail)

    line = {
        "metric": _metric(wl),
        "value": value, "unit": "pts/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if (sharded or probe_sharded) else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_dict(wl, f"point-sharded rows x{world} (one grid all-reduce per product)" if sharded else
                              f"probe columns sharded x{world} (one scalar all-reduce per evaluation)" if probe_sharded
                              else f"independent replicas x{world}" if world > 1 else "1 GPU"),
        "e2e": {"value": e2e_value, "unit": "pts/s", "h2d_bytes_per_step": int(V.nbytes),
                "d2h_bytes_per_step": int(8 * (10 + 2 * wl.r) if objective else 8 * (3 + gcg) if gradient else
                                          sum(o.numel() * 8 for o in Oh.values())),
                "api": "akm_kernel_mvm_pipelined (streaming host batches)" if pipelined else "synchronous host-buffer call"},
        "gpu_launches": int(launches_timed),
        "roofline": {"bound": "alu", "kernel": name, "achieved": achieved, "peak": PEAK_FP64_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / PEAK_FP64_TFLOPS, "traffic": traffic,
                     "peak_note": "FP64 FMA: 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz; measured DFMA 34.1 / DMMA 37.1 "
                                  "TFLOP/s (profiles/r01_fp64_peaks.txt)",
                     "algorithmic_flops_per_launch": flops_per_launch, "avg_launch_ms": per_launch_ms},
        "stages_ms_per_step": {k: stages[k + "_ms"] / K for k in ("spread", "fft", "interp", "epilogue", "exchange")},
        "stage_share": {k: stages[k + "_ms"] / stage_total for k in ("spread", "fft", "interp", "epilogue")},
        "hbm": {"algorithmic_bytes_per_step": alg_bytes, "achieved_gbs": alg_bytes / (ms_per_step * 1e-3) / 1e9,
                "peak_gbs": peaks.get("hbm_gbs"), "frac": alg_bytes / (ms_per_step * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0)},
        "hbm_stages": hbm_stages,
        "set_theta_ms": set_theta_ms,
        "set_theta_warm_ms": set_theta_warm_ms,
        "products_per_step": products_per_step,
        "plan": {"bin": info["bin"], "box": info["box"], "c_w": info["c_w"], "work_items_spread": info["work_items_spread"],
                 "work_items_interp": info["work_items_interp"], "max_bin_points": info["max_bin_points"]},
        "clocks": clocks,
    }
    if pipelined:   # the same K steps through the synchronous host-buffer call (no overlap), for reference
        line["e2e"]["synchronous_call_value"] = e2e_sync_value
    if objective:
        o = last["out"]
        line["objective"] = {"Z": o["Z"], "quad": o["quad"], "logdetM": o["logdetM"], "slq": o["slq"],
                             "cg_relres": o["cg_relres"], "cg_relres_true": o["cg_relres_true"],
                             "landmarks": o["landmarks"], "steps": o["steps"], "ms_per_evaluation": ms_per_step,
                             "ms_per_product": ms_per_step / products_per_step}
    if gradient:
        line["gradient"] = {"grad": last["out"]["grad"], "cg_relres_last": last["out"]["cg_hist"][-1],
                            "ms_per_evaluation": ms_per_step, "ms_per_product": ms_per_step / products_per_step}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl)
    plan.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
