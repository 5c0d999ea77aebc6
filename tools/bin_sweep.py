"""Per-stage device times of one workload's MVM at forced bin edges (akm_set_bin_override).

    python tools/bin_sweep.py --config c3 --bins 2 3 4 6 8 [--calls 30]

Prints one line per B: the mean per-call stage times (library CUDA events on the launching stream,
akm_set_profiling) and the whole call (CUDA events around the calls).  B = 0 is the cost model's
own choice.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2504_00480_b200 as akm  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--bins", type=int, nargs="+", default=[0])
    ap.add_argument("--calls", type=int, default=30)
    a = ap.parse_args()
    wl = workloads.CONFIGS[a.config]
    X = workloads.make_X(wl)
    V = workloads.make_V(wl)
    dev = torch.device("cuda:0")
    Xd, Vd = torch.from_numpy(X).to(dev), torch.from_numpy(V).to(dev)
    outs = {op: torch.empty_like(Vd) for op in wl.ops}
    for B in a.bins:
        plan = akm.Plan(0)
        plan.set_points(Xd, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
        if B:
            plan.set_bin_override([B] * len(wl.windows))
        plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
        call = lambda: plan.mvm_multi(Vd, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))
        for _ in range(5):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.calls):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.calls
        akm.akm_set_profiling(plan.handle, 1)
        akm.akm_get_stage_times(plan.handle, reset=True)
        for _ in range(a.calls):
            call()
        torch.cuda.synchronize()
        st = akm.akm_get_stage_times(plan.handle, reset=True)
        calls = max(1, st.get("calls", a.calls))
        stages = {k: round(v / calls, 4) for k, v in st.items() if k.endswith("_ms")}
        print(f"{a.config} B={B or 'auto'} bins={plan.info()['bin']} call {ms:.4f} ms stages {stages}", flush=True)
        plan.close()


if __name__ == "__main__":
    main()
