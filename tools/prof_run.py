"""Short driver for ncu / compute-sanitizer: set up one BASELINE.json workload and run a few MVM calls.

    python tools/prof_run.py --config c2 --calls 3
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
    ap.add_argument("--config", default="c2")
    ap.add_argument("--calls", type=int, default=3)
    ap.add_argument("--n", type=int, default=None)
    a = ap.parse_args()
    wl = workloads.CONFIGS[a.config]
    X = workloads.make_X(wl, n=a.n)
    V = workloads.make_V(wl, n=a.n)
    dev = torch.device("cuda:0")
    Xd, Vd = torch.from_numpy(X).to(dev), torch.from_numpy(V).to(dev)
    outs = {op: torch.empty_like(Vd) for op in wl.ops}
    plan = akm.Plan(0)
    plan.set_points(Xd, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
    if "reg_eps_I" in (wl.extra or {}):  # c3r: kappa_R with the near-field correction
        plan.set_regularization(wl.extra["reg_eps_I"], wl.extra["reg_p"])
    plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    for _ in range(a.calls):
        plan.mvm_multi(Vd, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))
    torch.cuda.synchronize()
    print("info", plan.info())
    plan.close()


if __name__ == "__main__":
    main()
