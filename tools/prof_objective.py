"""Kernel-time breakdown of one objective evaluation (c5) with the CUDA activity profiler (CUPTI via
torch.profiler; no nsys on this image).  Not a bench number: profiler overhead is included.

    python tools/prof_objective.py --config c5      (diagonal M)
    python tools/prof_objective.py --config c5a     (AAFN: set_theta builds the factors, then Z~)
"""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2504_00480_b200 as akm  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    a = ap.parse_args()
    wl = workloads.CONFIGS[a.config]
    X, V = workloads.make_X(wl), workloads.make_V(wl)
    dev = torch.device("cuda:0")
    Xd, Vd = torch.from_numpy(X).to(dev), torch.from_numpy(V).to(dev)
    yd, Zd = Vd[:, 0].contiguous(), Vd[:, 1:].contiguous()
    plan = akm.Plan(0)
    plan.set_points(Xd, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
    aafn = "aafn_kpw" in wl.extra
    if aafn:
        plan.set_preconditioner(wl.extra["aafn_kpw"])
    plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    cg, lz = wl.extra["cg_iters"], wl.extra["lanczos_steps"]

    def step():
        if aafn:
            plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
            plan.objective(yd, Zd, cg, lz)
        else:
            plan.objective_diag(yd, Zd, cg, lz)

    step()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    tot = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = ev.name.split("(")[0].replace("void ", "")[:60]
            tot[k][0] += 1
            tot[k][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    s = sum(v[1] for v in tot.values())
    print(f"{'kernel':62s} {'calls':>6s} {'ms':>9s} {'share':>6s}")
    for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:62s} {c:6d} {t / 1e3:9.3f} {100 * t / s:5.1f}%")
    print(f"total kernel time {s / 1e3:.3f} ms")
    plan.close()


if __name__ == "__main__":
    main()
