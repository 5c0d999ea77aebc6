"""Cost of deterministic spreading (akm_set_deterministic): ms per product with float64 atomics vs
integer limbs, on a BASELINE.json workload (``python tools/det_cost.py c4``)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import workloads, paper_2504_00480_b200 as akm

for name in sys.argv[1:] or ["c4"]:
    wl = workloads.CONFIGS[name]
    dev = torch.device('cuda:0')
    X = torch.from_numpy(workloads.make_X(wl)).to(dev)
    V = torch.from_numpy(np.ascontiguousarray(workloads.make_V(wl))).to(dev)
    outs = {op: torch.empty_like(V) for op in wl.ops}
    for det in (False, True):
        plan = akm.Plan(0)
        plan.set_points(X, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
        plan.set_deterministic(det)
        plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
        for _ in range(3):
            plan.mvm_multi(V, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            plan.mvm_multi(V, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))
        e1.record()
        torch.cuda.synchronize()
        print(name, "deterministic" if det else "float64 atomics", round(e0.elapsed_time(e1) / 10, 4), "ms / product")
        plan.close()
