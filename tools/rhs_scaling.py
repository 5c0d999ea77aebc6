"""ms per K-hat V product and per RHS column at r = 1, 2, 4, 11 on a BASELINE.json workload:
``python tools/rhs_scaling.py c4``."""
import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import workloads, paper_2504_00480_b200 as akm
wl = workloads.CONFIGS[sys.argv[1]]
dev = torch.device('cuda:0')
X = torch.from_numpy(workloads.make_X(wl)).to(dev)
plan = akm.Plan(0)
plan.set_points(X, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
for r in (1, 2, 4, 11):
    V = torch.randn(X.shape[0], r, dtype=torch.float64, device=dev)
    Y = torch.empty_like(V)
    for _ in range(3): plan.mvm(V, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): plan.mvm(V, Y)
    e1.record(); torch.cuda.synchronize()
    print(sys.argv[1], "r", r, "ms/product", round(e0.elapsed_time(e1) / 20, 4), "per column", round(e0.elapsed_time(e1) / 20 / r, 4))
