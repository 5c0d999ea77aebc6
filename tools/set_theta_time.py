"""Wall time of akm_set_theta on a 1% ell change (Gaussian windows re-bin), per workload:
``python tools/set_theta_time.py c4 c5``; AKM_SETUP_TIMES=1 prints the stages."""
import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import workloads, paper_2504_00480_b200 as akm
dev = torch.device('cuda:0')
for name in sys.argv[1:]:
    wl = workloads.CONFIGS[name]
    X = workloads.make_X(wl)
    Xd = torch.from_numpy(X).to(dev)
    plan = akm.Plan(0)
    t0 = time.perf_counter(); plan.set_points(Xd, wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B); torch.cuda.synchronize(); t1 = time.perf_counter()
    plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps); torch.cuda.synchronize(); t2 = time.perf_counter()
    ts = []
    for k in range(6):
        ell = wl.ell * (1.0 + 0.01 * (k + 1))
        a = time.perf_counter(); plan.set_theta(wl.sigma_f, ell, wl.sigma_eps); torch.cuda.synchronize(); ts.append((time.perf_counter() - a) * 1e3)
    ts2 = []
    for k in range(4):
        a = time.perf_counter(); plan.set_theta(wl.sigma_f * (1 + 0.01 * k), wl.ell, wl.sigma_eps); torch.cuda.synchronize(); ts2.append((time.perf_counter() - a) * 1e3)
    print(name, f"set_points {1e3*(t1-t0):.2f} ms, first set_theta {1e3*(t2-t1):.2f} ms, ell-change {np.median(ts):.2f} ms {np.round(ts,2)}, sigma_f-change {np.median(ts2):.2f} ms")
    plan.close()
