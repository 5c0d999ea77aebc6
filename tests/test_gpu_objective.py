"""GPU parity of the config-5 driver (akm_objective_diag, §8(a) S8) against the Krylov oracle
(oracle/krylov.py) driven by the float64 dense products (oracle/dense.c).

Gates:
  * SLQ samples (full reorthogonalisation) <= 1e-8 relative: MVM perturbations of ~1e-13 move them
    by ~1e-11;
  * CG term y^T x: <= 1e-8 where 50 iterations converge (theta with a larger noise level); at
    BASELINE.json's theta 50 unconverged iterations amplify 1e-13 product noise to ~5e-4, so <= 1e-2;
  * log det M and n log 2 pi are closed forms (exact).
"""
import math

import numpy as np
import pytest

import workloads
from oracle import dense_apply
from oracle import krylov as KR

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def akm():
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_2504_00480_b200 as mod
    return mod


def _inputs(n, n_z, seed=0):
    wl = workloads.CONFIGS["c5"]
    X = workloads.make_X(wl, n=n)
    V = workloads.make_V(wl, n=n, r=1 + n_z, seed=2005 + seed)
    return wl, X, np.ascontiguousarray(V[:, 0]), np.ascontiguousarray(V[:, 1:])


def _gpu(akm, wl, X, theta, y, Z, cg, L, host=False, deterministic=False):
    plan = akm.Plan(0)
    dev = torch.device("cuda:0")
    if deterministic:
        plan.set_deterministic(True)
    plan.set_points(torch.from_numpy(X).to(dev), wl.windows, wl.family, wl.N, wl.sigma_over, wl.m, wl.eps_B)
    plan.set_theta(*theta)
    if host:
        out = plan.objective_diag(y, Z, cg, L)
    else:
        out = plan.objective_diag(torch.from_numpy(y).to(dev), torch.from_numpy(Z).to(dev), cg, L)
    plan.close()
    return out


def _oracle(wl, X, theta, y, Z, cg, L):
    def apply_K(B):
        return dense_apply(X, wl.windows, wl.family, theta, np.ascontiguousarray(B), ops=("K",))["K"]
    c = theta[0] ** 2 * len(wl.windows) + theta[2] ** 2
    return KR.objective_diag(apply_K, y, Z, c, cg, L)


def test_objective_converged_theta_matches_oracle(akm):
    wl, X, y, Z = _inputs(3000, 10)
    theta = (0.5, 0.5, 1.0)                             # CG reaches ~3e-13 in 50 iterations here
    g = _gpu(akm, wl, X, theta, y, Z, 50, 30)
    o = _oracle(wl, X, theta, y, Z, 50, 30)
    assert o["cg_hist"][-1] < 1e-9                      # converged: the CG term is well determined
    assert g["products"] == 50
    assert g["steps"] == o["steps"] == [30] * 10
    assert g["quad"] == pytest.approx(o["quad"], rel=1e-8)
    for a, b in zip(g["samples"], o["samples"]):
        assert a == pytest.approx(b, rel=1e-8)
    assert g["logdetM"] == pytest.approx(3000 * math.log(3 * 0.25 + 1.0), rel=1e-14)
    assert g["Z"] == pytest.approx(o["Z"], rel=1e-8)
    # residual histories agree until the first near-zero-curvature spike (iteration ~8 here, where
    # CG's recursive residual amplifies 1e-13 product differences), and both end converged
    np.testing.assert_allclose(g["cg_hist"][:6], o["cg_hist"][:6], rtol=1e-5)
    assert g["cg_hist"][-1] < 1e-9


def test_objective_baseline_theta_matches_oracle(akm):
    wl, X, y, Z = _inputs(3000, 10, seed=1)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    g = _gpu(akm, wl, X, theta, y, Z, 50, 30)
    o = _oracle(wl, X, theta, y, Z, 50, 30)
    for a, b in zip(g["samples"], o["samples"]):
        assert a == pytest.approx(b, rel=1e-8)
    assert g["quad"] == pytest.approx(o["quad"], rel=1e-2)   # unconverged CG: see module docstring
    assert g["slq"] == pytest.approx(o["slq"], rel=1e-8)


def test_objective_breakdown_and_edge_budgets(akm):
    # n = 12 points, 20 Lanczos steps: Krylov space exhausted -> breakdown before step 13
    wl, X, y, Z = _inputs(12, 3, seed=2)
    theta = (1.0, 0.3, 0.5)
    g = _gpu(akm, wl, X, theta, y, Z, 12, 20)
    o = _oracle(wl, X, theta, y, Z, 12, 20)
    assert all(s <= 12 for s in g["steps"]) and g["steps"] == o["steps"]
    for a, b in zip(g["samples"], o["samples"]):
        assert a == pytest.approx(b, rel=1e-8, abs=1e-10)
    # only CG / only SLQ
    g0 = _gpu(akm, wl, X, theta, y, Z, 0, 5)
    assert g0["quad"] == 0.0 and g0["products"] == 5
    g1 = _gpu(akm, wl, X, theta, y, Z, 6, 0)
    assert g1["slq"] == 0.0 and g1["steps"] == [0, 0, 0]


def test_objective_host_inputs_match_device(akm):
    """Host and device inputs run the same kernels; in deterministic mode (integer-limb spreading,
    akm_set_deterministic) the two evaluations agree bit for bit.  (With float atomics the spreading
    sums in arrival order: 20 CG steps amplify those last-bit differences to ~3e-11 of Z.)"""
    wl, X, y, Z = _inputs(2000, 4, seed=3)
    theta = (1.0, 0.5, 0.2)
    a = _gpu(akm, wl, X, theta, y, Z, 20, 10, deterministic=True)
    b = _gpu(akm, wl, X, theta, y, Z, 20, 10, host=True, deterministic=True)
    assert a["Z"] == b["Z"] and a["samples"] == b["samples"]
    c = _gpu(akm, wl, X, theta, y, Z, 20, 10)
    assert c["Z"] == pytest.approx(a["Z"], rel=1e-9)


def test_objective_full_size_c5_invariants(akm):
    """BASELINE.json c5 at full size: 50 block products at r = 11, closed-form terms, sane SLQ."""
    wl = workloads.CONFIGS["c5"]
    X = workloads.make_X(wl)
    V = workloads.make_V(wl)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    g = _gpu(akm, wl, X, theta, np.ascontiguousarray(V[:, 0]), np.ascontiguousarray(V[:, 1:]), 50, 30)
    n = wl.n
    c = 3.0 + wl.sigma_eps ** 2
    assert g["products"] == 50 and g["steps"] == [30] * 10
    assert g["logdetM"] == pytest.approx(n * math.log(c), rel=1e-14)
    assert g["n_log_2pi"] == pytest.approx(n * math.log(2 * math.pi), rel=1e-14)
    # log of the eigenvalues of M^{-1} Khat lies in [log(sigma_eps^2 / c), log(lambda_max / c)] and
    # lambda_max <= n * sigma_f^2 P + sigma_eps^2 (Gershgorin); SLQ samples are n x a weighted mean
    lo, hi = n * math.log(wl.sigma_eps ** 2 / c), n * math.log((n * 3.0 + wl.sigma_eps ** 2) / c)
    assert all(lo <= s <= hi for s in g["samples"])
    assert np.std(g["samples"]) <= 0.05 * abs(np.mean(g["samples"]))   # Hutchinson spread is small here
    # 50 CG iterations do not converge at this theta (cond ~1e7): the residual is only finite
    assert 0.0 < g["cg_relres"] < 1e3 and math.isfinite(g["Z"])


def test_objective_max_probes_matches_oracle(akm):
    """n_z = AKM_MAX_PROBES (R = 32 columns per block): the widest reorthogonalisation shapes."""
    assert akm.AKM_MAX_PROBES == 31
    wl, X, y, Z = _inputs(1500, 31, seed=4)
    theta = (0.5, 0.5, 1.0)
    g = _gpu(akm, wl, X, theta, y, Z, 12, 12)
    o = _oracle(wl, X, theta, y, Z, 12, 12)
    assert g["steps"] == o["steps"] == [12] * 31
    for a, b in zip(g["samples"], o["samples"]):
        assert a == pytest.approx(b, rel=1e-8)
    assert g["quad"] == pytest.approx(o["quad"], rel=1e-6)
