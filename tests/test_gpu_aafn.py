"""GPU parity of the AAFN preconditioner (akm_set_preconditioner / akm_precond_apply /
akm_objective) against oracle/aafn.py.

* landmarks (FPS per window, merged): integer work, bit-exact;
* U^{-1} T, U^{-T} T and log det M (diagonal FSAI, fill = 1) within 1e-10 of the float64 oracle;
* the AAFN objective (CG + SLQ on S_op = U^{-1} K^ U^{-T}) against the oracle driver with the dense
  K^ (the GPU's product is the NFFT one, ~1e-12 away): every term within 1e-8;
* c5 at full size (n = 5e5, BASELINE.json configs[4]): 50 AAFN-PCG iterations reach a true relative
  residual <= 1e-3, where the diagonal preconditioner diverges (VERDICT r1 Missing 1).
"""
import numpy as np
import pytest

import workloads
from oracle import aafn as A

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def akm():
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_2504_00480_b200 as mod
    return mod


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def _plan(akm, X, wl, kpw, theta=None):
    dev = torch.device("cuda:0")
    plan = akm.Plan(0)
    plan.set_points(torch.from_numpy(np.ascontiguousarray(X)).to(dev), wl.windows, wl.family, wl.N, wl.sigma_over,
                    wl.m, wl.eps_B)
    plan.set_preconditioner(kpw)
    plan.set_theta(*(theta or (wl.sigma_f, wl.ell, wl.sigma_eps)))
    return plan


@pytest.mark.parametrize("name,n,kpw", [("c5", 5000, 25), ("c3", 4000, 40), ("c1", 2000, 60)])
def test_landmarks_bit_exact(akm, name, n, kpw):
    wl = workloads.CONFIGS[name]
    X = workloads.make_X(wl, n=n)
    plan = _plan(akm, X, wl, kpw)
    dev = torch.device("cuda:0")
    T = torch.zeros((n, 1), dtype=torch.float64, device=dev)
    out = torch.empty_like(T)
    _, lm = plan.precond_apply(T, out)
    plan.close()
    want = A.landmarks(X, wl.windows, kpw)
    np.testing.assert_array_equal(lm, want)


def test_factor_and_applications(akm):
    wl = workloads.CONFIGS["c5"]
    n, r, kpw = 3000, 3, 30
    X = workloads.make_X(wl, n=n)
    th = (wl.sigma_f, wl.ell, wl.sigma_eps)
    plan = _plan(akm, X, wl, kpw)
    pre = A.Aafn(X, wl.windows, wl.family, th, kpw, 1)
    dev = torch.device("cuda:0")
    T = np.random.default_rng(1).standard_normal((n, r))
    Td = torch.from_numpy(T).to(dev)
    for transpose in (False, True):
        out = torch.empty_like(Td)
        logdet, lm = plan.precond_apply(Td, out, transpose=transpose)
        want = pre.U_invT(T) if transpose else pre.U_inv(T)
        assert rel(out.cpu().numpy(), want) <= 1e-10, (transpose, rel(out.cpu().numpy(), want))
        assert logdet == pytest.approx(pre.logdet, rel=1e-10)
    np.testing.assert_array_equal(lm, pre.lm)
    plan.close()


def test_objective_vs_oracle(akm):
    """100 landmarks per window: 50 CG iterations converge to ~4e-8 (with 40 per window they stop at
    ~2e-3, where y^T x still moves by 1e-5 under the 1e-12 difference between the NFFT and dense products)."""
    wl = workloads.CONFIGS["c5"]
    n, n_z, kpw = 3000, 4, 100
    X = workloads.make_X(wl, n=n)
    V = workloads.make_V(wl, n=n, r=1 + n_z)
    th = (wl.sigma_f, wl.ell, wl.sigma_eps)
    plan = _plan(akm, X, wl, kpw)
    dev = torch.device("cuda:0")
    y = torch.from_numpy(np.ascontiguousarray(V[:, 0])).to(dev)
    Z = torch.from_numpy(np.ascontiguousarray(V[:, 1:])).to(dev)
    got = plan.objective(y, Z, 50, 20)
    plan.close()
    K = A.khat_dense(X, wl.windows, wl.family, th)
    pre = A.Aafn(X, wl.windows, wl.family, th, kpw, 1)
    want = A.objective_aafn(lambda B: K @ B, V[:, 0], V[:, 1:], pre, 50, 20)
    assert got["landmarks"] == pre.lm.size
    assert got["logdetM"] == pytest.approx(want["logdetM"], rel=1e-10)
    assert got["quad"] == pytest.approx(want["quad"], rel=1e-8)
    assert got["slq"] == pytest.approx(want["slq"], rel=1e-8)
    assert got["Z"] == pytest.approx(want["Z"], rel=1e-8)
    assert got["cg_relres_true"] <= 1e-6 and want["cg_relres_true"] <= 1e-6


def test_c5_full_size_cg_converges(akm):
    """BASELINE.json configs[4] (n = 5e5, three 3-D Gaussian windows, theta = (1, 0.5, 0.05), 50 CG
    iterations, 30 Lanczos steps, 10 probes): with AAFN (800 landmarks per window, 2396 after merging)
    the 50-iteration CG solution has a true relative residual <= 1e-3; with M = diag(K^) it does not
    converge.  (At n = 5e5 the Nystrom part needs many landmarks: 100 per window stop at ~0.17.)"""
    wl = workloads.CONFIGS["c5"]
    X = workloads.make_X(wl)
    V = workloads.make_V(wl)
    dev = torch.device("cuda:0")
    y = torch.from_numpy(np.ascontiguousarray(V[:, 0])).to(dev)
    Z = torch.from_numpy(np.ascontiguousarray(V[:, 1:])).to(dev)
    plan = _plan(akm, X, wl, 800)
    got = plan.objective(y, Z, 50, 30)
    diag = plan.objective_diag(y, Z, 50, 30)
    plan.close()
    assert got["cg_relres_true"] <= 1e-3, got["cg_relres_true"]
    assert diag["cg_relres_true"] > 1e-1
    assert np.isfinite(got["Z"]) and got["landmarks"] > 2000
    # both estimate the same log det K^ = log det M + tr logm(M^{-1} K^) (eq. 1.3): the AAFN split is
    # far more accurate, so the two agree only to the diagonal estimator's own SLQ spread
    assert got["logdetM"] + got["slq"] == pytest.approx(diag["logdetM"] + diag["slq"], rel=2e-2)


def test_gradient_aafn_vs_oracle(akm):
    """akm_gradient with AAFN (plain Hutchinson form with AAFN-PCG solves) against oracle/aafn.py
    gradient_aafn on the dense K^ (theta where 50 iterations converge: 1e-8), and against the diagonal-M
    estimator there (the control variates cancel for Rademacher probes once the solves converge)."""
    from oracle import dense_apply
    wl = workloads.CONFIGS["c5"]
    n, n_z, kpw = 3000, 4, 100
    X = workloads.make_X(wl, n=n)
    V = workloads.make_V(wl, n=n, r=1 + n_z)
    th = (0.5, 0.5, 1.0)
    plan = _plan(akm, X, wl, kpw, th)
    dev = torch.device("cuda:0")
    y = torch.from_numpy(np.ascontiguousarray(V[:, 0])).to(dev)
    Z = torch.from_numpy(np.ascontiguousarray(V[:, 1:])).to(dev)
    got = plan.gradient(y, Z, 50)["grad"]
    diag = plan.gradient_diag(y, Z, 50)["grad"]
    plan.close()
    K = A.khat_dense(X, wl.windows, wl.family, th)

    def dK(B):
        o = dense_apply(X, wl.windows, wl.family, th, np.ascontiguousarray(B), ops=("dell", "dsf", "dse"))
        return {"ell": o["dell"], "sf": o["dsf"], "se": o["dse"]}

    pre = A.Aafn(X, wl.windows, wl.family, th, kpw, 1)
    want = A.gradient_aafn(lambda B: K @ B, dK, V[:, 0], V[:, 1:], pre, 50)["grad"]
    for j in ("sf", "ell", "se"):
        assert got[j] == pytest.approx(want[j], rel=1e-8, abs=1e-8 * abs(want["se"])), j
        assert got[j] == pytest.approx(diag[j], rel=1e-7, abs=1e-7 * abs(want["se"])), j


def test_aafn_edge_cases(akm):
    """Every point a landmark (k_per_window >= n): M = K^, so S_op = I and one CG step solves the
    system; n = 1; switching back to the diagonal preconditioner; argument errors."""
    wl = workloads.CONFIGS["c2"]
    dev = torch.device("cuda:0")
    X = workloads.make_X(wl, n=60)
    V = workloads.make_V(wl, n=60, r=3)
    th = (wl.sigma_f, wl.ell, wl.sigma_eps)
    plan = _plan(akm, X, wl, 100)                 # 100 per window >= n = 60: all points are landmarks
    y = torch.from_numpy(np.ascontiguousarray(V[:, 0])).to(dev)
    Z = torch.from_numpy(np.ascontiguousarray(V[:, 1:])).to(dev)
    o = plan.objective(y, Z, 3, 3)
    assert o["landmarks"] == 60
    K = A.khat_dense(X, wl.windows, wl.family, th)
    assert o["logdetM"] == pytest.approx(np.linalg.slogdet(K)[1], rel=1e-10)
    assert abs(o["slq"]) <= 1e-7 * 60                      # logm(M^{-1} K^) = 0 up to the NFFT product's error
    assert o["cg_relres_true"] <= 1e-8
    plan.set_preconditioner(0)                            # back to M = diag K^
    d = plan.objective(y, Z, 3, 3)
    assert d["landmarks"] == 0
    assert d["logdetM"] == pytest.approx(60 * np.log(th[0] ** 2 * 3 + th[2] ** 2), rel=1e-14)
    with pytest.raises(akm.AkmError):
        plan.set_preconditioner(-1)
    plan.close()
    # n = 1: M = [sigma_f^2 P + sigma_eps^2]
    X1 = np.array([[0.2, 0.5, 0.9]])
    p1 = akm.Plan(0)
    p1.set_points(torch.from_numpy(X1).to(dev), [(0, 1), (2,)], 0)
    p1.set_preconditioner(5)
    p1.set_theta(1.3, 0.4, 0.5)
    T = torch.ones((1, 1), dtype=torch.float64, device=dev)
    out = torch.empty_like(T)
    logdet, lm = p1.precond_apply(T, out)
    assert list(lm) == [0]
    assert logdet == pytest.approx(np.log(1.3**2 * 2 + 0.25), rel=1e-14)
    assert out.item() == pytest.approx(1.0 / np.sqrt(1.3**2 * 2 + 0.25), rel=1e-14)
    p1.close()
