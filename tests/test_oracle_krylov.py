"""Pins of the Krylov oracle (oracle/krylov.py): CG, Lanczos/SLQ and the eq. (1.4) assembly.

Each test ties the oracle to something other than itself: hand-solvable systems,
direct solves and eigendecompositions of explicit matrices, the identity of eq. (1.3), and the
exact objective eq. (1.2) -- which eq. (1.4) reproduces exactly when the Krylov budgets equal n and
the probes are sqrt(n) e_j (Gauss quadrature with n nodes is exact; Hutchinson over the scaled
identity basis is the trace)."""
import math

import numpy as np
import pytest

import workloads
from oracle import dense_apply
from oracle import krylov as KR


def _spd(n, seed, cond=50.0):
    rng = np.random.default_rng(seed)
    Qm, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.geomspace(1.0, cond, n)
    return (Qm * lam) @ Qm.T, lam


def _logm_quad(A, z):
    lam, U = np.linalg.eigh(A)
    c = U.T @ z
    return float(np.sum(c * c * np.log(lam)))


def test_pcg_spec_examples():
    x, _ = KR.pcg(lambda B: B, np.array([3.0, -1.0, 2.0]), 1)
    np.testing.assert_allclose(x, [3.0, -1.0, 2.0], rtol=0, atol=1e-15)
    A = np.diag([2.0, 1.0])
    x, _ = KR.pcg(lambda B: A @ B, np.array([2.0, 1.0]), 2)
    np.testing.assert_allclose(x, [1.0, 1.0], rtol=1e-14)


def test_pcg_matches_direct_solve_and_preconditioning():
    A, _ = _spd(40, 1, cond=30.0)
    b = np.random.default_rng(2).standard_normal(40)
    x, hist = KR.pcg(lambda B: A @ B, b, 120)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9)
    assert hist[-1] < 1e-9
    # Jacobi preconditioning of a badly scaled diagonal converges in one step
    D = np.diag(np.geomspace(1, 1e6, 40))
    x, _ = KR.pcg(lambda B: D @ B, b, 1, minv_diag=1.0 / np.diag(D))
    np.testing.assert_allclose(x, b / np.diag(D), rtol=1e-12)


def test_lanczos_full_basis_reproduces_spectrum_and_logm_quadform():
    A, lam = _spd(24, 3, cond=100.0)
    z = np.where(np.random.default_rng(4).random(24) < 0.5, -1.0, 1.0)
    al, be = KR.lanczos(lambda B: A @ B, z, 24)
    assert len(al) == 24 and len(be) == 23
    T = np.diag(al) + np.diag(be, 1) + np.diag(be, -1)
    np.testing.assert_allclose(np.linalg.eigvalsh(T), lam, rtol=1e-10)
    # Gauss quadrature with n nodes is exact: z^T logm(A) z
    assert KR.slq_sample(al, be, float(z @ z)) == pytest.approx(_logm_quad(A, z), rel=1e-10)


def test_lanczos_spec_diagonal_example_and_breakdown():
    """diag(1..10) with 10 steps matches the dense log-det quadratic form."""
    A = np.diag(np.arange(1.0, 11.0))
    z = np.ones(10)
    al, be = KR.lanczos(lambda B: A @ B, z, 10)
    assert KR.slq_sample(al, be, 10.0) == pytest.approx(float(np.sum(np.log(np.arange(1.0, 11.0)))), rel=1e-12)
    # invariant subspace of dimension 2 -> breakdown after 2 steps, still exact on that subspace
    A2 = np.diag([1.0, 1.0, 4.0, 4.0, 4.0])
    al, be = KR.lanczos(lambda B: A2 @ B, np.ones(5), 5)
    assert len(al) == 2
    assert KR.slq_sample(al, be, 5.0) == pytest.approx(3 * math.log(4.0), rel=1e-12)


def _dense_khat(X, windows, family, theta):
    n = X.shape[0]
    return dense_apply(X, windows, family, theta, np.eye(n), ops=("K",))["K"]


@pytest.mark.parametrize("family", [0, 1])
def test_objective_equals_exact_eq12_with_full_budgets(family):
    wl = workloads.CONFIGS["c5"]
    n = 36
    X = workloads.make_X(wl, n=n)
    theta = (1.1, 0.4, 0.3)
    K = _dense_khat(X, wl.windows, family, theta)
    y = np.random.default_rng(5).standard_normal(n)
    Zp = math.sqrt(n) * np.eye(n)                        # Hutchinson over the scaled identity = trace
    dM = np.diag(K).copy()
    out = KR.objective_diag(lambda B: K @ B, y, Zp, dM, cg_iters=n, lanczos_steps=n)
    sign, logdet = np.linalg.slogdet(K)
    assert sign > 0
    exact = 0.5 * (y @ np.linalg.solve(K, y) + logdet + n * math.log(2 * math.pi))   # eq. (1.2)
    assert out["quad"] == pytest.approx(float(y @ np.linalg.solve(K, y)), rel=1e-8)
    assert out["logdetM"] + out["slq"] == pytest.approx(logdet, rel=1e-8)            # eq. (1.3)
    assert out["Z"] == pytest.approx(exact, rel=1e-8)


def test_objective_diag_matches_eigen_quadforms_for_rademacher_probes():
    wl = workloads.CONFIGS["c5"]
    n = 60
    X = workloads.make_X(wl, n=n)
    theta = (wl.sigma_f, wl.ell, 0.2)
    K = _dense_khat(X, wl.windows, wl.family, theta)
    rng = np.random.default_rng(6)
    y = rng.standard_normal(n)
    Zp = np.where(rng.random((n, 4)) < 0.5, -1.0, 1.0)
    c = theta[0] ** 2 * len(wl.windows) + theta[2] ** 2        # diag(Khat): kappa(0) = 1 per window
    np.testing.assert_allclose(np.diag(K), c, rtol=1e-14)
    out = KR.objective_diag(lambda B: K @ B, y, Zp, c, cg_iters=n, lanczos_steps=n)
    for i in range(4):
        assert out["samples"][i] == pytest.approx(_logm_quad(K / c, Zp[:, i]), rel=1e-8, abs=1e-8)
    assert out["logdetM"] == pytest.approx(n * math.log(c), rel=1e-15)
