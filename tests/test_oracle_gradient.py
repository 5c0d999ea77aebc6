"""Pins of the gradient oracle (oracle/krylov.py gradient_diag; eq. (div))
against the mathematics, not against itself:

* with the scaled unit vectors z_i = sqrt(n) e_i (so (1/n_z) sum z_i z_i^T = I exactly) and converged
  CG, the estimator IS the exact gradient of Z = 1/2 (y^T Khat^{-1} y + log det Khat + n log 2 pi)
  (eq. 1.2; the log det M terms cancel) -> central finite differences of the dense Z in each of
  sigma_f, ell, sigma_eps;
* with Rademacher probes (||z||^2 = n) the preconditioner terms n dc/c and -(dc/c) ||z||^2 cancel
  exactly, so the result does not depend on dc.
"""
import numpy as np
import pytest

from oracle import dense_apply
from oracle import krylov as KR


def _setup(family, n=30, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.random((n, 5))
    windows = [(0, 1, 2), (3, 4)]
    return X, windows, rng.standard_normal(n)


def _ops(X, windows, family, theta):
    n = X.shape[0]
    K = dense_apply(X, windows, family, theta, np.eye(n), ops=("K",))["K"]

    def dK(B):
        o = dense_apply(X, windows, family, theta, B, ops=("dell", "dsf", "dse"))
        return {"ell": o["dell"], "sf": o["dsf"], "se": o["dse"]}

    return K, dK


@pytest.mark.parametrize("family", [0, 1])
def test_gradient_exact_trace_probes_match_fd_of_dense_objective(family):
    X, windows, y = _setup(family)
    n = X.shape[0]
    theta = (1.2, 0.4, 0.3)
    K, dK = _ops(X, windows, family, theta)
    c = theta[0] ** 2 * len(windows) + theta[2] ** 2
    dc = {"sf": 2 * theta[0] * len(windows), "ell": 0.0, "se": 2 * theta[2]}
    g = KR.gradient_diag(lambda B: K @ B, dK, y, np.sqrt(n) * np.eye(n), c, dc, 200)["grad"]

    def Zd(th):
        Kt = dense_apply(X, windows, family, th, np.eye(n), ops=("K",))["K"]
        return 0.5 * (y @ np.linalg.solve(Kt, y) + np.linalg.slogdet(Kt)[1])

    for j, idx in (("sf", 0), ("ell", 1), ("se", 2)):
        h = 1e-5 * theta[idx]
        tp, tm = list(theta), list(theta)
        tp[idx] += h
        tm[idx] -= h
        fd = (Zd(tuple(tp)) - Zd(tuple(tm))) / (2 * h)
        assert g[j] == pytest.approx(fd, rel=1e-7), j


def test_gradient_rademacher_preconditioner_terms_cancel():
    X, windows, y = _setup(0, n=40, seed=1)
    theta = (0.8, 0.5, 0.4)
    K, dK = _ops(X, windows, 0, theta)
    Z = np.where(np.random.default_rng(2).random((40, 6)) < 0.5, -1.0, 1.0)
    c = theta[0] ** 2 * 2 + theta[2] ** 2
    a = KR.gradient_diag(lambda B: K @ B, dK, y, Z, c, {"sf": 2 * theta[0] * 2, "ell": 0.0, "se": 2 * theta[2]}, 80)
    b = KR.gradient_diag(lambda B: K @ B, dK, y, Z, c, {"sf": 0.0, "ell": 0.0, "se": 0.0}, 80)
    for j in ("sf", "ell", "se"):
        assert a["grad"][j] == pytest.approx(b["grad"][j], rel=1e-13, abs=1e-12)
