"""Pins of the cross-product oracle (oracle/cross.py) against things other than
itself: the C dense oracle (pinned in test_oracle_dense.py) on the union with zero-padded V, the
square case K(X, X) V = Khat V - sigma_eps^2 V, brute-force loops, and the transposition identity
U^T (K_ts V) = V^T (K_st U)."""
import math

import numpy as np
import pytest

import workloads
from oracle import dense_apply
from oracle.cross import dense_cross


def _pts(n, p, seed):
    return np.random.default_rng(seed).random((n, p))


@pytest.mark.parametrize("family", [0, 1])
def test_cross_equals_union_product_rows(family):
    ns, nt, p = 150, 40, 5
    X = _pts(ns + nt, p, 1)
    V = np.random.default_rng(2).standard_normal((ns, 3))
    windows = [(0, 1, 2), (3, 4)]
    theta = (1.3, 0.4, 0.2)
    Vu = np.vstack([V, np.zeros((nt, 3))])
    union = dense_apply(X, windows, family, theta, Vu, ops=("K",))["K"]
    got = dense_cross(X[:ns], X[ns:], windows, family, theta, V)
    np.testing.assert_allclose(got, union[ns:], rtol=1e-12, atol=1e-12)


def test_cross_square_case_is_khat_without_noise():
    X = _pts(120, 3, 3)
    V = np.random.default_rng(4).standard_normal((120, 2))
    theta = (0.7, 0.25, 0.3)
    K = dense_apply(X, [(0, 1, 2)], 0, theta, V, ops=("K",))["K"]
    np.testing.assert_allclose(dense_cross(X, X, [(0, 1, 2)], 0, theta, V), K - theta[2] ** 2 * V, rtol=1e-12,
                               atol=1e-12)


@pytest.mark.parametrize("family", [0, 1])
def test_cross_brute_force_loops(family):
    Xs, Xt = _pts(7, 4, 5), _pts(5, 4, 6)
    V = np.random.default_rng(7).standard_normal((7, 2))
    windows = [(0, 2), (1, 3)]
    sf, ell, se = 1.1, 0.6, 0.5
    want = np.zeros((5, 2))
    for i in range(5):
        for j in range(7):
            for w in windows:
                rr = math.sqrt(sum((Xt[i, f] - Xs[j, f]) ** 2 for f in w))
                k = math.exp(-rr * rr / (2 * ell * ell)) if family == 0 else math.exp(-rr / ell)
                for c in range(2):
                    want[i, c] += sf * sf * k * V[j, c]
    np.testing.assert_allclose(dense_cross(Xs, Xt, windows, family, (sf, ell, se), V), want, rtol=1e-13, atol=1e-14)


def test_cross_transposition_identity():
    Xs, Xt = _pts(60, 3, 8), _pts(45, 3, 9)
    V = np.random.default_rng(10).standard_normal((60, 2))
    U = np.random.default_rng(11).standard_normal((45, 2))
    theta = (1.0, 0.3, 0.1)
    lhs = U.T @ dense_cross(Xs, Xt, [(0, 1, 2)], 1, theta, V)
    rhs = (V.T @ dense_cross(Xt, Xs, [(0, 1, 2)], 1, theta, U)).T
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12)


def test_cross_workload_x4_is_declared():
    wl = workloads.CONFIGS["x4"]
    assert wl.extra["n_src"] < wl.n and wl.units == (wl.n - wl.extra["n_src"]) * wl.r * len(wl.windows)
