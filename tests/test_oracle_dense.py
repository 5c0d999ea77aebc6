"""Pins of the float64 dense oracle (oracle/dense.c) against closed forms, invariants and
brute force -- SURVEY.md §4 tier 1.  CPU only."""
import math

import numpy as np
import pytest
from scipy.spatial.distance import cdist

from oracle import dense_apply, kernel_value

G, M = 0, 1


def _full_matrix(X, windows, family, theta):
    """K-hat assembled column by column from the oracle (K-hat e_j = column j)."""
    n = X.shape[0]
    return dense_apply(X, windows, family, theta, np.eye(n), ops=("K",))["K"]


# ---------------------------------------------------------------- kernel values
def test_kernel_worked_values():
    assert kernel_value(M, [0.3, 0.4], 0.5) == pytest.approx(math.exp(-1.0), rel=1e-15)       # ||r|| = ell
    assert kernel_value(G, [0.6, 0.8], 1.0) == pytest.approx(math.exp(-0.5), rel=1e-15)       # ||r|| = ell = 1
    assert kernel_value(M, [0.5, 0.0, 0.0], 0.5, deriv=True) == pytest.approx(2 * math.exp(-1.0), rel=1e-15)
    for fam in (G, M):
        assert kernel_value(fam, [0.0, 0.0, 0.0], 0.7) == 1.0
        assert kernel_value(fam, [0.0, 0.0, 0.0], 0.7, deriv=True) == 0.0


@pytest.mark.parametrize("family", [G, M])
def test_kernel_derivative_matches_central_difference(family):
    rng = np.random.default_rng(5)
    for _ in range(200):
        r = rng.uniform(-1, 1, size=rng.integers(1, 4))
        ell = rng.uniform(0.1, 2.0)
        h = 1e-5 * ell
        fd = (kernel_value(family, r, ell + h) - kernel_value(family, r, ell - h)) / (2 * h)
        an = kernel_value(family, r, ell, deriv=True)
        assert abs(fd - an) <= 1e-7 * max(1.0, abs(an))


# ---------------------------------------------------------------- operator pins
def test_scalar_case():
    X = np.array([[0.3, 0.1, 0.9, 0.5]])
    wins = [(0, 1), (2,), (3,)]
    for fam in (G, M):
        out = dense_apply(X, wins, fam, (1.3, 0.4, 0.2), np.array([[2.0]]))
        assert out["K"][0, 0] == pytest.approx((1.3**2 * 3 + 0.2**2) * 2.0, rel=1e-15)
        assert out["dell"][0, 0] == 0.0
        assert out["dsf"][0, 0] == pytest.approx(2 * 1.3 * 3 * 2.0, rel=1e-15)
        assert out["dse"][0, 0] == pytest.approx(2 * 0.2 * 2.0, rel=1e-15)


@pytest.mark.parametrize("family", [G, M])
def test_brute_force_cdist(family):
    """Tiny n: independent assembly with scipy's cdist (library routine) vs the oracle's product."""
    rng = np.random.default_rng(11)
    X = rng.random((40, 7))
    wins = [(0, 1, 2), (3, 4), (6,)]
    sf, ell, se = 0.8, 0.35, 0.15
    V = rng.standard_normal((40, 3))
    K = np.zeros((40, 40))
    Kd = np.zeros((40, 40))
    for w in wins:
        D = cdist(X[:, w], X[:, w])  # Euclidean distances
        if family == G:
            k = np.exp(-D**2 / (2 * ell**2))
            Kd += D**2 / ell**3 * k
        else:
            k = np.exp(-D / ell)
            Kd += D / ell**2 * k
        K += k
    out = dense_apply(X, wins, family, (sf, ell, se), V)
    np.testing.assert_allclose(out["K"], sf**2 * K @ V + se**2 * V, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(out["dell"], sf**2 * Kd @ V, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(out["dsf"], 2 * sf * K @ V, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(out["dse"], 2 * se * V, rtol=0, atol=0)


@pytest.mark.parametrize("family", [G, M])
def test_symmetry_columns_and_positive_definite(family):
    rng = np.random.default_rng(2)
    X = rng.random((50, 6))
    wins = [(0, 1, 2), (3, 4, 5)]
    theta = (1.0, 0.3, 0.1)
    Kh = _full_matrix(X, wins, family, theta)
    assert np.max(np.abs(Kh - Kh.T)) <= 1e-15
    np.testing.assert_allclose(np.diag(Kh), 1.0 * 2 + 0.01, rtol=1e-15)
    ev = np.linalg.eigvalsh(Kh)
    assert ev.min() >= 0.01 * (1 - 1e-10)
    u, v = rng.standard_normal(50), rng.standard_normal(50)
    Ku = dense_apply(X, wins, family, theta, u, ops=("K",))["K"][:, 0]
    Kv = dense_apply(X, wins, family, theta, v, ops=("K",))["K"][:, 0]
    assert abs(v @ Ku - u @ Kv) <= 1e-13 * abs(v @ Ku) + 1e-13


def test_gaussian_is_product_of_1d_factors():
    """exp(-||r||^2/2l^2) over window {a,b,c} = elementwise product of the 1-D window matrices."""
    rng = np.random.default_rng(3)
    X = rng.random((30, 3))
    theta = (1.0, 0.25, 0.0)
    K3 = _full_matrix(X, [(0, 1, 2)], G, theta)
    K1 = [_full_matrix(X, [(t,)], G, theta) for t in range(3)]
    np.testing.assert_allclose(K3, K1[0] * K1[1] * K1[2], rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("family", [G, M])
def test_additivity_over_windows(family):
    rng = np.random.default_rng(4)
    X = rng.random((60, 6))
    V = rng.standard_normal((60, 2))
    A, B = [(0, 1, 2)], [(3,), (4, 5)]
    th = (1.1, 0.4, 0.0)
    both = dense_apply(X, A + B, family, th, V)
    a = dense_apply(X, A, family, th, V)
    b = dense_apply(X, B, family, th, V)
    for op in ("K", "dell", "dsf"):
        np.testing.assert_allclose(both[op], a[op] + b[op], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("family", [G, M])
def test_derivatives_match_central_differences(family):
    rng = np.random.default_rng(6)
    X = rng.random((80, 5))
    V = rng.standard_normal((80, 2))
    wins = [(0, 1, 2), (3, 4)]
    sf, ell, se = 0.9, 0.3, 0.2
    base = dense_apply(X, wins, family, (sf, ell, se), V)
    h = 1e-5
    for k, op in ((1, "dell"), (0, "dsf"), (2, "dse")):
        tp = [sf, ell, se]
        tm = [sf, ell, se]
        tp[k] += h * tp[k]
        tm[k] -= h * tm[k]
        fd = (dense_apply(X, wins, family, tp, V, ops=("K",))["K"] - dense_apply(X, wins, family, tm, V, ops=("K",))["K"]) \
            / (tp[k] - tm[k])
        assert np.linalg.norm(fd - base[op]) <= 1e-7 * np.linalg.norm(base[op])


def test_row_subset_matches_full():
    rng = np.random.default_rng(7)
    X = rng.random((100, 3))
    V = rng.standard_normal((100, 4))
    rows = np.array([0, 17, 50, 99], dtype=np.int64)
    full = dense_apply(X, [(0, 1, 2)], M, (1, 0.5, 0.1), V)
    sub = dense_apply(X, [(0, 1, 2)], M, (1, 0.5, 0.1), V, rows=rows)
    for op in full:
        np.testing.assert_array_equal(sub[op], full[op][rows])
