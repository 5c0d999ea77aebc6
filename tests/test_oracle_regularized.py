"""Pins of the boundary-regularised kernel oracle (oracle/regularized.py).

* two-point Taylor interpolation is exact on polynomials of degree <= 2p - 1 and matches the
  prescribed derivatives at both ends (the defining property of the basis);
* the closed-form radial derivatives agree with central finite differences of the plain kernels of
  oracle/fourier.py (eqs. 1.1, 2.2, 2.3);
* kappa_R is continuous with p - 1 continuous derivatives at eps_I and 1/2 - eps_B, equals kappa
  in between, is flat (kappa(1/2)) beyond 1/2, and p = 0 gives the plain samples (to the rounding of r = sqrt(r^2));
* the regularised fast sum + near-field correction approximates the dense float64 sums far better
  than the plain method where the Matern cusp limits it (3-D, N = 32: 2.4e-3 -> <= 3e-4), and with
  eps_I = 0 it is the plain truncated-Fourier operator (outer smoothing never changes a used value).
"""
import math

import numpy as np
import pytest

from oracle import dense_apply
from oracle import fourier as F
from oracle import regularized as R


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6])
def test_two_point_taylor_exact_on_polynomials(p):
    rng = np.random.default_rng(p)
    c = rng.standard_normal(2 * p)                    # degree 2p - 1
    poly = np.polynomial.Polynomial(c)
    a, b = -0.3, 0.7
    fa = np.array([poly.deriv(q)(a) if q else poly(a) for q in range(p)])
    fb = np.array([poly.deriv(q)(b) if q else poly(b) for q in range(p)])
    r = np.linspace(a, b, 101)
    assert np.max(np.abs(R.two_point_taylor(fa, fb, a, b, r) - poly(r))) <= 1e-12 * np.max(np.abs(c))
    # a random (non-polynomial) end-data set: the interpolant's derivatives match it at both ends
    fa, fb = rng.standard_normal(p), rng.standard_normal(p)
    T = np.polynomial.Polynomial.fit(r, R.two_point_taylor(fa, fb, a, b, r), 2 * p - 1).convert()
    for q in range(p):
        Tq = T.deriv(q) if q else T
        assert Tq(a) == pytest.approx(fa[q], abs=1e-7 * (1 + abs(fa[q])))
        assert Tq(b) == pytest.approx(fb[q], abs=1e-7 * (1 + abs(fb[q])))


@pytest.mark.parametrize("family,deriv", [(0, False), (0, True), (1, False), (1, True)])
def test_radial_derivatives_vs_finite_differences(family, deriv):
    ell, r, h = 0.17, 0.23, 1e-3
    d = R.radial_derivatives(family, r, ell, deriv, 4)
    f = lambda x: F.kernel_radial(family, x * x, ell, deriv)
    assert d[0] == pytest.approx(f(r), rel=1e-14)
    fd1 = (-f(r + 2 * h) + 8 * f(r + h) - 8 * f(r - h) + f(r - 2 * h)) / (12 * h)          # O(h^4) stencils
    fd2 = (-f(r + 2 * h) + 16 * f(r + h) - 30 * f(r) + 16 * f(r - h) - f(r - 2 * h)) / (12 * h * h)
    fd3 = (f(r + 2 * h) - 2 * f(r + h) + 2 * f(r - h) - f(r - 2 * h)) / (2 * h**3)
    assert d[1] == pytest.approx(fd1, rel=1e-8)
    assert d[2] == pytest.approx(fd2, rel=1e-6)
    assert d[3] == pytest.approx(fd3, rel=1e-3)


@pytest.mark.parametrize("family", [0, 1])
def test_kernel_R_structure(family):
    ell, eI, eB, p = 0.2, 0.05, 1.0 / 16, 4
    f = lambda x: F.kernel_radial(family, np.asarray(x) ** 2, ell)
    mid = np.linspace(eI * 1.001, 0.5 - eB, 50)
    np.testing.assert_array_equal(R.kernel_R(family, mid, ell, False, eI, eB, p), f(mid))
    assert np.all(R.kernel_R(family, np.array([0.51, 0.6, 0.8]), ell, False, eI, eB, p) == f(0.5))
    h = 1e-6
    for x0 in (eI, 0.5 - eB, 0.5):                   # C^1 across every junction (p >= 2)
        lo = R.kernel_R(family, np.array([x0 - h, x0 - 2 * h]), ell, False, eI, eB, p)
        hi = R.kernel_R(family, np.array([x0 + h, x0 + 2 * h]), ell, False, eI, eB, p)
        assert abs(lo[0] - hi[0]) <= 1e-5 * max(1.0, abs(lo[0]))
        assert abs((lo[0] - lo[1]) - (hi[1] - hi[0])) <= 1e-9
    # the inner polynomial is even: kappa_R is smooth through r = 0 (no cusp)
    r = np.array([0.0, 1e-3, 2e-3])
    v = R.kernel_R(family, r, ell, False, eI, eB, p)
    assert abs((v[2] - v[1]) - 3 * (v[1] - v[0])) <= 2e-2 * abs(v[1] - v[0])   # v0 + c r^2 (a cusp gives 1:1)
    # p = 0: the plain samples
    for d in (1, 2, 3):
        np.testing.assert_allclose(R.kernel_samples_R(family, ell, 16, d, True, eI, eB, 0),
                                   F.kernel_samples(family, ell, 16, d, True), rtol=4e-15, atol=0)


def test_regularised_fastsum_beats_the_cusp_floor():
    rng = np.random.default_rng(41)
    n = 2000
    X = rng.random((n, 6))
    V = rng.standard_normal((n, 2))
    windows = [(0, 1, 2), (3, 4, 5)]
    th = (0.9, 0.6, 0.15)
    ops = ("K", "dell", "dsf")
    de = dense_apply(X, windows, 1, th, V, ops=ops)
    plain = F.additive_fastsum(X, windows, 1, th, V, 32, 1.0 / 16, ops=ops)
    reg = R.additive_fastsum_R(X, windows, 1, th, V, 32, 1.0 / 16, 1.0 / 16, 4, ops=ops)
    for op in ops:
        e_plain = np.linalg.norm(plain[op] - de[op]) / np.linalg.norm(de[op])
        e_reg = np.linalg.norm(reg[op] - de[op]) / np.linalg.norm(de[op])
        assert e_plain > 1e-3 and e_reg <= 3e-4, (op, e_plain, e_reg)
    # outer smoothing only: no used kernel value changes, so the operator is the plain one up to the
    # truncation of the (smoothed) boundary, far below the method error
    outer = R.additive_fastsum_R(X, windows, 1, th, V, 32, 1.0 / 16, 0.0, 4, ops=("K",))
    assert np.linalg.norm(outer["K"] - plain["K"]) <= 2e-3 * np.linalg.norm(plain["K"])
    # Gaussian: inner smoothing + near field is harmless (no cusp to remove)
    deg = dense_apply(X, windows, 0, (1.0, 0.3, 0.1), V, ops=("K",))
    g = R.additive_fastsum_R(X, windows, 0, (1.0, 0.3, 0.1), V, 32, 1.0 / 16, 1.0 / 32, 4, ops=("K",))
    assert np.linalg.norm(g["K"] - deg["K"]) <= 1e-6 * np.linalg.norm(deg["K"])


def test_near_field_brute_force_small():
    """near_field against explicit double loops on a handful of points."""
    rng = np.random.default_rng(3)
    xs = rng.uniform(-0.05, 0.05, size=(12, 2))
    V = rng.standard_normal((12, 2))
    eI, p, ell = 0.06, 3, 0.1
    got = R.near_field(xs, V, 1, ell, False, eI, p)
    d = R.radial_derivatives(1, eI, ell, False, p)
    da = d * np.array([1.0, -1.0, 1.0])
    want = np.zeros_like(V)
    for i in range(12):
        for j in range(12):
            r = math.dist(xs[i], xs[j])
            if r < eI:
                w = math.exp(-r / ell) - R.two_point_taylor(da, d, -eI, eI, np.array([r]))[0]
                want[i] += w * V[j]
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-14)
