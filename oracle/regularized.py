"""Boundary-regularised kernel kappa_R and its fast summation.  TEST INFRASTRUCTURE ONLY.

The paper replaces each windowed kernel by "a smooth or at least continuous periodic function
kappa_R" before truncating its Fourier series (eq. 3.1), and notes "It is possible to
smoothen the inner or outer boundaries [potts2003fast] but in our implementation, the outer
boundary smoothing is set to zero".  This module is that regularisation, written out for
the radial kernels of eqs. 1.1 / 2.2 / 2.3 as a function of r = ||x|| in the scaled coordinates:

    kappa_R(r) = T_I(r)          0 <= r <= eps_I            (inner: removes the Matern cusp at 0)
               = kappa(r)        eps_I < r <= 1/2 - eps_B
               = T_B(r)          1/2 - eps_B < r <= 1/2     (outer: flattens the boundary of the cell)
               = kappa(1/2)      r > 1/2

* T_I is the two-point Taylor interpolant of degree 2p - 1 of the even extension kappa(|r|) on
  [-eps_I, eps_I]: it matches kappa's derivatives of orders 0..p-1 at r = +-eps_I.  (The even
  extension makes T_I an even polynomial, i.e. a polynomial in ||x||^2, smooth in x.)
* T_B is the two-point Taylor interpolant on [1/2 - eps_B, 1/2] matching kappa's derivatives 0..p-1
  at 1/2 - eps_B and the constant kappa(1/2) (derivatives zero) at 1/2.
* eps_I = 0 switches the inner part off, p = 0 switches both off (kappa_R = the plain periodic
  continuation, the paper's implementation).

Two-point Taylor interpolation on [a, b], h = b - a, t = (r - a)/h (Hermite interpolation with p
derivatives at both ends; the explicit basis of the cited fast-summation literature):
    T(r) = sum_{q<p} [ h^q f^(q)(a) B_q(t) + (-h)^q f^(q)(b) B_q(1 - t) ] / q!,
    B_q(t) = t^q (1 - t)^p sum_{s=0}^{p-1-q} C(p-1+s, s) t^s.

Because the points are scaled into the ball of radius 1/4 - eps_B/2, every difference has
r <= 1/2 - eps_B: the outer part never changes a kernel value the product uses.  The inner part
does, for pairs closer than eps_I; the product is restored by the near-field correction
    S_i += sum_{j : ||x~_i - x~_j|| < eps_I} (kappa - T_I)(||x~_i - x~_j||) v_j
computed by brute force here.  The ell-derivative regularises kappa^der the same way (the
interpolation is linear in the function and its nodes do not depend on ell, so eq. 3.5 still
holds for kappa_R).
"""
from __future__ import annotations

import math

import numpy as np

from .fourier import (GAUSSIAN, fourier_coefficients, index_set, kernel_radial, ndft_adjoint, ndft_forward,
                      window_scaling)


def radial_derivatives(family, r, ell, deriv, p):
    """f^(q)(r), q = 0..p-1, of the radial kernel f(r) = P_0(r) e^{alpha r + beta r^2}:
    Gaussian kappa = e^{-r^2/(2 ell^2)} (P_0 = 1), kappa^der = r^2/ell^3 kappa (eq. 2.3);
    Matern kappa = e^{-r/ell} (P_0 = 1), kappa^der = r/ell^2 kappa.
    Derivatives by the recursion P_{q+1} = P_q' + (alpha + 2 beta r) P_q (numpy polynomials)."""
    P = np.polynomial.Polynomial
    if family == GAUSSIAN:
        alpha, beta = 0.0, -1.0 / (2.0 * ell * ell)
        P0 = P([0.0, 0.0, 1.0 / ell**3]) if deriv else P([1.0])
    else:
        alpha, beta = -1.0 / ell, 0.0
        P0 = P([0.0, 1.0 / ell**2]) if deriv else P([1.0])
    lin = P([alpha, 2.0 * beta])
    e = math.exp(alpha * r + beta * r * r)
    out, Pq = [], P0
    for _ in range(p):
        out.append(Pq(r) * e)
        Pq = Pq.deriv() + lin * Pq
    return np.array(out)


def _basis(q, p, t):
    t = np.asarray(t, dtype=np.float64)
    s = sum(math.comb(p - 1 + j, j) * t**j for j in range(p - q))
    return t**q * (1.0 - t) ** p * s


def two_point_taylor(fa, fb, a, b, r):
    """T(r) on [a, b] with T^(q)(a) = fa[q], T^(q)(b) = fb[q], q < p = len(fa)."""
    p = len(fa)
    h = b - a
    t = (np.asarray(r, dtype=np.float64) - a) / h
    out = np.zeros_like(t)
    for q in range(p):
        out += (h**q * fa[q] * _basis(q, p, t) + (-h) ** q * fb[q] * _basis(q, p, 1.0 - t)) / math.factorial(q)
    return out


def kernel_R(family, r, ell, deriv, eps_I, eps_B, p):
    """kappa_R(r) (or its ell-derivative kernel) at radii r >= 0 (module docstring)."""
    r = np.asarray(r, dtype=np.float64)
    out = kernel_radial(family, r * r, ell, deriv)
    if p <= 0:
        return out
    if eps_I > 0:
        d = radial_derivatives(family, eps_I, ell, deriv, p)
        da = d * np.array([(-1.0) ** q for q in range(p)])       # even extension at -eps_I
        m = r <= eps_I
        out[m] = two_point_taylor(da, d, -eps_I, eps_I, r[m])
    if eps_B > 0:
        a = 0.5 - eps_B
        fa = radial_derivatives(family, a, ell, deriv, p)
        fb = np.zeros(p)
        fb[0] = radial_derivatives(family, 0.5, ell, deriv, 1)[0]
        m = (r > a) & (r <= 0.5)
        out[m] = two_point_taylor(fa, fb, a, 0.5, r[m])
        out[r > 0.5] = fb[0]
    return out


def kernel_samples_R(family, ell, N, d, deriv, eps_I, eps_B, p):
    """kappa_R(l/N) for l in I_N^d (eq. 3.2's samples of the regularised kernel)."""
    l = index_set(N) / N
    grids = np.meshgrid(*([l] * d), indexing="ij")
    r = np.sqrt(sum(g * g for g in grids))
    return kernel_R(family, r, ell, deriv, eps_I, eps_B, p)


def near_field(xs, V, family, ell, deriv, eps_I, p, rows=None):
    """sum_{j : ||x_i - x_j|| < eps_I} (kappa - T_I)(||x_i - x_j||) V_j for i in rows (brute force)."""
    xs = np.atleast_2d(xs)
    V = np.asarray(V, dtype=np.float64).reshape(xs.shape[0], -1)
    rows = np.arange(xs.shape[0]) if rows is None else np.asarray(rows)
    out = np.zeros((rows.size, V.shape[1]))
    if eps_I <= 0 or p <= 0:
        return out
    d = radial_derivatives(family, eps_I, ell, deriv, p)
    da = d * np.array([(-1.0) ** q for q in range(p)])
    for k0 in range(0, rows.size, 64):
        blk = rows[k0:k0 + 64]
        rr = np.sqrt(((xs[blk][:, None, :] - xs[None, :, :]) ** 2).sum(axis=2))   # (rows, n) distances
        bi, j = np.nonzero(rr < eps_I)
        r = rr[bi, j]
        w = kernel_radial(family, r * r, ell, deriv) - two_point_taylor(da, d, -eps_I, eps_I, r)
        np.add.at(out, k0 + bi, w[:, None] * V[j])
    return out


def additive_fastsum_R(X, windows, family, theta, V, N, eps_B, eps_I, p, ops=("K", "dell", "dsf"), rows=None,
                       near=True):
    """The truncated-Fourier operator (eq. 3.3, exact sums) of kappa_R per window, plus the near-field
    correction (near=True), assembled like fourier.additive_fastsum (sigma_f^2, sigma_eps^2 V, 1/c_w for
    the ell-derivative, reading R7).  eps_I is in the scaled coordinates of every window."""
    X = np.asarray(X, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64).reshape(X.shape[0], -1)
    sf, ell, se = theta
    Vo = V if rows is None else V[rows]
    S, SD = np.zeros_like(Vo), np.zeros_like(Vo)
    for win in windows:
        Xw = X[:, list(win)]
        _, c, xs = window_scaling(Xw, family, ell, N, eps_B)
        ell_eff = ell / c
        xo = xs if rows is None else xs[rows]
        for deriv in (False, True):
            if deriv and "dell" not in ops:
                continue
            b = fourier_coefficients(kernel_samples_R(family, ell_eff, N, xs.shape[1], deriv, eps_I, eps_B, p))
            h = np.real(ndft_forward(xo, b[None, ...] * ndft_adjoint(xs, V, N)))
            if near:
                h = h + near_field(xs, V, family, ell_eff, deriv, eps_I, p, rows)
            if deriv:
                SD += h / c
            else:
                S += h
    out = {}
    if "K" in ops:
        out["K"] = sf * sf * S + se * se * Vo
    if "dell" in ops:
        out["dell"] = sf * sf * SD
    if "dsf" in ops:
        out["dsf"] = 2.0 * sf * S
    return out
