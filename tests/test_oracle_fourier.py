"""Pins of the Fourier-side oracle (oracle/fourier.py, oracle/bounds.py) -- SURVEY.md §4 tier 2.

Each test ties the oracle to something other than itself: the paper's printed Fig. 2
coefficients, closed forms (constant / cosine), interpolation at the grid nodes,
quadrature of the window, the paper's error bounds, and the dense oracle."""
import math
import os

import numpy as np
import pytest
from scipy.integrate import quad

import workloads
from oracle import bounds, dense_apply
from oracle import fourier as F

HERE = os.path.dirname(os.path.abspath(__file__))
G, M = 0, 1


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ---------------------------------------------------------------- eq. (3.2)
def test_fig2_printed_coefficients():
    """PAPER.md Fig. 2: 1-D Matern(1/2), ell = 0.3, m = 8."""
    gold = np.loadtxt(os.path.join(HERE, "golden", "fig2_matern_l0.3_m8.txt"))
    b = F.fourier_coefficients(F.kernel_samples(M, 0.3, 8, 1))
    for k, val in gold:
        bk = b[int(k) + 4]
        assert abs(bk.imag) < 1e-16
        assert bk.real == pytest.approx(val, rel=2e-15)
    # evenness b_k = b_{-k} for |k| < N/2
    for k in range(1, 4):
        assert b[4 + k].real == pytest.approx(b[4 - k].real, rel=1e-14)


def test_coefficients_closed_forms():
    for d in (1, 2, 3):
        b = F.fourier_coefficients(np.ones((8,) * d))
        ref = np.zeros((8,) * d)
        ref[(4,) * d] = 1.0
        np.testing.assert_allclose(b, ref, atol=1e-15)
    l = F.index_set(8) / 8
    b = F.fourier_coefficients(np.cos(2 * np.pi * l))
    ref = np.zeros(8)
    ref[4 + 1] = ref[4 - 1] = 0.5
    np.testing.assert_allclose(b, ref, atol=1e-15)


@pytest.mark.parametrize("family,d", [(G, 3), (M, 3), (M, 2), (G, 1)])
def test_truncated_series_interpolates_samples(family, d):
    """kappa_RF(l/N) = kappa(l/N) at every node (Fig. 2 caption: 'interpolating m samples')."""
    N = 8 if d == 3 else 16
    s = F.kernel_samples(family, 0.11, N, d)
    b = F.fourier_coefficients(s)
    nodes = np.stack(np.meshgrid(*([F.index_set(N) / N] * d), indexing="ij"), axis=-1).reshape(-1, d)
    vals = np.real(F.ndft_forward(nodes, b[None, ...]))[:, 0]
    np.testing.assert_allclose(vals, s.reshape(-1), atol=5e-16 * N**d)


@pytest.mark.parametrize("family", [G, M])
def test_eq35_derivative_coefficients(family):
    """eq. (3.5): b_k(kappa_der) = d/d ell b_k(kappa) (central difference)."""
    ell, h = 0.07, 1e-6
    bd = F.fourier_coefficients(F.kernel_samples(family, ell, 16, 3, deriv=True))
    fd = (F.fourier_coefficients(F.kernel_samples(family, ell + h, 16, 3))
          - F.fourier_coefficients(F.kernel_samples(family, ell - h, 16, 3))) / (2 * h)
    assert np.max(np.abs(fd - bd)) <= 1e-7 * np.max(np.abs(bd))


# ---------------------------------------------------------------- §4 bounds
@pytest.mark.parametrize("ell", [0.05, 0.1, 0.2])
@pytest.mark.parametrize("N", [8, 16])
def test_theorems_44_45_dominate_periodized_error(ell, N):
    rng = np.random.default_rng(12)
    r = rng.uniform(-0.5, 0.5, size=(400, 3))
    nodes = np.stack(np.meshgrid(*([F.index_set(N) / N] * 3), indexing="ij"), axis=-1).reshape(-1, 3)
    img = 3 if ell < 0.15 else 5
    for deriv, bound in ((False, bounds.thm44(N, ell)), (True, bounds.thm45(N, ell))):
        s = bounds.periodized(M, nodes, ell, deriv, images=img).reshape((N,) * 3)
        b = F.fourier_coefficients(s)
        approx = np.real(F.ndft_forward(r, b[None, ...]))[:, 0]
        exact = bounds.periodized(M, r, ell, deriv, images=img)
        err = np.max(np.abs(approx - exact))
        assert err <= bound, (err, bound)


def test_lemma42_and_spec_values():
    assert bounds.delta_m(0.05) == pytest.approx(1.098e-2, rel=1e-3)
    assert bounds.thm44(32, 0.1) == pytest.approx(0.2840, rel=1e-3)
    assert bounds.thm45(32, 0.1) == pytest.approx(2.888, rel=1e-3)
    # Lemma 4.2 dominates the periodization gap |kappa - kappa~| on [-1/2,1/2)^3
    rng = np.random.default_rng(1)
    r = rng.uniform(-0.5, 0.5, size=(500, 3))
    for ell in (0.05, 0.1):
        gap = np.max(np.abs(F.kernel_radial(M, (r * r).sum(1), ell) - bounds.periodized(M, r, ell, images=3)))
        assert gap <= bounds.delta_m(ell)


# ---------------------------------------------------------------- App. A window + NFFT
@pytest.mark.parametrize("n_g,m", [(64, 6), (256, 8), (32, 4)])
def test_kb_fourier_transform_matches_quadrature(n_g, m):
    """The I0 closed form is the transform of the untruncated window; truncation moves it by
    O(e^{-beta m}) relative on the frequencies the method uses (|k| <= N/2 = n_g/4)."""
    tol = max(100 * math.exp(-F.kb_beta(2.0) * m), 1e-13)
    for k in (0, 3, n_g // 8, n_g // 4):
        num = quad(lambda x: F.kb_phi(np.array([x]), n_g, m, 2.0)[0] * math.cos(2 * math.pi * k * x),
                   -m / n_g, m / n_g, limit=400, epsabs=0, epsrel=2e-14, points=[0])[0]
        assert F.kb_phi_hat(k, n_g, m, 2.0) == pytest.approx(num, rel=tol)


def test_nfft_forward_within_eqA3_bound_1d():
    rng = np.random.default_rng(8)
    N, sigma = 16, 2.0
    x = rng.uniform(-0.5, 0.5, size=(100, 1))
    fhat = (rng.standard_normal(N) + 1j * rng.standard_normal(N))[None, :]
    exact = F.ndft_forward(x, fhat)
    errs = []
    for s in (2, 4, 6, 8):
        approx = F.nfft_forward(x, fhat, int(sigma * N), s, sigma)
        err = np.max(np.abs(approx - exact))
        assert err <= np.sum(np.abs(fhat)) * bounds.nfft_bound(s, sigma)
        errs.append(err)
    assert all(errs[i + 1] < errs[i] for i in range(len(errs) - 1))


def test_eqA3_bound_two_sided():
    """eq. (A.3) pinned from both sides (VERDICT r1 Weak 1).
    (i) SPEC's printed evaluation at s = 8, sigma = 2: 4 pi (8 + 2.8284) 0.8409 e^{-2 pi 8 0.7071};
    (ii) SPEC's printed ratio s = 4 -> 8 at sigma = 2: e^{-17.77} times the polynomial factor
         (8 + sqrt 8)/(4 + 2);
    (iii) the measured 1-D NFFT error per unit ||b||_1 sits below the bound by at most 100x for s = 2..7
          (above that the float64 floor takes over): a wrong exponent or prefactor power moves the bound by
          far more than that at some s."""
    printed = 4.0 * math.pi * (8.0 + 2.8284) * 0.8409 * math.exp(-2.0 * math.pi * 8.0 * 0.7071)
    assert bounds.nfft_bound(8, 2.0) == pytest.approx(printed, rel=2e-3)
    ratio = bounds.nfft_bound(8, 2.0) / bounds.nfft_bound(4, 2.0)
    assert ratio == pytest.approx((8.0 + 2.8284) / 6.0 * math.exp(-17.77), rel=5e-3)
    rng = np.random.default_rng(8)
    N, sigma = 16, 2.0
    x = rng.uniform(-0.5, 0.5, size=(400, 1))
    fhat = (rng.standard_normal(N) + 1j * rng.standard_normal(N))[None, :]
    exact = F.ndft_forward(x, fhat)
    for s in (2, 3, 4, 5, 6, 7):
        err = np.max(np.abs(F.nfft_forward(x, fhat, int(sigma * N), s, sigma) - exact)) / np.sum(np.abs(fhat))
        b = bounds.nfft_bound(s, sigma)
        assert err <= b <= 100.0 * err, (s, err, b)


def test_nfft_adjoint_is_transpose_of_forward():
    rng = np.random.default_rng(9)
    N, n_g, m = 8, 16, 4
    x = rng.uniform(-0.25, 0.25, size=(30, 2))
    v = rng.standard_normal((30, 1))
    fhat = (rng.standard_normal((1, N, N)) + 1j * rng.standard_normal((1, N, N)))
    lhs = np.vdot(v[:, 0], F.nfft_forward(x, fhat, n_g, m, 2.0)[:, 0])          # <v, A fhat>
    rhs = np.vdot(F.nfft_adjoint(x, v, N, n_g, m, 2.0)[0], fhat[0])              # <A^H v, fhat>
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_nfft_fastsum_matches_ndft_and_improves_with_m():
    rng = np.random.default_rng(10)
    x = rng.uniform(-0.2, 0.2, size=(300, 3))
    V = rng.standard_normal((300, 2))
    b = F.fourier_coefficients(F.kernel_samples(G, 0.07, 16, 3))
    ref = F.trunc_fastsum(x, V, b)
    errs = [_rel(F.nfft_fastsum(x, V, b, 2.0, m), ref) for m in (2, 4, 6)]
    assert errs[2] <= 1e-10
    assert errs[0] > errs[1] > errs[2]


# ---------------------------------------------------------------- scaling + method vs dense
def test_window_scaling_reading():
    rng = np.random.default_rng(13)
    X = rng.standard_normal((500, 3)) * 3 + 1
    for fam, ell in ((G, 0.01), (G, 5.0), (M, 0.7)):
        center, c, xs = F.window_scaling(X, fam, ell, 32, 1 / 16)
        assert np.sqrt((xs**2).sum(1)).max() <= (0.25 - 1 / 32) * (1 + 1e-14)
        i, j = 3, 77
        assert F.kernel_radial(fam, ((X[i] - X[j])**2).sum(), ell) == pytest.approx(
            F.kernel_radial(fam, ((xs[i] - xs[j])**2).sum(), ell / c), rel=1e-13)


@pytest.mark.parametrize("cfg,n,tol", [("c1", 2000, 1e-6), ("c2", 3000, 1e-10), ("c3", 1500, 1e-3)])
def test_truncated_fourier_operator_vs_dense(cfg, n, tol):
    """Method error of eq. (3.3) (exact trigonometric sums, reading R2 scaling) vs the dense oracle."""
    wl = workloads.CONFIGS[cfg]
    X = workloads.make_X(wl, n=n)
    V = workloads.make_V(wl, n=n, r=min(wl.r, 3))
    th = (wl.sigma_f, wl.ell, wl.sigma_eps)
    ops = tuple(o for o in ("K", "dell") if o in wl.ops)
    fs = F.additive_fastsum(X, wl.windows, wl.family, th, V, wl.N, wl.eps_B, method="ndft", ops=ops)
    de = dense_apply(X, wl.windows, wl.family, th, V, ops=ops)
    for op in ops:
        assert _rel(fs[op], de[op]) <= tol, (op, _rel(fs[op], de[op]))
