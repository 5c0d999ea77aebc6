"""Fourier-side oracle (numpy, float64/complex128).  TEST INFRASTRUCTURE ONLY.

Written step by step from PAPER.md (P:L = line L):

* ``kernel_samples`` / ``fourier_coefficients``: eq. (3.1)-(3.2), P:144-153 --
  b_k = m^{-d} sum_{l in I_m} kappa_R(l/m) e^{-2 pi i l.k/m}, with kappa_R the plain
  periodic continuation sampled on [-1/2,1/2)^d (outer smoothing zero).
  (Paper's bandwidth m is called N here; SURVEY.md §0 crosswalk.)
* ``trunc_fastsum``: eq. (3.3), P:204-208 -- h(x_i) = Re sum_{k in I_N} b_k a_k e^{2 pi i k.x_i},
  a_k = sum_j v_j e^{-2 pi i k.x_j}; the real part per DESIGN.md reading R5 (Fig. 2).
* ``kb_phi`` / ``kb_phi_hat``: App. A Kaiser-Bessel window, P:1238-1249 (truncated);
  its Fourier transform c_k(phi) = I0(m sqrt(beta^2 - (2 pi k / n_g)^2)) / n_g is reading R4
  ("known explicitly in terms of the modified zero-order Bessel function"), pinned
  against quadrature in tests/test_oracle_fourier.py.
* ``nfft_adjoint`` / ``nfft_forward`` / ``nfft_fastsum``: App. A workflow, P:1219-1233 --
  step 1 b~_k = b_k / c_k(phi) on I_N and 0 elsewhere in I_{sigma N}; step 2 g = FFT(b~);
  step 3 sum of translates sum_l g_l phi~(x - l/(sigma N)); the adjoint is its transpose.
  The fast summation applies the adjoint for the inner sums and the forward NFFT for the
  outer sums.
* ``window_scaling``: scaling of each window's points into the ball of radius
  1/4 - eps_B/2 inside [-1/4,1/4)^d (BASELINE.json c1), with the scale factor of
  DESIGN.md reading R2 (Matern: fill the ball; Gaussian: c = max(R/rho, ell sqrt(2 pi N))).
* ``additive_fastsum``: per-window application summed with sigma_f^2 (eq. 2.1),
  plus sigma_eps^2 v; ell-derivative via the derivative-kernel coefficients
  (eq. 3.5) with the joint-scaling factor 1/c_w (reading R7).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import i0

GAUSSIAN = 0
MATERN12 = 1


# ----------------------------------------------------------------------------- kernels
def kernel_radial(family, rr, ell, deriv=False):
    """Sub-kernel (eq. 1.1 / 2.2) or its ell-derivative (eq. 2.3) as a function of ||r||^2."""
    rr = np.asarray(rr, dtype=np.float64)
    if family == GAUSSIAN:
        k = np.exp(-rr / (2.0 * ell * ell))
        return rr / ell**3 * k if deriv else k
    rn = np.sqrt(rr)
    k = np.exp(-rn / ell)
    return rn / ell**2 * k if deriv else k


def index_set(N):
    """I_N = {-N/2, ..., N/2 - 1}."""
    return np.arange(-N // 2, N // 2)


def kernel_samples(family, ell, N, d, deriv=False):
    """kappa_R(l/N) for l in I_N^d, array indexed [l_1 + N/2, ..., l_d + N/2] (eq. 3.2)."""
    l = index_set(N) / N
    grids = np.meshgrid(*([l] * d), indexing="ij")
    rr = sum(g * g for g in grids)
    return kernel_radial(family, rr, ell, deriv)


def fourier_coefficients(samples):
    """eq. (3.2): b_k = N^{-d} sum_{l in I_N} s_l e^{-2 pi i l.k / N}, k in I_N (complex array, index k+N/2).

    The d-fold sum is applied one axis at a time with the N x N matrix F[k,l] = e^{-2 pi i k l/N}
    (the exponential of a sum is the product of exponentials; no other reordering).
    """
    s = np.asarray(samples, dtype=np.complex128)
    d = s.ndim
    N = s.shape[0]
    k = index_set(N)
    F = np.exp(-2j * np.pi * np.outer(k, k) / N)  # F[k, l], both indexed from -N/2
    b = s
    for ax in range(d):
        b = np.moveaxis(np.tensordot(F, b, axes=([1], [ax])), 0, ax)
    return b / N**d


# ----------------------------------------------------------------------------- eq. (3.3)
def _exp_table(xs, N, sign):
    """E_t[j, k] = exp(sign * 2 pi i k x_{j,t}), k in I_N, for each axis t."""
    k = index_set(N)
    return [np.exp(sign * 2j * np.pi * np.outer(xs[:, t], k)) for t in range(xs.shape[1])]


def ndft_adjoint(xs, V, N):
    """a_k[c] = sum_j V[j,c] e^{-2 pi i k.x_j}, k in I_N^d (inner sums of eq. 3.3).  Returns (r, N, ..., N)."""
    xs = np.atleast_2d(xs)
    d = xs.shape[1]
    V = np.asarray(V, dtype=np.float64).reshape(xs.shape[0], -1)
    E = _exp_table(xs, N, -1.0)
    if d == 1:
        return (E[0].T @ V.astype(np.complex128)).T
    # the same sums as matrix products: with R[j, (b, c)] = prod_{t >= 1} E_t[j, k_t] (the row-wise outer
    # product of the other axes), a[col][a, (b, c)] = sum_j E_0[j, a] V[j, col] R[j, (b, c)]
    out = np.zeros((V.shape[1], N ** d), dtype=np.complex128)
    for j0 in range(0, xs.shape[0], 8192):
        j1 = min(xs.shape[0], j0 + 8192)
        R = _rowwise_outer([Et[j0:j1] for Et in E[1:]])
        for c in range(V.shape[1]):
            out[c] += ((E[0][j0:j1] * V[j0:j1, c:c + 1]).T @ R).ravel()
    return out.reshape((V.shape[1],) + (N,) * d)


def _rowwise_outer(mats):
    """R[j, (k_1, ..., k_q)] = prod_t mats[t][j, k_t] (row-major flattening)."""
    R = mats[0]
    for M in mats[1:]:
        R = (R[:, :, None] * M[:, None, :]).reshape(R.shape[0], -1)
    return R


def ndft_forward(xs, fhat):
    """f(x_i)[c] = sum_{k in I_N} fhat[c,k] e^{2 pi i k.x_i} (complex).  fhat shape (r, N, ..., N)."""
    xs = np.atleast_2d(xs)
    d = xs.shape[1]
    N = fhat.shape[1]
    E = _exp_table(xs, N, +1.0)
    if d == 1:
        return E[0] @ fhat.T
    # f[i, col] = sum_a E_0[i, a] sum_{(b, c)} fhat[col, a, (b, c)] R[i, (b, c)] (R as in ndft_adjoint)
    r = fhat.shape[0]
    F2 = fhat.reshape(r, N, -1)
    out = np.zeros((xs.shape[0], r), dtype=np.complex128)
    for i0 in range(0, xs.shape[0], 8192):
        i1 = min(xs.shape[0], i0 + 8192)
        R = _rowwise_outer([Et[i0:i1] for Et in E[1:]])
        for c in range(r):
            out[i0:i1, c] = np.sum((E[0][i0:i1] @ F2[c]) * R, axis=1)
    return out


def trunc_fastsum(xs, V, b, rows=None):
    """eq. (3.3) with the real part (reading R5): h_i = Re sum_{k in I_N} b_k a_k e^{2 pi i k.x_i}.
    ``rows`` evaluates the outer sum at those points only (the inner sums a_k run over all points)."""
    N = b.shape[0]
    a = ndft_adjoint(xs, V, N)
    xo = xs if rows is None else np.atleast_2d(xs)[rows]
    return np.real(ndft_forward(xo, b[None, ...] * a))


# ----------------------------------------------------------------------------- App. A: window
def kb_beta(sigma):
    """beta = pi (2 - 1/sigma) (App. A Kaiser-Bessel window)."""
    return math.pi * (2.0 - 1.0 / sigma)


def kb_phi(x, n_g, m, sigma):
    """Kaiser-Bessel window phi(x), truncated to |x| <= m/n_g.

    phi(x) = (1/pi) sinh(beta sqrt(m^2 - n_g^2 x^2)) / sqrt(m^2 - n_g^2 x^2); at |x| = m/n_g the
    limit beta/pi.  (Paper's s is m here, paper's sigma*m is n_g.)
    """
    x = np.asarray(x, dtype=np.float64)
    beta = kb_beta(sigma)
    arg = m * m - (n_g * x) ** 2
    out = np.zeros_like(x)
    pos = arg > 0
    sq = np.sqrt(arg[pos])
    out[pos] = np.sinh(beta * sq) / (math.pi * sq)
    out[arg == 0] = beta / math.pi
    return out


def kb_phi_hat(k, n_g, m, sigma):
    """c_k(phi) = integral phi(x) e^{-2 pi i k x} dx = I0(m sqrt(beta^2 - (2 pi k/n_g)^2)) / n_g (reading R4)."""
    k = np.asarray(k, dtype=np.float64)
    beta = kb_beta(sigma)
    w = 2.0 * math.pi * k / n_g
    return i0(m * np.sqrt(beta * beta - w * w)) / n_g


# ----------------------------------------------------------------------------- App. A: NFFT
def _window_weights(u_t, n_g, m, sigma):
    """For grid positions u = x*n_g (one axis): tap indices l (|u-l| <= m) and phi~(x - l/n_g)."""
    offs = np.arange(-m, m + 1)
    base = np.floor(u_t).astype(np.int64)
    L = base[:, None] + offs[None, :]                  # candidate taps, n x (2m+1)
    W = kb_phi((u_t[:, None] - L) / n_g, n_g, m, sigma)  # zero outside the support
    return L, W


def nfft_adjoint_grid(xs, V, n_g, m, sigma):
    """Spreading g_l = sum_j V_j phi~(x_j - l/n_g), l in I_{n_g}^d, stored at index l mod n_g.  Returns (r, n_g,...)."""
    xs = np.atleast_2d(xs)
    n, d = xs.shape
    V = np.asarray(V, dtype=np.float64).reshape(n, -1)
    r = V.shape[1]
    taps = [_window_weights(xs[:, t] * n_g, n_g, m, sigma) for t in range(d)]
    g = np.zeros((r,) + (n_g,) * d)
    T = 2 * m + 1
    for combo in np.ndindex(*([T] * d)):
        w = np.ones(n)
        idx = []
        for t, o in enumerate(combo):
            w = w * taps[t][1][:, o]
            idx.append(np.mod(taps[t][0][:, o], n_g))
        for c in range(r):
            np.add.at(g[c], tuple(idx), w * V[:, c])
    return g


def nfft_adjoint(xs, V, N, n_g, m, sigma):
    """Adjoint NFFT: a_k ~ sum_j v_j e^{-2 pi i k.x_j} for k in I_N^d (transpose of App. A steps 1-3)."""
    xs = np.atleast_2d(xs)
    d = xs.shape[1]
    g = nfft_adjoint_grid(xs, V, n_g, m, sigma)
    ghat = np.fft.fftn(g, axes=tuple(range(1, d + 1)))   # sum_l g_l e^{-2 pi i k.l/n_g}
    k = index_set(N)
    sel = np.ix_(*([np.mod(k, n_g)] * d))
    c1 = kb_phi_hat(k, n_g, m, sigma)
    ck = c1
    for _ in range(d - 1):
        ck = np.multiply.outer(ck, c1)
    return ghat[(slice(None),) + sel] / (n_g**d * ck[None, ...])


def nfft_forward(xs, fhat, n_g, m, sigma):
    """Forward NFFT (App. A steps 1-3): f(x_i) ~ sum_{k in I_N} fhat_k e^{2 pi i k.x_i}.  fhat (r, N, ..., N)."""
    xs = np.atleast_2d(xs)
    n, d = xs.shape
    r = fhat.shape[0]
    N = fhat.shape[1]
    k = index_set(N)
    c1 = kb_phi_hat(k, n_g, m, sigma)
    ck = c1
    for _ in range(d - 1):
        ck = np.multiply.outer(ck, c1)
    # step 1: b~_k = fhat_k / c_k(phi) on I_N, zero elsewhere in I_{n_g}
    bt = np.zeros((r,) + (n_g,) * d, dtype=np.complex128)
    sel = np.ix_(*([np.mod(k, n_g)] * d))
    bt[(slice(None),) + sel] = fhat / ck[None, ...]
    # step 2: g_l = n_g^{-d} sum_k b~_k e^{2 pi i k.l / n_g}  (so that FFT(g)_k c_k = fhat_k)
    g = np.fft.ifftn(bt, axes=tuple(range(1, d + 1)))
    # step 3: f(x_i) = sum_l g_l phi~(x_i - l/n_g)
    taps = [_window_weights(xs[:, t] * n_g, n_g, m, sigma) for t in range(d)]
    out = np.zeros((n, r), dtype=np.complex128)
    T = 2 * m + 1
    for combo in np.ndindex(*([T] * d)):
        w = np.ones(n)
        idx = []
        for t, o in enumerate(combo):
            w = w * taps[t][1][:, o]
            idx.append(np.mod(taps[t][0][:, o], n_g))
        for c in range(r):
            out[:, c] += w * g[c][tuple(idx)]
    return out


def nfft_fastsum(xs, V, b, sigma, m):
    """eq. (3.3) evaluated with adjoint NFFT -> multiply by b_k -> NFFT, real part (reading R5)."""
    N = b.shape[0]
    n_g = int(round(sigma * N))
    a = nfft_adjoint(xs, V, N, n_g, m, sigma)
    return np.real(nfft_forward(xs, b[None, ...] * a, n_g, m, sigma))


# ----------------------------------------------------------------------------- scaling + additive operator
def window_scaling(Xw, family, ell, N, eps_B):
    """Reading R2: center = bounding-box midpoint, R = max_i ||x_i - center||_2, rho = 1/4 - eps_B/2,
    c = R/rho (Matern) or max(R/rho, ell sqrt(2 pi N)) (Gaussian); R = 0 -> R/rho replaced by 1.
    Returns (center, c, scaled points (Xw - center)/c)."""
    Xw = np.asarray(Xw, dtype=np.float64)
    center = 0.5 * (Xw.min(axis=0) + Xw.max(axis=0))
    R = float(np.sqrt(((Xw - center) ** 2).sum(axis=1)).max()) if Xw.shape[0] else 0.0
    rho = 0.25 - eps_B / 2.0
    c = R / rho if R > 0 else 1.0
    if family == GAUSSIAN:
        c = max(c, ell * math.sqrt(2.0 * math.pi * N))
    return center, c, (Xw - center) / c


def additive_fastsum(X, windows, family, theta, V, N, eps_B=1.0 / 16, method="ndft", sigma=2.0, m=6,
                     ops=("K", "dell", "dsf", "dse"), scales=None, rows=None):
    """Truncated-Fourier (method='ndft', eq. 3.3) or NFFT (method='nfft', App. A) additive operator.

    Y = sigma_f^2 sum_w h_w + sigma_eps^2 V;  dY_ell = sigma_f^2 sum_w (1/c_w) h_w[b(kappa_der at ell/c_w)];
    dY_sf = 2 sigma_f sum_w h_w;  dY_se = 2 sigma_eps V.  ``scales`` optionally fixes c_w (list).
    ``rows`` (method 'ndft' only) returns the outputs at those rows only."""
    X = np.asarray(X, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64).reshape(X.shape[0], -1)
    sf, ell, se = theta
    if rows is not None and method != "ndft":
        raise ValueError("rows= needs method='ndft'")
    Vo = V if rows is None else V[rows]
    S = np.zeros_like(Vo)
    SD = np.zeros_like(Vo)
    for wi, win in enumerate(windows):
        Xw = X[:, list(win)]
        d = Xw.shape[1]
        center, c, xs = window_scaling(Xw, family, ell, N, eps_B)
        if scales is not None:
            c = float(scales[wi])
            xs = (Xw - center) / c
        ell_eff = ell / c
        for deriv in (False, True):
            if deriv and "dell" not in ops:
                continue
            b = fourier_coefficients(kernel_samples(family, ell_eff, N, d, deriv))
            if method == "ndft":
                h = trunc_fastsum(xs, V, b, rows)
            else:
                h = nfft_fastsum(xs, V, b, sigma, m)
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
    if "dse" in ops:
        out["dse"] = 2.0 * se * Vo
    return out
