"""Dense float64 cross products K_{*X} V for prediction.  TEST INFRASTRUCTURE ONLY.

SURVEY.md 8(f) f2: the posterior mean and variance of a GP need products of the kernel between
test points X_t and training points X_s with a block V,
with the additive kernel of eq. (1.1) and no noise term (sigma_eps^2 I only couples a
point with itself, and a test point is not a training point):

    Y_t[i] = sigma_f^2 * sum_w sum_j kappa(x_t[i]^{W_w} - x_s[j]^{W_w}; ell) * V[j]

kappa = exp(-|r|^2 / (2 ell^2)) (Gaussian) or exp(-|r| / ell) (Matern(1/2)).  Written
out plainly: pairwise differences per window, the kernel formula, a matrix product (library
primitive), summed over windows in order.  Pinned by tests/test_oracle_cross.py against the
C dense oracle (oracle/dense.c) and brute-force loops.
"""
from __future__ import annotations

import numpy as np


def dense_cross(Xs, Xt, windows, family, theta, V):
    """(n_t x r) array Y_t = sigma_f^2 sum_w K_w(X_t, X_s) V; Xs: n_s x p, Xt: n_t x p, V: n_s x r."""
    Xs = np.asarray(Xs, dtype=np.float64)
    Xt = np.asarray(Xt, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    if V.ndim == 1:
        V = V[:, None]
    sigma_f, ell, _ = (float(t) for t in theta)
    Y = np.zeros((Xt.shape[0], V.shape[1]), dtype=np.float64)
    for w in windows:
        cols = list(w)
        diff = Xt[:, None, cols] - Xs[None, :, cols]           # n_t x n_s x d
        r2 = np.sum(diff * diff, axis=2)
        if family == 0:
            K = np.exp(-r2 / (2.0 * ell * ell))
        else:
            K = np.exp(-np.sqrt(r2) / ell)
        Y += K @ V
    return sigma_f * sigma_f * Y
