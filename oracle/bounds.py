"""Closed-form error bounds of PAPER.md §4 and App. A.  TEST INFRASTRUCTURE ONLY.

Used as pins: the oracle's Fourier coefficients (eq. 3.2) and truncated series must
stay below these bounds, and the NFFT oracle below eq. (A.3).

* ``delta_m``     Lemma 4.2
* ``thm44``       Theorem 4.4: ||kappa~^m_ERR||_inf <= 8 / (pi^2 ell (m - 2 sqrt 3))
* ``thm45``       Theorem 4.5: 32/(3 ell^4 pi^4 (m-2sqrt3)^3) + 8/(ell^2 pi^2 (m-2sqrt3))
* ``nfft_bound``  eq. (A.3), per unit ||b||_1, d = 1

Lemma 4.3's delta^derm is not carried: it bounds nothing on the product path and
the only check available for it (dominance of a sampled periodisation gap, which it exceeds by
20-1500x) cannot tell a transcription error from the bound itself (Weak 1).
* ``periodized``  kappa~(r) = sum_{z in Z^d} kappa(r + z) (Def. 4.1), truncated image sum
"""
from __future__ import annotations

import itertools
import math

import numpy as np

from .fourier import kernel_radial

S3 = math.sqrt(3.0)


def delta_m(ell):
    a = 1.0 + 2.0 * S3 * ell
    return (3.0 * math.exp(-1.0 / (2.0 * S3 * ell)) * a + 3.0 * math.exp(-1.0 / (S3 * ell)) * a * a
            + math.exp(-3.0 / (2.0 * S3 * ell)) * a ** 3)


def thm44(m, ell):
    return 8.0 / (math.pi**2 * ell * (m - 2.0 * S3))


def thm45(m, ell):
    q = m - 2.0 * S3
    return 32.0 / (ell**4 * math.pi**4 * 3.0 * q**3) + 8.0 / (ell**2 * math.pi**2 * q)


def nfft_bound(s, sigma):
    """eq. (A.3) factor: 4 pi (s + sqrt s) (1 - 1/sigma)^{1/4} e^{-2 pi s sqrt(1 - 1/sigma)}."""
    return 4.0 * math.pi * (s + math.sqrt(s)) * (1.0 - 1.0 / sigma) ** 0.25 * math.exp(-2.0 * math.pi * s * math.sqrt(1.0 - 1.0 / sigma))


def periodized(family, r, ell, deriv=False, images=4):
    """kappa~(r) = sum_{z in Z^d, |z_t| <= images} kappa(r + z) for r of shape (n, d)."""
    r = np.atleast_2d(r)
    d = r.shape[1]
    out = np.zeros(r.shape[0])
    for z in itertools.product(range(-images, images + 1), repeat=d):
        rz = r + np.array(z, dtype=np.float64)[None, :]
        out += kernel_radial(family, (rz * rz).sum(axis=1), ell, deriv)
    return out
