"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no kernel, no scaling rule, no
Fourier coefficients): only the BASELINE.json configurations written out as
data, and seeded numpy generators for X (points), V (right-hand sides) and row
samples.  It is the one piece of code that both ``oracle/`` and the CUDA path
(via its tests and bench.py) consume.

Recipe (SURVEY.md §8(d) "Synthetic inputs"; BASELINE.json ``configs``):
  * generator: ``numpy.random.default_rng(seed)`` (PCG64);
  * seeds: X = 1000 + cfg, V = 2000 + cfg, row sample = 3000 + cfg;
  * X: c1, c3: ``rng.random((n, p))`` (uniform [0,1)); c2, c4, c5:
    ``rng.standard_normal((n, p))`` then per-column min-max to [0, 1]
    (reading R12);
  * V: c1, c2: one column ~ N(0,1); c3, c4, c5: column 0 ~ N(0,1), columns
    1..10 Rademacher (+-1 equiprobable) (readings R10, R11);
  * windows: consecutive features, 0-based here.

The paper's own workloads are UCI datasets (§5.3; Table 3,
P:1134-1168) that are not available; these synthetic sets stand in for them
(window shapes of Table 3, point counts spanning its range).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

GAUSSIAN = 0
MATERN12 = 1


@dataclass(frozen=True)
class Workload:
    name: str
    index: int                 # 1-based config number (seeds derive from it)
    n: int
    p: int
    windows: Tuple[Tuple[int, ...], ...]
    family: int
    sigma_f: float
    ell: float
    sigma_eps: float
    r: int
    N: int                     # bandwidth (paper's m), Fourier coefficients per axis
    sigma_over: float          # oversampling factor sigma (paper's sigma)
    m: int                     # window half-support in grid cells (paper's s)
    eps_B: float
    ops: Tuple[str, ...]       # requested products: subset of ("K", "dell", "dsf")
    x_kind: str                # "uniform" | "normal_minmax"
    v_kind: str                # "normal1" | "normal_plus_rademacher"
    description: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def units(self) -> int:
        """n * r * windows: the unit the throughput metric counts (BASELINE.json metric); for a
        cross-product workload (extra n_src) the TARGET points count: (n - n_src) * r * windows."""
        return (self.n - self.extra.get("n_src", 0)) * self.r * len(self.windows)


def _consecutive(start_count: int, size: int, count: int):
    return tuple(tuple(range(i * size, i * size + size)) for i in range(count))


CONFIGS = {
    "c1": Workload("c1", 1, 2000, 3, _consecutive(0, 3, 1), GAUSSIAN, 1.0, 0.2, 0.1, 1, 32, 2.0, 6, 1.0 / 16,
                   ("K",), "uniform", "normal1",
                   "n=2000 uniform [0,1]^3, one d=3 Gaussian window, K v, N=32, m=6"),
    "c2": Workload("c2", 2, 20000, 9, _consecutive(0, 3, 3), GAUSSIAN, 1.0, 0.5, 0.05, 1, 32, 2.0, 6, 1.0 / 16,
                   ("K", "dell"), "normal_minmax", "normal1",
                   "n=20000 p=9 N(0,1) min-max, 3 Gaussian windows of 3, K v + dK/dell v, N=32, m=6"),
    "c3": Workload("c3", 3, 100000, 8, _consecutive(0, 2, 4), MATERN12, 1.0, 1.0, 0.1, 11, 128, 2.0, 8, 1.0 / 16,
                   ("K",), "uniform", "normal_plus_rademacher",
                   "n=1e5 p=8 uniform, 4 Matern(1/2) windows of 2, r=11, N=128, m=8"),
    "c4": Workload("c4", 4, 1000000, 12, _consecutive(0, 3, 4), GAUSSIAN, 1.0, 0.3, 0.01, 11, 32, 2.0, 6, 1.0 / 16,
                   ("K", "dell", "dsf"), "normal_minmax", "normal_plus_rademacher",
                   "n=1e6 p=12 N(0,1) min-max, 4 Gaussian windows of 3, r=11, K/dell/dsf, N=32, m=6"),
    "c5": Workload("c5", 5, 500000, 9, _consecutive(0, 3, 3), GAUSSIAN, 1.0, 0.5, 0.05, 11, 32, 2.0, 6, 1.0 / 16,
                   ("K",), "normal_minmax", "normal_plus_rademacher",
                   "one Z~ evaluation: n=5e5 p=9, 3 Gaussian windows, 50 CG + 30 Lanczos, r=11 (theta per reading R10)",
                   extra={"cg_iters": 50, "lanczos_steps": 30, "n_z": 10}),
    # SURVEY.md 8(f) f2 (not a BASELINE.json config): prediction at c4 scale -- K_{*X} V from
    # 1e6 training points to 1e5 test points drawn with them (rows n_src.. of one c4-style X)
    "x4": Workload("x4", 6, 1100000, 12, _consecutive(0, 3, 4), GAUSSIAN, 1.0, 0.3, 0.01, 11, 32, 2.0, 6, 1.0 / 16,
                   ("K",), "normal_minmax", "normal_plus_rademacher",
                   "cross K_{*X} V: 1e6 training -> 1e5 test points, p=12 N(0,1) min-max, 4 Gaussian windows of 3, "
                   "r=11, N=32, m=6",
                   extra={"n_src": 1000000}),
    # SURVEY.md 8(f) f3 (not a BASELINE.json config): c5's objective with the AAFN preconditioner
    # (800 FPS landmarks per window, 2396 after merging); a step rebuilds the factors for theta
    "c5a": Workload("c5a", 5, 500000, 9, _consecutive(0, 3, 3), GAUSSIAN, 1.0, 0.5, 0.05, 11, 32, 2.0, 6, 1.0 / 16,
                    ("K",), "normal_minmax", "normal_plus_rademacher",
                    "one Z~ evaluation with AAFN (800 landmarks/window): set_theta + factor + 50 PCG + 30 Lanczos "
                    "on the split-preconditioned operator, n=5e5 p=9, 3 Gaussian windows, r=11",
                    extra={"cg_iters": 50, "lanczos_steps": 30, "n_z": 10, "aafn_kpw": 800}),
    # SURVEY.md 8(f) f4 (not a BASELINE.json config): c3 with the boundary-regularised kappa_R
    # (inner eps_I = 1/N, p = 2, near-field correction; outer eps_B): per-column error ~2e-4 at 1/4 of
    # the near-field pairs of eps_I = 2/N (tests/test_gpu_regularized.py checks both)
    "c3r": Workload("c3r", 3, 100000, 8, _consecutive(0, 2, 4), MATERN12, 1.0, 1.0, 0.1, 11, 128, 2.0, 8, 1.0 / 16,
                    ("K",), "uniform", "normal_plus_rademacher",
                    "c3 with kappa_R (eps_I = 1/N, p = 2, near-field correction): n=1e5, 4 Matern(1/2) windows of 2, "
                    "r=11, N=128, m=8",
                    extra={"reg_eps_I": 1.0 / 128, "reg_p": 2}),
    # SURVEY.md 8(f) f1 (not a BASELINE.json config): one gradient of Z~ at c5's sizes -- 50 block
    # PCG iterations on [y | Z] (r = 11) and one fused derivative product (dKhat/dell, dKhat/dsigma_f)
    "g5": Workload("g5", 5, 500000, 9, _consecutive(0, 3, 3), GAUSSIAN, 1.0, 0.5, 0.05, 11, 32, 2.0, 6, 1.0 / 16,
                   ("K",), "normal_minmax", "normal_plus_rademacher",
                   "one gradient of Z~: n=5e5 p=9, 3 Gaussian windows, 50 block-PCG iterations at r=11 + one "
                   "dKhat/dell, dKhat/dsigma_f product (theta per reading R10)",
                   extra={"grad_cg_iters": 50, "n_z": 10}),
}


def make_X(wl: Workload, n: int | None = None, seed: int | None = None) -> np.ndarray:
    """Points X (n x p, float64, C-contiguous)."""
    n = wl.n if n is None else n
    rng = np.random.default_rng(1000 + wl.index if seed is None else seed)
    if wl.x_kind == "uniform":
        X = rng.random((n, wl.p))
    elif wl.x_kind == "normal_minmax":
        X = rng.standard_normal((n, wl.p))
        lo = X.min(axis=0)
        hi = X.max(axis=0)
        X = (X - lo) / np.where(hi > lo, hi - lo, 1.0)
    else:
        raise ValueError(wl.x_kind)
    return np.ascontiguousarray(X, dtype=np.float64)


def make_V(wl: Workload, n: int | None = None, r: int | None = None, seed: int | None = None) -> np.ndarray:
    """Right-hand sides V (n x r, float64, row-major)."""
    n = wl.n if n is None else n
    r = wl.r if r is None else r
    rng = np.random.default_rng(2000 + wl.index if seed is None else seed)
    V = np.empty((n, r), dtype=np.float64)
    V[:, 0] = rng.standard_normal(n)
    if r > 1:
        if wl.v_kind == "normal_plus_rademacher":
            V[:, 1:] = np.where(rng.random((n, r - 1)) < 0.5, -1.0, 1.0)
        else:
            V[:, 1:] = rng.standard_normal((n, r - 1))
    return V


def make_rows(wl: Workload, count: int, n: int | None = None, seed: int | None = None) -> np.ndarray:
    """Seeded sorted subset of row indices (for row-sampled parity at full size)."""
    n = wl.n if n is None else n
    rng = np.random.default_rng(3000 + wl.index if seed is None else seed)
    count = min(count, n)
    return np.sort(rng.choice(n, size=count, replace=False)).astype(np.int64)


def windows_flat(windows) -> Tuple[np.ndarray, np.ndarray]:
    """(concatenated feature ids, lengths) as int32 arrays, the C-ABI's window encoding."""
    feat = np.array([f for w in windows for f in w], dtype=np.int32)
    lens = np.array([len(w) for w in windows], dtype=np.int32)
    return feat, lens


def random_problem(seed: int, n: int, p: int, windows, r: int, x_kind: str = "uniform") -> Tuple[np.ndarray, np.ndarray]:
    """Small seeded (X, V) pair for parity sweeps over shapes not in BASELINE.json."""
    rng = np.random.default_rng(seed)
    if x_kind == "uniform":
        X = rng.random((n, p))
    else:
        X = rng.standard_normal((n, p))
        lo, hi = X.min(axis=0), X.max(axis=0)
        X = (X - lo) / np.where(hi > lo, hi - lo, 1.0)
    V = rng.standard_normal((n, r))
    return np.ascontiguousarray(X), np.ascontiguousarray(V)
