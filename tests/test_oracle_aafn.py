"""Pins of the AAFN oracle (oracle/aafn.py; SPEC aafn-precond S:288-352).

FPS against hand-derived cases; the factorization against its defining identities (M = K^ with every
point a landmark, n = 1 scalar case, log det M = log det of the densely assembled M, symmetry and
positivity of M^{-1}, log det M -> log det K^ as k grows); the split-preconditioned objective against
the dense eq. (1.2) / (1.3) quantities; and the paper's Fig. 3 claim in miniature (AAFN-PCG needs no
more iterations than plain CG, and far fewer in the middle-ell regime)."""
import math

import numpy as np
import pytest

from oracle import aafn as A
from oracle import krylov as KR


def test_fps_hand_cases():
    pts = np.array([[0.0], [1.0], [2.0]])
    assert sorted(A.fps(pts, 2)) == [0, 2]            # SPEC: {2, 0} (seed tie -> lowest index)
    assert A.fps(pts, 1) == [0]
    assert sorted(A.fps(pts, 3)) == [0, 1, 2]         # k = n: every point
    sq = np.array([[0, 0], [1, 0], [0, 1], [1, 1], [0.5, 0.5], [0.52, 0.5]])
    p = A.fps(sq, 5)
    assert p[0] == 0 and set(p[1:4]) == {1, 2, 3} and p[4] in (4, 5)
    assert p[1] == 3                                  # opposite corner first (max-min distance sqrt 2)


def _problem(n, seed=0, p=6):
    rng = np.random.default_rng(seed)
    X = rng.random((n, p))
    return X, [(0, 1, 2), (3, 4, 5)][: p // 3], (0.8, 0.3, 0.2)


def test_all_landmarks_is_exact():
    X, W, th = _problem(40, 1)
    pre = A.Aafn(X, W, 0, th, 40, 1)
    K = A.khat_dense(X, W, 0, th)
    assert pre.lm.size == 40
    np.testing.assert_allclose(pre.assemble_M(), K, rtol=0, atol=1e-10 * np.abs(K).max())
    v = np.random.default_rng(2).standard_normal(40)
    u = pre.apply_inverse(v[:, None])[:, 0]
    assert np.linalg.norm(K @ u - v) <= 1e-10 * np.linalg.norm(v)
    x, hist = KR.pcg(lambda B: pre.U_inv(K @ pre.U_invT(B)), pre.U_inv(v[:, None])[:, 0], 3)
    assert hist[0] <= 1e-10                            # S_op = I: one iteration
    assert pre.logdet == pytest.approx(np.linalg.slogdet(K)[1], rel=1e-12)


def test_scalar_case():
    X = np.array([[0.2, 0.4, 0.6]])
    pre = A.Aafn(X, [(0, 1), (2,)], 1, (1.3, 0.5, 0.4), 3, 1)
    assert pre.logdet == pytest.approx(math.log(1.3**2 * 2 + 0.4**2), rel=1e-14)


@pytest.mark.parametrize("kpw,fill", [(5, 1), (5, 4), (12, 1), (12, 6)])
def test_logdet_symmetry_positivity(kpw, fill):
    X, W, th = _problem(120, 3)
    pre = A.Aafn(X, W, 1, th, kpw, fill)
    M = pre.assemble_M()
    assert np.abs(M - M.T).max() <= 1e-10 * np.abs(M).max()
    assert pre.logdet == pytest.approx(np.linalg.slogdet(M)[1], rel=1e-8)
    rng = np.random.default_rng(4)
    for _ in range(20):
        u, v = rng.standard_normal(120), rng.standard_normal(120)
        Mu, Mv = pre.apply_inverse(u[:, None])[:, 0], pre.apply_inverse(v[:, None])[:, 0]
        assert abs(Mu @ v - u @ Mv) <= 1e-10 * (abs(Mu @ v) + 1e-300)
        assert v @ Mv > 0
    # M^{-1} M = I
    assert np.abs(pre.apply_inverse(M) - np.eye(120)).max() <= 1e-8


def test_two_points_one_landmark():
    X = np.array([[0.1, 0.2, 0.3], [0.4, 0.1, 0.9]])
    th = (1.0, 0.5, 0.3)
    pre = A.Aafn(X, [(0, 1, 2)], 0, th, 1, 1)
    K = A.khat_dense(X, [(0, 1, 2)], 0, th)
    lm = pre.lm[0]
    o = 1 - lm
    S = K[o, o] - K[o, lm] ** 2 / K[lm, lm]            # 2 x 2 Schur complement by hand
    assert pre.logdet == pytest.approx(math.log(K[lm, lm]) + math.log(S), rel=1e-13)
    np.testing.assert_allclose(pre.assemble_M(), K, rtol=1e-12)   # one landmark + exact 1x1 Schur = K


def test_logdet_converges_with_rank():
    X, W, th = _problem(50, 5)
    K = A.khat_dense(X, W, 0, th)
    ref = np.linalg.slogdet(K)[1]
    errs = [abs(A.Aafn(X, W, 0, th, k, 10).logdet - ref) for k in (2, 5, 10, 25)]
    assert all(b <= a * (1 + 1e-9) for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] <= 1e-8 * abs(ref)


def test_objective_identities():
    """Split-preconditioned objective: with M = K^ the SLQ correction vanishes; in general
    log det K^ = log det M + tr logm(M^{-1} K^) (eq. 1.3), checked with n Lanczos steps and probes
    sqrt(n) e_j (exact trace), and y^T x equals y^T K^{-1} y once CG has converged."""
    X, W, th = _problem(30, 7)
    K = A.khat_dense(X, W, 1, th)
    y = np.random.default_rng(8).standard_normal(30)
    Z = math.sqrt(30) * np.eye(30)
    full = A.Aafn(X, W, 1, th, 30, 1)
    o = A.objective_aafn(lambda B: K @ B, y, Z, full, 5, 3)
    assert abs(o["slq"]) <= 1e-8 * 30
    pre = A.Aafn(X, W, 1, th, 4, 3)
    o = A.objective_aafn(lambda B: K @ B, y, Z, pre, 30, 30)
    assert o["logdetM"] + o["slq"] == pytest.approx(np.linalg.slogdet(K)[1], rel=1e-8)
    assert o["quad"] == pytest.approx(y @ np.linalg.solve(K, y), rel=1e-8)
    assert o["cg_relres_true"] <= 1e-8


@pytest.mark.parametrize("family", [0, 1])
def test_fig3_in_miniature(family):
    """PAPER Fig. 3: 6-D hypercube of side n^{1/3}, windows [[1,2,3],[4,5,6]], sigma_f^2 = 1/P,
    sigma_eps^2 = 0.01, tol 1e-4, cap 200: AAFN-PCG never needs more iterations than CG, and far fewer
    at a middle ell.  (n = 600 instead of 3000, 60 landmarks per window, fill 10.)"""
    n = 600
    rng = np.random.default_rng(11)
    X = rng.random((n, 6)) * n ** (1 / 3)
    W = [(0, 1, 2), (3, 4, 5)]
    b = rng.uniform(-0.5, 0.5, n)

    def iters(apply, rhs):
        x, hist = KR.pcg(apply, rhs, 200)
        return next((i + 1 for i, h in enumerate(hist) if h <= 1e-4), 201)

    counts = []
    for ell in (0.5, 2.0, 8.0):
        th = (math.sqrt(0.5), ell, 0.1)
        K = A.khat_dense(X, W, family, th)
        plain = iters(lambda B: K @ B, b)
        pre = A.Aafn(X, W, family, th, 60, 10)
        pc = iters(lambda B: pre.U_inv(K @ pre.U_invT(B)), pre.U_inv(b[:, None])[:, 0])
        counts.append((plain, pc))
        assert pc <= plain, (ell, plain, pc)
    assert max(p - q for p, q in counts) >= 10, counts


@pytest.mark.parametrize("family", [0, 1])
def test_gradient_aafn_exact_trace_matches_fd(family):
    """With probes sqrt(n) e_j (exact trace) and converged solves the AAFN gradient is the exact gradient
    of eq. (1.2) -> central finite differences of the dense objective; with Rademacher probes it equals
    the diagonal-M estimator once both solves have converged (the control variates cancel there)."""
    from oracle import dense_apply
    rng = np.random.default_rng(family)
    n = 30
    X = rng.random((n, 5))
    W = [(0, 1, 2), (3, 4)]
    y = rng.standard_normal(n)
    theta = (1.2, 0.4, 0.3)
    K = A.khat_dense(X, W, family, theta)

    def dK(B):
        o = dense_apply(X, W, family, theta, B, ops=("dell", "dsf", "dse"))
        return {"ell": o["dell"], "sf": o["dsf"], "se": o["dse"]}

    pre = A.Aafn(X, W, family, theta, 4, 3)
    g = A.gradient_aafn(lambda B: K @ B, dK, y, math.sqrt(n) * np.eye(n), pre, 200)["grad"]

    def Zd(th):
        Kt = A.khat_dense(X, W, family, th)
        return 0.5 * (y @ np.linalg.solve(Kt, y) + np.linalg.slogdet(Kt)[1])

    for j, idx in (("sf", 0), ("ell", 1), ("se", 2)):
        h = 1e-5 * theta[idx]
        tp, tm = list(theta), list(theta)
        tp[idx] += h
        tm[idx] -= h
        assert g[j] == pytest.approx((Zd(tuple(tp)) - Zd(tuple(tm))) / (2 * h), rel=1e-7), j
    Zr = np.where(rng.random((n, 5)) < 0.5, -1.0, 1.0)
    ga = A.gradient_aafn(lambda B: K @ B, dK, y, Zr, pre, 200)["grad"]
    c = theta[0] ** 2 * 2 + theta[2] ** 2
    gd = KR.gradient_diag(lambda B: K @ B, dK, y, Zr, c, {"sf": 4 * theta[0], "ell": 0.0, "se": 2 * theta[2]}, 200)["grad"]
    for j in ("sf", "ell", "se"):
        assert ga[j] == pytest.approx(gd[j], rel=1e-9)
