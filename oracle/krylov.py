"""Krylov estimators of the preconditioned objective Z~(theta) (eq. 1.4).  TEST INFRASTRUCTURE ONLY.

Written from PAPER.md §1 in the paper's order, with the readings of DESIGN.md:

* ``pcg``: preconditioned conjugate gradients for alpha = Khat^{-1} Y ("the preconditioned
  Conjugate Gradient (CG) algorithm is used to approximate Khat^{-1} Y"), started at x0 = 0
   and run for a fixed number of iterations (BASELINE.json c5: 50; reading R11).
* ``lanczos``: the Lanczos tridiagonalisation behind stochastic Lanczos quadrature ("SLQ")
  with full reorthogonalisation by classical Gram-Schmidt applied twice (reading R11), stopped
  early on breakdown beta_j <= 1e-12 ||S q_j|| (reading R14).
* ``slq_sample``: z^T logm(S) z ~= ||z||^2 sum_j tau_j^2 log theta_j with (theta_j, tau_j) the
  eigenvalues and first eigenvector components of T (Gauss quadrature).
* ``objective_diag``: eq. (1.4) with M = diag(Khat) (reading R11):
  Z~ = 1/2 (Y^T alpha + log det M + (1/n_z) sum_i z_i^T logm(M^{-1} Khat) z_i + n log 2 pi),
  where the SLQ runs on the symmetric form S = M^{-1/2} Khat M^{-1/2} (same trace).

The operator is passed in as ``apply_K(B) -> Khat B`` for an n x c block (the tests use the
dense float64 oracle, oracle/dense.c).  The CG direction and the n_z Lanczos vectors are applied
together as one n x (1 + n_z) block per iteration, like the GPU driver; column c of Khat B
depends only on column c of B, so this is the same arithmetic as one product per column.
"""
from __future__ import annotations

import math

import numpy as np

BREAKDOWN_REL = 1e-12


def pcg(apply_A, b, iters, minv_diag=None):
    """Fixed-iteration PCG from x0 = 0.  Returns (x, relative residual history)."""
    b = np.asarray(b, dtype=np.float64)
    minv = np.ones_like(b) if minv_diag is None else np.asarray(minv_diag, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    z = minv * r
    p = z.copy()
    rz = float(r @ z)
    bn = float(np.linalg.norm(b))
    hist = []
    for _ in range(iters):
        if rz == 0.0:
            break
        Ap = apply_A(p[:, None])[:, 0]
        a = rz / float(p @ Ap)
        x = x + a * p
        r = r - a * Ap
        z = minv * r
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
        hist.append(float(np.linalg.norm(r)) / bn)
    return x, hist


def lanczos(apply_S, z, steps):
    """Lanczos on symmetric S from q_1 = z/||z|| with full reorthogonalisation (CGS2).

    Returns (alpha[k], beta[k-1]) of the k x k tridiagonal T (k = steps unless breakdown)."""
    z = np.asarray(z, dtype=np.float64)
    Q = [z / np.linalg.norm(z)]
    alpha, beta = [], []
    for j in range(steps):
        q = Q[j]
        w = apply_S(q[:, None])[:, 0]
        wn = float(np.linalg.norm(w))
        a = float(q @ w)
        w = w - a * q
        if j > 0:
            w = w - beta[j - 1] * Q[j - 1]
        B = np.stack(Q, axis=1)
        for _ in range(2):                      # classical Gram-Schmidt, twice
            w = w - B @ (B.T @ w)
        alpha.append(a)
        if j == steps - 1:
            break
        bj = float(np.linalg.norm(w))
        if bj <= BREAKDOWN_REL * wn:             # breakdown: truncate T here (reading R14)
            break
        beta.append(bj)
        Q.append(w / bj)
    return np.array(alpha), np.array(beta)


def slq_sample(alpha, beta, znorm2):
    """||z||^2 sum_j tau_j^2 log theta_j from T = tridiag(beta, alpha, beta)."""
    k = len(alpha)
    T = np.diag(alpha)
    if k > 1:
        T += np.diag(beta[: k - 1], 1) + np.diag(beta[: k - 1], -1)
    theta, U = np.linalg.eigh(T)
    tau2 = U[0, :] ** 2
    return float(znorm2 * np.sum(tau2 * np.log(theta)))


def objective_diag(apply_K, y, Z, diagM, cg_iters, lanczos_steps):
    """eq. (1.4) with a diagonal preconditioner M = diag(diagM).  Returns a dict of the terms.

    The CG direction and the Lanczos vectors go through apply_K as one block per iteration."""
    y = np.asarray(y, dtype=np.float64)
    Z = np.asarray(Z, dtype=np.float64)
    n, n_z = Z.shape
    dM = np.asarray(diagM, dtype=np.float64) * np.ones(n)
    s = 1.0 / np.sqrt(dM)                       # S = M^{-1/2} Khat M^{-1/2}

    # CG state (x0 = 0)
    x = np.zeros(n)
    r = y.copy()
    zc = r / dM
    p = zc.copy()
    rz = float(r @ zc)
    yn = float(np.linalg.norm(y))
    cg_hist = []
    # Lanczos state per probe
    Q = [[Z[:, i] / np.linalg.norm(Z[:, i])] for i in range(n_z)]
    alpha = [[] for _ in range(n_z)]
    beta = [[] for _ in range(n_z)]
    live = [True] * n_z

    for t in range(max(cg_iters, lanczos_steps)):
        cols, who = [], []
        if t < cg_iters and rz != 0.0:
            cols.append(p)
            who.append(("cg", -1))
        if t < lanczos_steps:
            for i in range(n_z):
                if live[i]:
                    cols.append(s * Q[i][t])
                    who.append(("lz", i))
        if not cols:
            break
        KB = apply_K(np.stack(cols, axis=1))
        for c, (kind, i) in enumerate(who):
            if kind == "cg":
                Ap = KB[:, c]
                a = rz / float(p @ Ap)
                x = x + a * p
                r = r - a * Ap
                zc = r / dM
                rz_new = float(r @ zc)
                p = zc + (rz_new / rz) * p
                rz = rz_new
                cg_hist.append(float(np.linalg.norm(r)) / yn)
            else:
                q = Q[i][t]
                w = s * KB[:, c]
                wn = float(np.linalg.norm(w))
                a = float(q @ w)
                w = w - a * q
                if t > 0:
                    w = w - beta[i][t - 1] * Q[i][t - 1]
                B = np.stack(Q[i], axis=1)
                for _ in range(2):
                    w = w - B @ (B.T @ w)
                alpha[i].append(a)
                if t == lanczos_steps - 1:
                    live[i] = False
                    continue
                bj = float(np.linalg.norm(w))
                if bj <= BREAKDOWN_REL * wn:
                    live[i] = False
                    continue
                beta[i].append(bj)
                Q[i].append(w / bj)

    quad = float(y @ x)
    logdetM = float(np.sum(np.log(dM)))
    samples = [slq_sample(np.array(alpha[i]), np.array(beta[i]), float(Z[:, i] @ Z[:, i])) for i in range(n_z)]
    slq = float(np.mean(samples))
    Zt = 0.5 * (quad + logdetM + slq + n * math.log(2.0 * math.pi))
    return {"Z": Zt, "quad": quad, "logdetM": logdetM, "slq": slq, "samples": samples, "x": x,
            "cg_hist": cg_hist, "steps": [len(a) for a in alpha], "alpha": alpha, "beta": beta}


def gradient_diag(apply_K, apply_dK, y, Z, c, dc, cg_iters):
    """eq. (div) with M = c I (reading R11), for theta = (sigma_f, ell, sigma_eps):

        dZ~/dtheta_j ~= 1/2 ( -alpha^T dKhat_j alpha + tr(M^{-1} dM_j)
                              + (1/n_z) sum_i z_i^T (M^{-1} Khat)^{-1} d(M^{-1} Khat)_j z_i ).

    With M = c I:  tr(M^{-1} dM_j) = n dc_j / c  and
    (M^{-1} Khat)^{-1} d(M^{-1} Khat)_j = Khat^{-1} dKhat_j - (dc_j / c) I, so the probe term is
    z_i^T w_i' - (dc_j / c) z_i^T z_i with w_i' = Khat^{-1} dKhat_j z_i; by symmetry of Khat,
    z_i^T Khat^{-1} dKhat_j z_i = (Khat^{-1} z_i)^T (dKhat_j z_i).  alpha = Khat^{-1} y and
    Khat^{-1} z_i come from fixed-iteration PCG (``pcg``, M^{-1} = 1/c) from x0 = 0.

    apply_K(B) -> Khat B; apply_dK(B) -> dict j -> dKhat_j B for j in ("sf", "ell", "se").
    dc: dict j -> dc/dtheta_j.  Returns dict j -> gradient component, plus the solves."""
    y = np.asarray(y, dtype=np.float64)
    Z = np.asarray(Z, dtype=np.float64)
    n, n_z = Z.shape
    minv = np.full(n, 1.0 / c)
    alpha, _ = pcg(apply_K, y, cg_iters, minv)
    W = np.stack([pcg(apply_K, Z[:, i], cg_iters, minv)[0] for i in range(n_z)], axis=1)
    D = apply_dK(np.column_stack([alpha, Z]))
    grad = {}
    for j, Dj in D.items():
        quad = -float(alpha @ Dj[:, 0])
        probes = np.mean([float(W[:, i] @ Dj[:, 1 + i]) - dc[j] / c * float(Z[:, i] @ Z[:, i]) for i in range(n_z)])
        grad[j] = 0.5 * (quad + n * dc[j] / c + probes)
    return {"grad": grad, "alpha": alpha, "W": W}
