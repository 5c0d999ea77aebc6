"""AAFN preconditioner.  TEST INFRASTRUCTURE ONLY.

PAPER.md §2.3: "the AFN preconditioner identifies k landmark points ... This process
adaptively divides the matrix into a 2x2 block structure, where the (1,1) block corresponds to the
landmark points, and the (2,2) block corresponds to the remaining data.  The preconditioner M is
then constructed by the Cholesky factorization of the (1,1) block and the approximate inverse of
the Schur complement.  For additive kernels, we apply farthest point sampling (FPS) to select the
landmark points from each feature window and then merge the data indices of these selections to
form the (1,1) block."  §5 fixes the landmark budget; the adaptive rank
estimate of the cited AFN is not reproduced (SPEC aafn-precond DESIGN DECISIONS).

Written out (reading R15):
  * fps(points, k): greedy maximin; seed = the point farthest from the window centroid, then the
    point maximising the minimum distance to the picks; ties -> lowest index.
  * landmarks = union of the per-window picks, deduplicated in pick order (window 0's picks first).
  * with the rows permuted [landmarks; others], K^ = [K11 K12; K21 K22], K11 = L11 L11^T (Cholesky),
    Schur complement S = K22 - K21 K11^{-1} K12, approximated through a sparse lower-triangular
    G with G S G^T ~ I (FSAI): row a (in the natural order of the non-landmark points) has the
    pattern P_a = {a} and its fill-1 nearest non-landmark predecessors (smaller index) under the
    summed windowed Euclidean distance; g = S[P_a, P_a]^{-1} e_a, G[a, P_a] = g / sqrt(g_a).
  * M = U U^T with U = [L11, 0; K21 L11^{-T}, G^{-1}], so
        M^{-1} = U^{-T} U^{-1},  log det M = 2 sum log diag L11 - 2 sum log diag G,
        U^{-1} [t1; t2] = [L11^{-1} t1;  G (t2 - K21 L11^{-T} L11^{-1} t1)].
  * The preconditioned Krylov methods run on the symmetric S_op = U^{-1} K^ U^{-T} (SPEC S:385,
    "split-preconditioned operator"): PCG for K^ x = y is CG on S_op x^ = U^{-1} y, x = U^{-T} x^.
Dense matrices throughout: n up to a few thousand.
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

from .fourier import kernel_radial


def khat_dense(X, windows, family, theta, rows=None, cols=None):
    """Entries of K^ = sigma_f^2 sum_w K_w + sigma_eps^2 I (eqs. 1.1, 2.1)."""
    X = np.asarray(X, dtype=np.float64)
    rows = np.arange(X.shape[0]) if rows is None else np.asarray(rows)
    cols = np.arange(X.shape[0]) if cols is None else np.asarray(cols)
    sf, ell, se = theta
    K = np.zeros((rows.size, cols.size))
    for win in windows:
        A = X[np.ix_(rows, list(win))]
        B = X[np.ix_(cols, list(win))]
        rr = ((A[:, None, :] - B[None, :, :]) ** 2).sum(axis=2)
        K += kernel_radial(family, rr, ell)
    K *= sf * sf
    K += se * se * (rows[:, None] == cols[None, :])
    return K


def fps(points, k):
    """Farthest point sampling (greedy maximin)."""
    P = np.asarray(points, dtype=np.float64)
    n = P.shape[0]
    k = min(k, n)
    c = P.mean(axis=0)
    d0 = ((P - c) ** 2).sum(axis=1)
    first = int(np.flatnonzero(d0 == d0.max())[0])
    picks = [first]
    dmin = ((P - P[first]) ** 2).sum(axis=1)
    dmin[first] = -1.0
    while len(picks) < k:
        j = int(np.flatnonzero(dmin == dmin.max())[0])
        picks.append(j)
        dmin = np.minimum(dmin, ((P - P[j]) ** 2).sum(axis=1))
        dmin[picks] = -1.0
    return picks


def landmarks(X, windows, k_per_window):
    seen, out = set(), []
    for win in windows:
        for j in fps(np.asarray(X)[:, list(win)], k_per_window):
            if j not in seen:
                seen.add(j)
                out.append(j)
    return np.array(out, dtype=np.int64)


class Aafn:
    def __init__(self, X, windows, family, theta, k_per_window, fill):
        X = np.asarray(X, dtype=np.float64)
        n = X.shape[0]
        self.n = n
        self.lm = landmarks(X, windows, k_per_window)
        mask = np.ones(n, dtype=bool)
        mask[self.lm] = False
        self.rest = np.flatnonzero(mask)                      # natural order of the non-landmark points
        K11 = khat_dense(X, windows, family, theta, self.lm, self.lm)
        self.L11 = np.linalg.cholesky(K11)
        K21 = khat_dense(X, windows, family, theta, self.rest, self.lm)
        self.Phi = solve_triangular(self.L11, K21.T, lower=True).T    # K21 L11^{-T}
        m = self.rest.size
        self.G = np.zeros((m, m))
        # FSAI of S = K22 - Phi Phi^T on the nearest-predecessor pattern
        Xr = X[self.rest]
        for a in range(m):
            if a > 0 and fill > 1:
                dist = np.zeros(a)
                for win in windows:
                    dist += np.sqrt(((Xr[:a][:, list(win)] - Xr[a, list(win)]) ** 2).sum(axis=1))
                nb = np.argsort(dist, kind="stable")[:fill - 1]
                pat = np.concatenate([np.sort(nb), [a]])
            else:
                pat = np.array([a])
            Spp = (khat_dense(X, windows, family, theta, self.rest[pat], self.rest[pat])
                   - self.Phi[pat] @ self.Phi[pat].T)
            e = np.zeros(pat.size)
            e[-1] = 1.0
            g = np.linalg.solve(Spp, e)
            self.G[a, pat] = g / np.sqrt(g[-1])
        self.logdet = 2.0 * np.sum(np.log(np.diag(self.L11))) - 2.0 * np.sum(np.log(np.diag(self.G)))

    def U_inv(self, T):
        """U^{-1} T (T: n x r in the user's row order; result in the same order)."""
        T = np.asarray(T, dtype=np.float64).reshape(self.n, -1)
        y1 = solve_triangular(self.L11, T[self.lm], lower=True)
        y2 = self.G @ (T[self.rest] - self.Phi @ y1)
        out = np.empty_like(T)
        out[self.lm], out[self.rest] = y1, y2
        return out

    def U_invT(self, Y):
        """U^{-T} Y: w2 = G^T y2, w1 = L11^{-T} (y1 - Phi^T w2)."""
        Y = np.asarray(Y, dtype=np.float64).reshape(self.n, -1)
        w2 = self.G.T @ Y[self.rest]
        w1 = solve_triangular(self.L11.T, Y[self.lm] - self.Phi.T @ w2, lower=False)
        out = np.empty_like(Y)
        out[self.lm], out[self.rest] = w1, w2
        return out

    def apply_inverse(self, V):
        return self.U_invT(self.U_inv(V))

    def assemble_M(self):
        """M = U U^T densely (for tests): U = U^{-1} inverted column by column."""
        Uinv = self.U_inv(np.eye(self.n))
        U = np.linalg.inv(Uinv)
        return U @ U.T


def objective_aafn(apply_K, y, Z, pre, cg_iters, lanczos_steps):
    """eq. (1.4) with M = AAFN (reading R15): CG and Lanczos on S_op = U^{-1} K^ U^{-T},
    column 0 = U^{-1} y, probes z_i unchanged; log det M from the factors.  Reuses the diagonal-M
    driver of oracle/krylov.py with M = I on S_op."""
    from . import krylov
    yh = pre.U_inv(np.asarray(y, dtype=np.float64)[:, None])[:, 0]
    S = lambda B: pre.U_inv(apply_K(pre.U_invT(B)))
    out = krylov.objective_diag(S, yh, Z, np.ones(yh.size), cg_iters, lanczos_steps)
    n = yh.size
    out["logdetM"] = pre.logdet
    out["Z"] = 0.5 * (out["quad"] + pre.logdet + out["slq"] + n * np.log(2.0 * np.pi))
    x = pre.U_invT(out["x"][:, None])[:, 0]
    out["x"] = x
    out["cg_relres_true"] = float(np.linalg.norm(y - apply_K(x[:, None])[:, 0]) / np.linalg.norm(y))
    return out


def gradient_aafn(apply_K, apply_dK, y, Z, pre, cg_iters):
    """Gradient of Z~ with AAFN solves (SPEC krylov-estimators DESIGN DECISIONS: eq. (div)'s
    control-variate term needs dM/dtheta, which AAFN does not define, so the plain Hutchinson form
    with preconditioned solves is used -- reading R15):
        dZ~/dtheta_j ~= 1/2 ( -alpha^T dKhat_j alpha + (1/n_z) sum_i (Khat^{-1} z_i)^T dKhat_j z_i ),
    every Khat^{-1} b by CG on S_op = U^{-1} Khat U^{-T} from U^{-1} b, mapped back by U^{-T}."""
    from . import krylov
    y = np.asarray(y, dtype=np.float64)
    Z = np.asarray(Z, dtype=np.float64)
    S = lambda B: pre.U_inv(apply_K(pre.U_invT(B)))

    def solve(b):
        xh, _ = krylov.pcg(S, pre.U_inv(b[:, None])[:, 0], cg_iters)
        return pre.U_invT(xh[:, None])[:, 0]

    alpha = solve(y)
    W = np.stack([solve(Z[:, i]) for i in range(Z.shape[1])], axis=1)
    D = apply_dK(np.column_stack([alpha, Z]))
    grad = {j: 0.5 * (-float(alpha @ Dj[:, 0]) + np.mean([float(W[:, i] @ Dj[:, 1 + i]) for i in range(Z.shape[1])]))
            for j, Dj in D.items()}
    return {"grad": grad, "alpha": alpha, "W": W}
