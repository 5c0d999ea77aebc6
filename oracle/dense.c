/*
 * oracle/dense.c -- TEST INFRASTRUCTURE ONLY (never linked into the product path).
 *
 * Plain float64 dense direct sums of the regularized additive kernel products
 * that the NFFT fast summation approximates.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * What it computes (PAPER.md = P):
 *   kernels (eq. 1.1, P:22-26 / eq. 2.2), sub-kernel without sigma_f^2:
 *       Gaussian  kappa(r) = exp(-||r||^2 / (2 ell^2))
 *       Matern1/2 kappa(r) = exp(-||r|| / ell)
 *   ell-derivative kernels (eq. 2.3):
 *       Gaussian  kappa_der(r) = ||r||^2 / ell^3 * kappa(r)
 *       Matern1/2 kappa_der(r) = ||r||   / ell^2 * kappa(r)
 *   additive kernel (eq. 2.1) over disjoint windows W_w:
 *       K = sigma_f^2 sum_w K_w,  Khat = K + sigma_eps^2 I
 *   products, for every requested row i and column c:
 *       Y[i,c]      = sigma_f^2 sum_w sum_j kappa(x_i^W - x_j^W) V[j,c] + sigma_eps^2 V[i,c]
 *       dY_ell[i,c] = sigma_f^2 sum_w sum_j kappa_der(x_i^W - x_j^W) V[j,c]
 *       dY_sf[i,c]  = 2 sigma_f sum_w sum_j kappa(x_i^W - x_j^W) V[j,c]      (d Khat / d sigma_f)
 *       dY_se[i,c]  = 2 sigma_eps V[i,c]                                       (d Khat / d sigma_eps)
 *   (sigma_f / sigma_eps derivatives: "straightforward"; written out in SPEC S:146.)
 *
 * Coordinates are the user's: no scaling, no periodization.  Loops: rows in parallel
 * (OpenMP), then windows, then j, then columns.  No fast-math.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

enum { ORACLE_GAUSSIAN = 0, ORACLE_MATERN12 = 1 };

/* Returns 0 on success, -1 on bad arguments.  X is n x p row-major (ld = p), V is n x r
 * row-major, outputs are nrows x r row-major; rows == NULL means rows 0..n-1 (nrows = n).
 * Any output pointer may be NULL. */
int oracle_dense_apply(int64_t n, int32_t p, const double* X, int32_t P, const int32_t* win_feat,
                       const int32_t* win_len, int32_t family, double sigma_f, double ell, double sigma_eps,
                       int32_t r, const double* V, int64_t nrows, const int64_t* rows, double* Y, double* dY_ell,
                       double* dY_sf, double* dY_se) {
  if (n < 0 || p <= 0 || P <= 0 || r <= 0 || ell <= 0.0) return -1;
  if (family != ORACLE_GAUSSIAN && family != ORACLE_MATERN12) return -1;
  if (rows == NULL) nrows = n;

#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t q = 0; q < nrows; ++q) {
    const int64_t i = rows ? rows[q] : q;
    double sK[64], sD[64];
    for (int32_t c0 = 0; c0 < r; c0 += 64) {
      const int32_t cn = (r - c0) < 64 ? (r - c0) : 64;
      for (int32_t c = 0; c < cn; ++c) { sK[c] = 0.0; sD[c] = 0.0; }
      int32_t off = 0;
      for (int32_t w = 0; w < P; ++w) {
        const int32_t* feats = win_feat + off;
        const int32_t dw = win_len[w];
        for (int64_t j = 0; j < n; ++j) {
          double rr = 0.0; /* ||x_i^W - x_j^W||^2 */
          for (int32_t t = 0; t < dw; ++t) {
            const double diff = X[i * p + feats[t]] - X[j * p + feats[t]];
            rr += diff * diff;
          }
          double kap, kder;
          if (family == ORACLE_GAUSSIAN) {
            kap = exp(-rr / (2.0 * ell * ell));
            kder = rr / (ell * ell * ell) * kap;
          } else {
            const double rn = sqrt(rr);
            kap = exp(-rn / ell);
            kder = rn / (ell * ell) * kap;
          }
          for (int32_t c = 0; c < cn; ++c) {
            const double v = V[j * r + c0 + c];
            sK[c] += kap * v;
            sD[c] += kder * v;
          }
        }
        off += dw;
      }
      for (int32_t c = 0; c < cn; ++c) {
        const double vi = V[i * r + c0 + c];
        if (Y) Y[q * r + c0 + c] = sigma_f * sigma_f * sK[c] + sigma_eps * sigma_eps * vi;
        if (dY_ell) dY_ell[q * r + c0 + c] = sigma_f * sigma_f * sD[c];
        if (dY_sf) dY_sf[q * r + c0 + c] = 2.0 * sigma_f * sK[c];
        if (dY_se) dY_se[q * r + c0 + c] = 2.0 * sigma_eps * vi;
      }
    }
  }
  return 0;
}

/* Single sub-kernel entry kappa(x - y) (no sigma_f), for pins against SPEC's worked values. */
double oracle_kernel_value(int32_t family, const double* rvec, int32_t d, double ell, int32_t deriv) {
  double rr = 0.0;
  for (int32_t t = 0; t < d; ++t) rr += rvec[t] * rvec[t];
  if (family == ORACLE_GAUSSIAN) {
    const double k = exp(-rr / (2.0 * ell * ell));
    return deriv ? rr / (ell * ell * ell) * k : k;
  }
  const double rn = sqrt(rr);
  const double k = exp(-rn / ell);
  return deriv ? rn / (ell * ell) * k : k;
}
