// regularize.cu -- boundary-regularised kernel kappa_R ("It is possible
// to smoothen the inner or outer boundaries") and the near-field correction of the inner part.
//
// kappa_R(r), r = ||x~|| in a window's scaled coordinates (f4):
//   r <= eps_I              T_I(r): the polynomial of degree 2p-1 matching kappa's derivatives of
//                           orders 0..p-1 at r = +-eps_I (kappa extended evenly to r < 0).  It is even,
//                           so it is found here as T_I(r) = sum_{k<p} a_k (r/eps_I)^{2k} from the p
//                           conditions at +eps_I (the mirrored ones then hold by symmetry, and the
//                           Hermite interpolant is unique);
//   eps_I < r <= 1/2-eps_B  kappa(r);
//   1/2-eps_B < r <= 1/2    T_B(r) = sum_{k<2p} c_k t^k, t = (r - (1/2 - eps_B)) / eps_B: kappa's
//                           derivatives 0..p-1 at t = 0, the constant kappa(1/2) (derivatives 0) at t = 1;
//   r > 1/2                 kappa(1/2).
// The samples kappa_R(l/N) feed eq. (3.2) unchanged (setup_kernels.cu k_cos_dft_axis).  Scaled points
// lie in the ball of radius 1/4 - eps_B/2, so T_B never replaces a kernel value the product uses;
// T_I does for pairs closer than eps_I, and k_near_field adds sum_j (kappa - T_I)(r_ij) v_j back.
// kappa^der (the ell-derivative kernel, eq. 2.3) is regularised the same way.
#include <cuda_runtime.h>

#include <algorithm>

#include "akm_internal.cuh"

namespace akm {

// f^(q)(r), q < p, of f(r) = Q(r) e^{alpha r + beta r^2}: Gaussian alpha = 0, beta = -1/(2 ell^2),
// Matern alpha = -1/ell, beta = 0; Q = 1 (kappa), r^2/ell^3 (Gaussian kappa^der), r/ell^2 (Matern
// kappa^der).  Each derivative maps Q to Q' + (alpha + 2 beta r) Q.
__device__ void radial_derivs(int family, int deriv, double ell, double r, int p, double* out) {
  constexpr int L = kRegMaxP + 4;
  double Q[L], Qn[L];
  for (int k = 0; k < L; ++k) Q[k] = 0.0;
  double alpha, beta;
  if (family == 0) {
    alpha = 0.0;
    beta = -0.5 / (ell * ell);
    if (deriv) Q[2] = 1.0 / (ell * ell * ell); else Q[0] = 1.0;
  } else {
    alpha = -1.0 / ell;
    beta = 0.0;
    if (deriv) Q[1] = 1.0 / (ell * ell); else Q[0] = 1.0;
  }
  const double e = exp(alpha * r + beta * r * r);
  for (int q = 0; q < p; ++q) {
    double v = 0.0;
    for (int k = L - 1; k >= 0; --k) v = v * r + Q[k];
    out[q] = v * e;
    for (int k = 0; k < L; ++k) {
      double t = (k + 1 < L ? (k + 1) * Q[k + 1] : 0.0) + alpha * Q[k];
      if (k >= 1) t += 2.0 * beta * Q[k - 1];
      Qn[k] = t;
    }
    for (int k = 0; k < L; ++k) Q[k] = Qn[k];
  }
}

// Gaussian elimination with partial pivoting on a small dense system (n <= kRegMaxP), in place.
__device__ void small_solve(int n, double* A /* n x n row-major */, double* b) {
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int i = c + 1; i < n; ++i)
      if (fabs(A[i * n + c]) > fabs(A[piv * n + c])) piv = i;
    if (piv != c) {
      for (int k = 0; k < n; ++k) {
        const double t = A[c * n + k];
        A[c * n + k] = A[piv * n + k];
        A[piv * n + k] = t;
      }
      const double t = b[c];
      b[c] = b[piv];
      b[piv] = t;
    }
    for (int i = c + 1; i < n; ++i) {
      const double f = A[i * n + c] / A[c * n + c];
      for (int k = c; k < n; ++k) A[i * n + k] -= f * A[c * n + k];
      b[i] -= f * b[c];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= A[i * n + k] * b[k];
    b[i] = s / A[i * n + i];
  }
}

// d^q/ds^q s^j at s = 1: j! / (j - q)! (0 if q > j)
__device__ __forceinline__ double falling(int j, int q) {
  if (q > j) return 0.0;
  double v = 1.0;
  for (int t = 0; t < q; ++t) v *= (double)(j - t);
  return v;
}

// One thread per operator (0: kappa, 1: kappa^der) of one window.
// out[op * kRegStride + 0 .. p-1]:          a_k of T_I (powers (r/eps_I)^{2k});
// out[op * kRegStride + kRegMaxP .. +2p-1]: c_k of T_B (powers t^k).
__global__ void k_reg_coef(int family, double ell, double eps_I, double eps_B, int p, double* __restrict__ out) {
  const int op = threadIdx.x;
  if (op >= 2 || p <= 0) return;
  double* o = out + op * kRegStride;
  double f[kRegMaxP];
  double A[kRegMaxP * kRegMaxP], b[kRegMaxP];
  if (eps_I > 0.0) {
    // sum_k a_k d^q/ds^q s^{2k} |_{s=1} = eps_I^q f^(q)(eps_I),  q < p
    radial_derivs(family, op, ell, eps_I, p, f);
    double sc = 1.0;
    for (int q = 0; q < p; ++q) {
      for (int k = 0; k < p; ++k) A[q * p + k] = falling(2 * k, q);
      b[q] = sc * f[q];
      sc *= eps_I;
    }
    small_solve(p, A, b);
    for (int k = 0; k < p; ++k) o[k] = b[k];
    // Near-field weight (kappa - T_I)(r), r < eps_I, as one polynomial in t = s (Matern) or s^2
    // (Gaussian), s = r / eps_I: kappa = pre * t^op * exp(-x t) (x = eps_I/ell resp. eps_I^2/(2 ell^2);
    // pre = 1 for kappa, eps_I/ell^2 resp. eps_I^2/ell^3 for kappa^der) expanded in its Taylor series,
    // truncated where the tail bound pre x^(J+1)/(J+1)! e^x (t <= 1) drops below 1e-17, minus T_I.
    // nf[0] = degree, or -1 where the series is too long or x > 1.5 (cancellation): the kernel then
    // evaluates kappa directly.
    double* nf = o + kRegNfOff;
    const double x = (family == 0) ? eps_I * eps_I / (2.0 * ell * ell) : eps_I / ell;
    const double pre = (op == 0) ? 1.0 : ((family == 0) ? eps_I * eps_I / (ell * ell * ell) : eps_I / (ell * ell));
    const int tdeg = (family == 0) ? p - 1 : 2 * p - 2;  // degree of T_I in t
    for (int k = 0; k < kRegNfLen; ++k) nf[k] = 0.0;
    nf[0] = -1.0;
    if (x <= 1.5) {
      const double ex = exp(x);
      double term = pre;  // pre x^j / j!
      int J = 0;
      double c[kRegNfLen - 1];
      for (int k = 0; k < kRegNfLen - 1; ++k) c[k] = 0.0;
      bool ok = false;
      for (; J + op < kRegNfLen - 1; ++J) {
        c[J + op] = ((J & 1) ? -term : term);
        const double next = term * x / (double)(J + 1);
        if (next * ex < 1e-17) { ok = true; break; }
        term = next;
      }
      if (ok) {
        const int deg = max(J + op, tdeg);
        for (int k = 0; k < p; ++k) c[(family == 0) ? k : 2 * k] -= o[k];
        nf[0] = (double)deg;
        for (int k = 0; k <= deg; ++k) nf[1 + k] = c[k];
      }
    }
  }
  if (eps_B > 0.0) {
    // t = 0: c_q = eps_B^q f^(q)(1/2 - eps_B) / q!;  t = 1: value f(1/2), derivatives 0
    radial_derivs(family, op, ell, 0.5 - eps_B, p, f);
    double sc = 1.0, fact = 1.0;
    double* c = o + kRegMaxP;
    for (int q = 0; q < p; ++q) {
      if (q > 0) fact *= (double)q;
      c[q] = sc * f[q] / fact;
      sc *= eps_B;
    }
    double fb;
    radial_derivs(family, op, ell, 0.5, 1, &fb);
    for (int q = 0; q < p; ++q) {
      double rhs = (q == 0) ? fb : 0.0;
      for (int k = 0; k < p; ++k) rhs -= c[k] * falling(k, q);
      for (int k = 0; k < p; ++k) A[q * p + k] = falling(p + k, q);
      b[q] = rhs;
    }
    small_solve(p, A, b);
    for (int k = 0; k < p; ++k) c[p + k] = b[k];
  }
}

cudaError_t launch_reg_coef(int family, double ell_eff, double eps_I, double eps_B, int p, double* coef, cudaStream_t s) {
  k_reg_coef<<<1, 32, 0, s>>>(family, ell_eff, eps_I, eps_B, p, coef);
  return cudaGetLastError();
}

__device__ __forceinline__ double kernel_plain(int family, int deriv, double ell, double r) {
  if (family == 0) {
    const double k = exp(-r * r / (2.0 * ell * ell));
    return deriv ? r * r / (ell * ell * ell) * k : k;
  }
  const double k = exp(-r / ell);
  return deriv ? r / (ell * ell) * k : k;
}

__device__ __forceinline__ double reg_inner(const double* __restrict__ a, int p, double s2) {
  double v = a[p - 1];
  for (int k = p - 2; k >= 0; --k) v = fma(v, s2, a[k]);
  return v;
}

// kappa_R(r) at the nodes l/N of I_N^d (the samples of eq. 3.2), regularised (see the file comment)
__global__ void k_kernel_samples_reg(int family, int d, int N, double ell, int deriv, double eps_I, double eps_B,
                                     int p, const double* __restrict__ coef, double* __restrict__ out) {
  long long total = 1;
  for (int t = 0; t < d; ++t) total *= N;
  const double* a = coef + deriv * kRegStride;
  const double* c = a + kRegMaxP;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long rem = idx;
    double rr = 0.0;
    for (int t = 0; t < d; ++t) {
      const int li = (int)(rem % N) - N / 2;
      rem /= N;
      const double x = (double)li / (double)N;
      rr += x * x;
    }
    const double r = sqrt(rr);
    double v;
    if (eps_I > 0.0 && r <= eps_I) {
      v = reg_inner(a, p, rr / (eps_I * eps_I));
    } else if (eps_B > 0.0 && r > 0.5) {
      double cs = 0.0;
      for (int k = 2 * p - 1; k >= 0; --k) cs = cs + c[k];  // T_B(t = 1)
      v = cs;
    } else if (eps_B > 0.0 && r > 0.5 - eps_B) {
      const double t = (r - (0.5 - eps_B)) / eps_B;
      double cs = c[2 * p - 1];
      for (int k = 2 * p - 2; k >= 0; --k) cs = fma(cs, t, c[k]);
      v = cs;
    } else {
      v = kernel_plain(family, deriv, ell, r);
    }
    out[idx] = v;
  }
}

cudaError_t launch_kernel_samples_reg(int family, int d, int N, double ell_eff, int deriv, double eps_I, double eps_B,
                                      int p, const double* coef, double* out, cudaStream_t s) {
  long long total = 1;
  for (int t = 0; t < d; ++t) total *= N;
  const int blocks = (int)((total + 255) / 256);
  k_kernel_samples_reg<<<blocks, 256, 0, s>>>(family, d, N, ell_eff, deriv, eps_I, eps_B, p, coef, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ near-field correction
// One CTA per interpolation item (<= 128 target points of one bin), each warp on its own 32 targets:
// it lists, in a fixed order, the (cell, class) point ranges of every grid cell whose box comes
// closer than eps_I to the bounding box of its targets (ballot compaction over the candidate cells),
// then streams those source points through a warp-private slice of shared memory, 32 at a time
// (scaled coordinates and the rc values of their rows of the bin-sorted copy of V).  Each lane
// accumulates, for its target, sum_{r_ij < eps_I} (kappa - T_I)(r_ij) v_j for kappa (slot K) and
// kappa^der / c_w (slot L) -- the weights as one series in r (k_reg_coef) where it converges fast,
// else kappa evaluated directly -- and adds it to the window's partial output (written by the
// interpolation before, read by the epilogue after).
constexpr int kNfThreads = 128;
constexpr int kNfMaxRc = 12;

__global__ void k_sort_v(long long n, int P, int r, const int* __restrict__ perm, const double* __restrict__ V,
                         long long ldv, double* __restrict__ Vs) {
  const long long total = (long long)P * n * r;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long wp = idx / r;
    const int c = (int)(idx - wp * r);
    Vs[idx] = V[(long long)perm[wp] * ldv + c];
  }
}

// Warp-independent: each warp owns 32 consecutive targets of its CTA's item, lists the candidate
// cell ranges itself and streams the candidates through a warp-private slice of shared memory
// (__syncwarp only: no CTA barrier, a warp with no targets left is done).
constexpr int kNfWarps = kNfThreads / 32;
constexpr int kNfWarpRanges = 256;
constexpr int kNfUnroll = 4;
constexpr int kNfCoef = 28;  // series coefficients 0..22, zero-padded to 27 (Horner in steps of 4)

// sqrt(x) for x in [0, 1]: rsqrt.approx, one Newton step, then a residual correction (t + y (x - t^2)/2)
// to within an ulp; x is moved off 0 by 1e-280 (t(0) = 1e-140 instead of 0: below rounding in the weight)
__device__ __forceinline__ double sqrt_unit(double x) {
  x += 1e-280;
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x, y * y, 1.5);
  const double t = x * y;
  return fma(0.5 * y, fma(-t, t, x), t);
}
// HAS_L: the kappa^der operator is applied too (its 12 accumulators cost registers otherwise).
template <bool HAS_L>
__global__ void __launch_bounds__(kNfThreads, HAS_L ? 3 : 5) k_near_field(
    const WinTable* __restrict__ tabp, const WorkItem* __restrict__ items, const int2* __restrict__ cell_tab,
    const long long* __restrict__ cell_off, const double* __restrict__ u_sorted, const int* __restrict__ perm,
    const double* __restrict__ Vs, long long n, int r0, int rc, int r_total, int ops, int slotK, int slotL, int family,
    double ell, double eps_I, int p, const double* __restrict__ coef, double* __restrict__ part) {
  __shared__ double su_all[kNfWarps][3][32];
  __shared__ __align__(16) double sv_all[kNfWarps][32 * kNfMaxRc];
  __shared__ double sc_all[kNfWarps][2][kNfCoef];
  __shared__ int rstart_all[kNfWarps][kNfWarpRanges], rpre_all[kNfWarps][kNfWarpRanges + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const WorkItem it = items[blockIdx.x];
  if (wid * 32 >= it.count) return;
  double (*su)[32] = su_all[wid];
  double* sv = sv_all[wid];
  int* rstart = rstart_all[wid];
  int* rpre = rpre_all[wid];
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[it.win];
  const int w = it.win;
  const double* uw = u_sorted + (long long)w * 3 * n;
  const int* pw = perm + (long long)w * n;
  const double* vw = Vs + (long long)w * n * r_total + r0;
  const double inv_ng = 1.0 / (double)tab.n_g;
  const double ell_eff = ell * g.scale * inv_ng;  // ell / c_w
  const double inv_c = g.scale * inv_ng;
  const double E = eps_I * (double)tab.n_g;       // eps_I in grid units
  const double E2 = E * E;
  const double inv_eps2 = 1.0 / (eps_I * eps_I);
  const double* aK = coef + (long long)w * 2 * kRegStride;
  const double* aL = aK + kRegStride;
  const bool active = wid * 32 + lane < it.count;
  const int pos = it.start + (active ? wid * 32 + lane : 0);
  double ut[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) ut[a] = (a >= 3 - g.d) ? uw[(long long)a * n + pos] : 0.0;
  double accK[kNfMaxRc], accL[HAS_L ? kNfMaxRc : 1];
#pragma unroll
  for (int c = 0; c < kNfMaxRc; ++c) accK[c] = 0.0;
#pragma unroll
  for (int c = 0; c < (HAS_L ? kNfMaxRc : 1); ++c) accL[c] = 0.0;
  // the near-field series of both operators (k_reg_coef), if usable, in warp-private shared memory
  const int degK = (int)aK[kRegNfOff], degL = HAS_L ? (int)aL[kRegNfOff] : 0;
  const bool poly = degK >= 0 && degL >= 0;
  const int degK4 = (degK + 3) & ~3, degL4 = (degL + 3) & ~3;  // Horner runs in steps of 4
  double (*sc)[kNfCoef] = sc_all[wid];
  if (lane < kNfCoef) {
    sc[0][lane] = (lane < kRegNfLen - 1) ? aK[kRegNfOff + 1 + lane] : 0.0;
    if constexpr (HAS_L) sc[1][lane] = (lane < kRegNfLen - 1) ? aL[kRegNfOff + 1 + lane] : 0.0;
  }
  const double inv_E2 = 1.0 / E2;
  // candidate cells: those whose box comes closer than eps_I to the bounding box of this warp's
  // targets (cell c of axis a covers u - (box_lo + m - 1) in [c, c + 1)), in a fixed order; the
  // index window is widened by one cell and the gap test given a relative slack of 1e-12, so rounding
  // can only add candidates (the per-pair test q2 < E2 decides)
  int lo[3], ext[3];
  double tlo[3], thi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool real = a >= 3 - g.d;
    double mn = active ? ut[a] : 1e300, mx = active ? ut[a] : -1e300;
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const double off = (double)(g.box_lo[a] + tab.m - 1);
    tlo[a] = real ? mn - off : 0.0;
    thi[a] = real ? mx - off : 0.0;
    lo[a] = real ? max(0, (int)floor(tlo[a] - E) - 1) : 0;
    const int hi = real ? min(g.ncell[a] - 1, (int)floor(thi[a] + E) + 1) : 0;
    ext[a] = max(0, hi - lo[a] + 1);
  }
  const double E2s = E2 * (1.0 + 1e-12);
  const int total = ext[0] * ext[1] * ext[2];
  for (int q0 = 0; q0 < total;) {
    // the (start, count) ranges of the next cells closer than eps_I to the bin (ballot compaction)
    int count = 0, acc = 0, q = q0;
    for (; q < total && count <= kNfWarpRanges - 64; q += 32) {
      const int qq = q + lane;
      int cnt[2] = {0, 0}, cs[2] = {0, 0};
      bool near = false;
      if (qq < total) {
        const int cc[3] = {lo[0] + qq / (ext[1] * ext[2]), lo[1] + (qq / ext[2]) % ext[1], lo[2] + qq % ext[2]};
        double gap2 = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double gp =
              (a >= 3 - g.d) ? fmax(0.0, fmax(tlo[a] - (double)(cc[a] + 1), (double)cc[a] - thi[a])) : 0.0;
          gap2 += gp * gp;
        }
        near = gap2 < E2s;
        if (near) {
          const long long slot = cell_off[w] + 2 * (((long long)cc[0] * g.ncell[1] + cc[1]) * g.ncell[2] + cc[2]);
          const int2 a0 = cell_tab[slot], a1 = cell_tab[slot + 1];
          cs[0] = a0.x; cnt[0] = a0.y; cs[1] = a1.x; cnt[1] = a1.y;
        }
      }
      for (int cls = 0; cls < 2; ++cls) {
        const bool has = near && cnt[cls] > 0;
        const unsigned bal = __ballot_sync(0xffffffffu, has);
        const int before = __popc(bal & ((1u << lane) - 1u));
        int v = has ? cnt[cls] : 0;  // inclusive running sum of the counts in lane order
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (has) {
          rstart[count + before] = cs[cls];
          rpre[count + before + 1] = acc + v;
        }
        count += __popc(bal);
        acc += __shfl_sync(0xffffffffu, v, 31);
      }
    }
    if (lane == 0) rpre[0] = 0;
    __syncwarp();
    q0 = q;
    const int nr = count, ncand = acc;
    for (int f0 = 0; f0 < ncand; f0 += 32) {
      const int cnt = min(32, ncand - f0);
      if (lane < cnt) {
        const int f = f0 + lane;
        int a = 0, b = nr - 1;  // range with rpre[a] <= f < rpre[a + 1]
        while (a < b) {
          const int mid = (a + b + 1) >> 1;
          if (rpre[mid] <= f) a = mid; else b = mid - 1;
        }
        const int sp = rstart[a] + (f - rpre[a]);
#pragma unroll
        for (int t = 0; t < 3; ++t) su[t][lane] = (t >= 3 - g.d) ? uw[(long long)t * n + sp] : 0.0;
#pragma unroll
        for (int c = 0; c < kNfMaxRc; ++c) sv[lane * kNfMaxRc + c] = (c < rc) ? vw[(long long)sp * r_total + c] : 0.0;
      } else {  // padding sources: far away (weight 0 for every target), zero values
#pragma unroll
        for (int t = 0; t < 3; ++t) su[t][lane] = 1e150;
#pragma unroll
        for (int c = 0; c < kNfMaxRc; ++c) sv[lane * kNfMaxRc + c] = 0.0;
      }
      __syncwarp();
      // kNfUnroll sources at a time (independent weight chains); every lane takes part, lanes without
      // a target or out of range with q2 = E2 (weight 0), and groups no lane needs are skipped
      for (int j0 = 0; j0 < cnt; j0 += kNfUnroll) {
        double q2[kNfUnroll];
        bool in[kNfUnroll], any = false;
#pragma unroll
        for (int u = 0; u < kNfUnroll; ++u) {
          const int j = j0 + u;  // < 32: rows cnt..31 hold padding sources
          const double d0 = ut[0] - su[0][j], d1 = ut[1] - su[1][j], d2 = ut[2] - su[2][j];
          q2[u] = fma(d2, d2, fma(d1, d1, d0 * d0));
          in[u] = active && q2[u] < E2;
          any |= in[u];
        }
        if (!__any_sync(0xffffffffu, any)) continue;
        double wK[kNfUnroll], wL[kNfUnroll];
        if (poly) {
          double t[kNfUnroll];
#pragma unroll
          for (int u = 0; u < kNfUnroll; ++u) {
            const double s2 = in[u] ? q2[u] * inv_E2 : 1.0;  // < 1 where the weight is used
            t[u] = (family == 0) ? s2 : sqrt_unit(s2);
            wK[u] = sc[0][degK4];
            if constexpr (HAS_L) wL[u] = sc[1][degL4];
          }
          // Horner from the padded degree (the coefficients past the degree are zero: exact)
          for (int k = degK4 - 4; k >= 0; k -= 4) {
#pragma unroll
            for (int kk = 3; kk >= 0; --kk) {
              const double c = sc[0][k + kk];
#pragma unroll
              for (int u = 0; u < kNfUnroll; ++u) wK[u] = fma(wK[u], t[u], c);
            }
          }
          if constexpr (HAS_L) {
            for (int k = degL4 - 4; k >= 0; k -= 4) {
#pragma unroll
              for (int kk = 3; kk >= 0; --kk) {
                const double c = sc[1][k + kk];
#pragma unroll
                for (int u = 0; u < kNfUnroll; ++u) wL[u] = fma(wL[u], t[u], c);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < kNfUnroll; ++u) {
            wK[u] = in[u] ? wK[u] : 0.0;
            if constexpr (HAS_L) wL[u] = in[u] ? wL[u] * inv_c : 0.0;
          }
        } else {
#pragma unroll
          for (int u = 0; u < kNfUnroll; ++u) {
            wK[u] = 0.0;
            if constexpr (HAS_L) wL[u] = 0.0;
            if (in[u]) {
              const double r = sqrt(q2[u]) * inv_ng;
              const double s2 = r * r * inv_eps2;
              wK[u] = kernel_plain(family, 0, ell_eff, r) - reg_inner(aK, p, s2);
              if constexpr (HAS_L) wL[u] = (kernel_plain(family, 1, ell_eff, r) - reg_inner(aL, p, s2)) * inv_c;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kNfUnroll; ++u) {  // all kNfMaxRc columns (zero-padded past rc)
          const double2* vrow = reinterpret_cast<const double2*>(sv + (j0 + u) * kNfMaxRc);
#pragma unroll
          for (int c2 = 0; c2 < kNfMaxRc / 2; ++c2) {
            const double2 v = vrow[c2];
            accK[2 * c2] = fma(wK[u], v.x, accK[2 * c2]);
            accK[2 * c2 + 1] = fma(wK[u], v.y, accK[2 * c2 + 1]);
            if constexpr (HAS_L) {
              accL[2 * c2] = fma(wL[u], v.x, accL[2 * c2]);
              accL[2 * c2 + 1] = fma(wL[u], v.y, accL[2 * c2 + 1]);
            }
          }
        }
      }
      __syncwarp();
    }
  }
  if (!active) return;
  const long long i = pw[pos];
  double* out = part + (((long long)w * n + i) * ops) * r_total + r0;
#pragma unroll
  for (int c = 0; c < kNfMaxRc; ++c) {
    if (c < rc) {
      if (slotK >= 0) out[(long long)slotK * r_total + c] += accK[c];
      if constexpr (HAS_L) out[(long long)slotL * r_total + c] += accL[HAS_L ? c : 0];
    }
  }
}

cudaError_t launch_near_field(const WinTable* dtab, const WorkItem* items, int n_items, const int2* cell_tab,
                              const long long* cell_off, const double* u_sorted, const int* perm, const double* V,
                              long long ldv, double* Vs, long long n, int P, int r, int ops, int slotK, int slotL,
                              int family, double ell, double eps_I, int p, const double* coef, double* part,
                              cudaStream_t s) {
  if (n_items <= 0) return cudaSuccess;
  {
    const long long total = (long long)P * n * r;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 32);
    k_sort_v<<<blocks, 256, 0, s>>>(n, P, r, perm, V, ldv, Vs);
  }
  for (int r0 = 0; r0 < r; r0 += kNfMaxRc) {
    const int rc = (r - r0 < kNfMaxRc) ? r - r0 : kNfMaxRc;
    auto kern = (slotL >= 0) ? k_near_field<true> : k_near_field<false>;
    kern<<<n_items, kNfThreads, 0, s>>>(dtab, items, cell_tab, cell_off, u_sorted, perm, Vs, n, r0, rc, r, ops, slotK,
                                        slotL, family, ell, eps_I, p, coef, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int near_field_launches(int r) { return 1 + (r + kNfMaxRc - 1) / kNfMaxRc; }

}  // namespace akm
