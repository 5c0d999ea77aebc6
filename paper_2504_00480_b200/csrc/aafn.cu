// aafn.cu -- the AAFN preconditioner (§2.3; reading R15).
//
// "the AFN preconditioner identifies k landmark points ... divides the matrix into a 2x2 block
// structure ... The preconditioner M is then constructed by the Cholesky factorization of the (1,1)
// block and the approximate inverse of the Schur complement.  For additive kernels, we apply farthest
// point sampling (FPS) to select the landmark points from each feature window and then merge the data
// indices of these selections to form the (1,1) block."  With [landmarks; others]:
//     Khat = [K11 K12; K21 K22],  K11 = L11 L11^T,  S = K22 - Phi Phi^T,  Phi = K21 L11^{-T},
//     M = U U^T,  U = [L11, 0; Phi, G^{-1}],  G S G^T ~ I (FSAI; built here with the diagonal pattern,
//     fill = 1: G = diag(S_aa^{-1/2})),
//     log det M = 2 sum log diag L11 - 2 sum log diag G,
//     U^{-1}[t1; t2] = [y1 = L11^{-1} t1;  G (t2 - Phi y1)],
//     U^{-T}[y1; y2] = [L11^{-T} (y1 - Phi^T w2);  w2 = G^T y2].
// The Krylov drivers (plan.cu) run on S_op = U^{-1} Khat U^{-T}.
// Kernel entries are the exact sub-kernels (eqs. 1.1/2.2) in the user's coordinates.
// Every block here is n x R row-major; L11^{-1} (k x k, lower) is formed once so that the per-step
// triangular solves are small dense products.
#include <cuda_runtime.h>

#include <algorithm>

#include "akm_internal.cuh"

namespace akm {

// ---------------------------------------------------------------- farthest point sampling
// Squared Euclidean distance without FMA contraction (the oracle's numpy sum of squares, term order
// 0..d-1), so the argmax decisions are taken on identical doubles.
__device__ __forceinline__ double sqdist(const double* __restrict__ Xc, int nf, long long i, const int* cols, int d,
                                         const double* __restrict__ ref) {
  double s = 0.0;
  for (int t = 0; t < d; ++t) {
    const double e = __dsub_rn(Xc[i * nf + cols[t]], ref[t]);
    s = __dadd_rn(s, __dmul_rn(e, e));
  }
  return s;
}

// (d, i) ordered by larger d, then smaller i
__device__ __forceinline__ bool better(double d, long long i, double bd, long long bi) {
  return d > bd || (d == bd && i < bi);
}

__device__ void block_argmax(double d, long long i, double* sd, long long* si, double* out_d, long long* out_i) {
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, d, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (better(od, oi, d, i)) { d = od; i = oi; }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) { sd[wid] = d; si[wid] = i; }
  __syncthreads();
  if (wid == 0) {
    d = lane < nw ? sd[lane] : -INFINITY;
    i = lane < nw ? si[lane] : (1LL << 62);
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, d, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, i, o);
      if (better(od, oi, d, i)) { d = od; i = oi; }
    }
    if (lane == 0) { *out_d = d; *out_i = i; }
  }
}

struct FpsArgs {
  int nf, d;
  int cols[3];
};

constexpr int kFpsBlocks = 296;
constexpr int kFpsThreads = 256;

// column sums of the window's coordinates (per block, fixed order), for the centroid
__global__ void k_fps_sums(const double* __restrict__ Xc, long long n, FpsArgs a, double* __restrict__ part) {
  __shared__ double sm[3][kFpsThreads];
  double s[3] = {0.0, 0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    for (int t = 0; t < a.d; ++t) s[t] += Xc[i * a.nf + a.cols[t]];
  for (int t = 0; t < 3; ++t) sm[t][threadIdx.x] = s[t];
  __syncthreads();
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int k = 0; k < blockDim.x; ++k) acc += sm[threadIdx.x][k];
    part[blockIdx.x * 3 + threadIdx.x] = acc;
  }
}

// seed distances: dmin[i] = ||x_i - centroid||^2 (the centroid from the block sums, fixed order)
__global__ void k_fps_seed(const double* __restrict__ Xc, long long n, FpsArgs a, const double* __restrict__ part,
                           double* __restrict__ dmin, double* __restrict__ bd, long long* __restrict__ bi) {
  __shared__ double sd[32];
  __shared__ long long si[32];
  __shared__ double c[3];
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int b = 0; b < kFpsBlocks; ++b) acc += part[b * 3 + threadIdx.x];
    c[threadIdx.x] = acc / (double)n;
  }
  __syncthreads();
  double best = -INFINITY;
  long long besti = 1LL << 62;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double dd = sqdist(Xc, a.nf, i, a.cols, a.d, c);
    dmin[i] = dd;
    if (better(dd, i, best, besti)) { best = dd; besti = i; }
  }
  block_argmax(best, besti, sd, si, bd + blockIdx.x, bi + blockIdx.x);
}

// the winner of the previous round becomes pick t; then dmin <- min(dmin, ||x - x_pick||^2), picks
// excluded (-1), and the block argmax of the next round
__global__ void k_fps_step(const double* __restrict__ Xc, long long n, FpsArgs a, int t, int replace, int* __restrict__ picks,
                           double* __restrict__ dmin, const double* __restrict__ bd_in, const long long* __restrict__ bi_in,
                           double* __restrict__ bd, long long* __restrict__ bi) {
  __shared__ double sd[32];
  __shared__ long long si[32];
  __shared__ long long pick;
  __shared__ double ref[3];
  if (threadIdx.x < 32) {
    double d = -INFINITY;
    long long i = 1LL << 62;
    for (int b = threadIdx.x; b < kFpsBlocks; b += 32)
      if (better(bd_in[b], bi_in[b], d, i)) { d = bd_in[b]; i = bi_in[b]; }
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, d, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, i, o);
      if (better(od, oi, d, i)) { d = od; i = oi; }
    }
    if (threadIdx.x == 0) {
      pick = i;
      if (blockIdx.x == 0) picks[t] = (int)i;
    }
  }
  __syncthreads();
  if (threadIdx.x < a.d) ref[threadIdx.x] = Xc[pick * a.nf + a.cols[threadIdx.x]];
  __syncthreads();
  double best = -INFINITY;
  long long besti = 1LL << 62;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double dd = dmin[i];
    if (dd >= 0.0) {
      if (i == pick) {
        dd = -1.0;
      } else {
        const double e = sqdist(Xc, a.nf, i, a.cols, a.d, ref);
        dd = replace ? e : fmin(dd, e);  // after the seed: distances to the picks only
      }
      dmin[i] = dd;
    }
    if (better(dd, i, best, besti)) { best = dd; besti = i; }
  }
  block_argmax(best, besti, sd, si, bd + blockIdx.x, bi + blockIdx.x);
}

size_t fps_scratch_bytes() { return sizeof(double) * kFpsBlocks * 3 + 2 * kFpsBlocks * (sizeof(double) + sizeof(long long)); }

// k picks of one window into picks[0..k); dmin: n doubles; scratch: fps_scratch_bytes()
cudaError_t launch_fps(const double* Xc, long long n, int nf, const int* cols, int d, int k, int* picks, double* dmin,
                       void* scratch, cudaStream_t s) {
  FpsArgs a{nf, d, {cols[0], d > 1 ? cols[1] : 0, d > 2 ? cols[2] : 0}};
  double* part = static_cast<double*>(scratch);
  double* bd0 = part + kFpsBlocks * 3;
  long long* bi0 = reinterpret_cast<long long*>(bd0 + kFpsBlocks);
  double* bd1 = reinterpret_cast<double*>(bi0 + kFpsBlocks);
  long long* bi1 = reinterpret_cast<long long*>(bd1 + kFpsBlocks);
  k_fps_sums<<<kFpsBlocks, kFpsThreads, 0, s>>>(Xc, n, a, part);
  k_fps_seed<<<kFpsBlocks, kFpsThreads, 0, s>>>(Xc, n, a, part, dmin, bd0, bi0);
  for (int t = 0; t < k; ++t) {
    const bool even = (t % 2) == 0;
    k_fps_step<<<kFpsBlocks, kFpsThreads, 0, s>>>(Xc, n, a, t, t == 0, picks, dmin, even ? bd0 : bd1, even ? bi0 : bi1,
                                                  even ? bd1 : bd0, even ? bi1 : bi0);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- kernel entries
struct KhatArgs {
  int P, nf, family;
  double sf2, se2, ell;
  int d[kMaxWin];
  int col0[kMaxWin];  // first compact column of window w (its d columns are consecutive)
};

__device__ __forceinline__ double khat_entry(const double* __restrict__ Xc, const KhatArgs& a, long long i, long long j) {
  double acc = 0.0;
  for (int w = 0; w < a.P; ++w) {
    double rr = 0.0;
    for (int t = 0; t < a.d[w]; ++t) {
      const double e = Xc[i * a.nf + a.col0[w] + t] - Xc[j * a.nf + a.col0[w] + t];
      rr = fma(e, e, rr);
    }
    acc += (a.family == 0) ? exp(-rr / (2.0 * a.ell * a.ell)) : exp(-sqrt(rr) / a.ell);
  }
  return a.sf2 * acc + (i == j ? a.se2 : 0.0);
}

// K11[p][q] = Khat(lm[p], lm[q])
__global__ void k_khat_lm(const double* __restrict__ Xc, KhatArgs a, const int* __restrict__ lm, int k,
                          double* __restrict__ K11) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)k * k;
       idx += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(idx / k), q = (int)(idx % k);
    K11[idx] = khat_entry(Xc, a, lm[p], lm[q]);
  }
}

// ---------------------------------------------------------------- small dense factorizations (one CTA)
// In place lower Cholesky of A (k x k row-major; the strict upper part is zeroed).  flag = 1 on a
// non-positive pivot.  Left-looking: column j from the finished columns < j.
__global__ void k_cholesky(int k, double* __restrict__ A, double jitter, int* __restrict__ flag) {
  __shared__ double piv;
  for (int j = 0; j < k; ++j) {
    if (threadIdx.x == 0) {
      double s = A[(long long)j * k + j] + jitter;
      for (int p = 0; p < j; ++p) s -= A[(long long)j * k + p] * A[(long long)j * k + p];
      if (!(s > 0.0)) {
        *flag = 1;
        s = 1.0;
      }
      piv = sqrt(s);
      A[(long long)j * k + j] = piv;
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x) {
      double s = A[(long long)i * k + j];
      for (int p = 0; p < j; ++p) s -= A[(long long)i * k + p] * A[(long long)j * k + p];
      A[(long long)i * k + j] = s / piv;
    }
    __syncthreads();
  }
  for (long long idx = threadIdx.x; idx < (long long)k * k; idx += blockDim.x)
    if (idx % k > idx / k) A[idx] = 0.0;
}

// Linv = L^{-1} (lower), one column per thread: forward substitution of L x = e_c
__global__ void k_tri_inverse(int k, const double* __restrict__ L, double* __restrict__ Linv) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    for (int i = 0; i < c; ++i) Linv[(long long)i * k + c] = 0.0;
    for (int i = c; i < k; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int p = c; p < i; ++p) s -= L[(long long)i * k + p] * Linv[(long long)p * k + c];
      Linv[(long long)i * k + c] = s / L[(long long)i * k + i];
    }
  }
}

// logdet of the landmark block: 2 sum log L_jj (one warp, fixed order)
__global__ void k_logdiag(int k, const double* __restrict__ L, double* __restrict__ out) {
  double s = 0.0;
  for (int j = threadIdx.x; j < k; j += 32) s += log(L[(long long)j * k + j]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *out = 2.0 * s;
}

// ---------------------------------------------------------------- Phi = K21 L11^{-T} and G
// One CTA per 32 rows: K21 rows in shared memory (computed on the fly), Phi[a][j] = sum_{q<=j} Linv[j][q] K[a][q]
__global__ void k_phi(const double* __restrict__ Xc, KhatArgs a, long long n, const int* __restrict__ lm,
                      const int* __restrict__ lmpos, int k, int kPhiRows, const double* __restrict__ Linv,
                      double* __restrict__ Phi, double* __restrict__ Sdiag) {
  extern __shared__ double sk[];  // [kPhiRows][k]
  const long long r0 = (long long)blockIdx.x * kPhiRows;
  for (int idx = threadIdx.x; idx < kPhiRows * k; idx += blockDim.x) {
    const long long row = r0 + idx / k;
    const int q = idx % k;
    sk[idx] = (row < n && lmpos[row] < 0) ? khat_entry(Xc, a, row, lm[q]) : 0.0;
  }
  __syncthreads();
  // thread (row rr, column j): Phi = K Linv^T
  for (int idx = threadIdx.x; idx < kPhiRows * k; idx += blockDim.x) {
    const int rr = idx / k, j = idx % k;
    const long long row = r0 + rr;
    if (row >= n) continue;
    double s = 0.0;
    const double* kr = sk + (long long)rr * k;
    const double* li = Linv + (long long)j * k;
    for (int q = 0; q <= j; ++q) s = fma(li[q], kr[q], s);
    Phi[row * k + j] = s;
  }
  __syncthreads();
  // S_aa = Khat_aa - ||Phi_a||^2 (diagonal FSAI)
  for (int rr = threadIdx.x >> 5; rr < kPhiRows; rr += blockDim.x >> 5) {
    const long long row = r0 + rr;
    if (row >= n) continue;
    double s = 0.0;
    for (int j = threadIdx.x & 31; j < k; j += 32) s = fma(Phi[row * k + j], Phi[row * k + j], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) Sdiag[row] = (lmpos[row] < 0) ? khat_entry(Xc, a, row, row) - s : 1.0;
  }
}

// g_a = S_aa^{-1/2}; logdet part: sum log S_aa over non-landmark rows (per block, then final)
__global__ void k_gdiag(long long n, const int* __restrict__ lmpos, const double* __restrict__ Sdiag,
                        double* __restrict__ g, double* __restrict__ part, int* __restrict__ flag) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (lmpos[i] >= 0) {
      g[i] = 0.0;
      continue;
    }
    const double v = Sdiag[i];
    if (!(v > 0.0)) *flag = 2;
    g[i] = 1.0 / sqrt(v);
    s += log(v);
  }
  __shared__ double sm[256];
  sm[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int t = 0; t < blockDim.x; ++t) acc += sm[t];
    part[blockIdx.x] = acc;
  }
}

__global__ void k_sum_parts(int nblk, const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += part[b];
    *out = acc;
  }
}

// ---------------------------------------------------------------- applications
// y1 = Linv t1, t1 = T[lm] (k x R)
__global__ void k_lm_solve(int k, int R, const int* __restrict__ lm, const double* __restrict__ Linv,
                           const double* __restrict__ T, double* __restrict__ y1) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < k * R; idx += gridDim.x * blockDim.x) {
    const int j = idx / R, c = idx % R;
    double s = 0.0;
    for (int q = 0; q <= j; ++q) s = fma(Linv[(long long)j * k + q], T[(long long)lm[q] * R + c], s);
    y1[idx] = s;
  }
}

// out_a = g_a (T_a - Phi_a y1) for non-landmark rows, out_lm[j] = y1[j]; one warp per row
__global__ void k_uinv_rows(long long n, int k, int R, const int* __restrict__ lmpos, const double* __restrict__ Phi,
                            const double* __restrict__ g, const double* __restrict__ y1, const double* __restrict__ T,
                            double* __restrict__ out) {
  extern __shared__ double sy[];  // [k][R]
  for (int idx = threadIdx.x; idx < k * R; idx += blockDim.x) sy[idx] = y1[idx];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n; row += warps) {
    const int lp = lmpos[row];
    if (lp >= 0) {
      for (int c = lane; c < R; c += 32) out[row * R + c] = sy[lp * R + c];
      continue;
    }
    double acc[kKrMaxR];
#pragma unroll
    for (int c = 0; c < kKrMaxR; ++c) acc[c] = 0.0;
    for (int j = lane; j < k; j += 32) {
      const double ph = Phi[row * k + j];
#pragma unroll
      for (int c = 0; c < kKrMaxR; ++c)
        if (c < R) acc[c] = fma(ph, sy[j * R + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < kKrMaxR; ++c) {
      if (c < R) {
        double v = acc[c];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[c] = v;
      }
    }
    const double ga = g[row];
    for (int c = lane; c < R; c += 32) {
      double v = 0.0;
#pragma unroll
      for (int cc = 0; cc < kKrMaxR; ++cc)
        if (cc == c) v = acc[cc];
      out[row * R + c] = ga * (T[row * R + c] - v);
    }
  }
}

// U^{-T}: w2_a = g_a Y_a written to out (non-landmark rows), and per-block partials of Phi^T w2 (k x R)
constexpr int kUtBlocks = 296;
constexpr int kUtOwn = 8;  // outputs (j, c) per thread and pass
__global__ void k_uinvT_rows(long long n, int k, int R, const int* __restrict__ lmpos, const double* __restrict__ Phi,
                             const double* __restrict__ g, const double* __restrict__ Y, double* __restrict__ out,
                             double* __restrict__ part) {
  extern __shared__ double sw[];  // [32 rows][R]
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long a0 = (long long)blockIdx.x * per, a1 = min(n, a0 + per);
  const int kr = k * R;
  for (int base = 0; base < kr; base += kUtOwn * blockDim.x) {
    double acc[kUtOwn];
#pragma unroll
    for (int m = 0; m < kUtOwn; ++m) acc[m] = 0.0;
    for (long long b0 = a0; b0 < a1; b0 += 32) {
      const int cnt = (int)min((long long)32, a1 - b0);
      __syncthreads();
      for (int idx = threadIdx.x; idx < cnt * R; idx += blockDim.x) {
        const long long row = b0 + idx / R;
        const int c = idx % R;
        const double w = (lmpos[row] < 0) ? g[row] * Y[row * R + c] : 0.0;
        sw[idx] = w;
        if (base == 0 && lmpos[row] < 0) out[row * R + c] = w;
      }
      __syncthreads();
#pragma unroll
      for (int m = 0; m < kUtOwn; ++m) {
        const int idx = base + threadIdx.x + m * blockDim.x;
        if (idx < kr) {
          const int j = idx / R, c = idx % R;
          double s = acc[m];
          for (int rr = 0; rr < cnt; ++rr) s = fma(Phi[(b0 + rr) * k + j], sw[rr * R + c], s);
          acc[m] = s;
        }
      }
    }
#pragma unroll
    for (int m = 0; m < kUtOwn; ++m) {
      const int idx = base + threadIdx.x + m * blockDim.x;
      if (idx < kr) part[(long long)blockIdx.x * kr + idx] = acc[m];
    }
  }
}

// tmp[j][c] = Y[lm[j]][c] - sum_b part[b][j][c] (blocks in a fixed order)
__global__ void k_ut_reduce(int k, int R, int nblk, const int* __restrict__ lm, const double* __restrict__ Y,
                            const double* __restrict__ part, double* __restrict__ tmp) {
  const int kr = k * R;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kr; idx += gridDim.x * blockDim.x) {
    double u = 0.0;
    for (int b = 0; b < nblk; ++b) u += part[(long long)b * kr + idx];
    const int j = idx / R, c = idx % R;
    tmp[idx] = Y[(long long)lm[j] * R + c] - u;
  }
}

// w1 = Linv^T tmp, scattered to the landmark rows
__global__ void k_lm_solveT(int k, int R, const int* __restrict__ lm, const double* __restrict__ Linv,
                            const double* __restrict__ tmp, double* __restrict__ out) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < k * R; idx += gridDim.x * blockDim.x) {
    const int j = idx / R, c = idx % R;
    double s = 0.0;
    for (int q = j; q < k; ++q) s = fma(Linv[(long long)q * k + j], tmp[q * R + c], s);
    out[(long long)lm[j] * R + c] = s;
  }
}

// ---------------------------------------------------------------- host launchers
KhatArgs make_khat_args(const WinTable& tab, int nf, int family, double sf, double ell, double se) {
  KhatArgs a{};
  a.P = tab.P;
  a.nf = nf;
  a.family = family;
  a.sf2 = sf * sf;
  a.se2 = se * se;
  a.ell = ell;
  for (int w = 0; w < tab.P; ++w) {
    a.d[w] = tab.w[w].d;
    a.col0[w] = tab.w[w].feat[3 - tab.w[w].d];
  }
  return a;
}

cudaError_t launch_aafn_factor(const double* Xc, long long n, int nf, const WinTable& tab, int family, double sf,
                               double ell, double se, const int* lm, const int* lmpos, int k, double* L, double* Linv,
                               double* Phi, double* Sdiag, double* g, double* scal /* [0] logdet L, [1] sum log S */,
                               double* part, int* flag, double jitter, cudaStream_t s) {
  const KhatArgs a = make_khat_args(tab, nf, family, sf, ell, se);
  k_khat_lm<<<(int)std::min<long long>(((long long)k * k + 255) / 256, 1184), 256, 0, s>>>(Xc, a, lm, k, L);
  k_cholesky<<<1, 1024, 0, s>>>(k, L, jitter, flag);
  k_tri_inverse<<<(k + 127) / 128, 128, 0, s>>>(k, L, Linv);
  k_logdiag<<<1, 32, 0, s>>>(k, L, scal);
  const int kPhiRows = std::max(1, std::min(32, (int)((200 * 1024) / (sizeof(double) * k))));
  const size_t smem = sizeof(double) * kPhiRows * k;
  cudaError_t e = cudaFuncSetAttribute(k_phi, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  k_phi<<<(int)((n + kPhiRows - 1) / kPhiRows), 256, smem, s>>>(Xc, a, n, lm, lmpos, k, kPhiRows, Linv, Phi, Sdiag);
  k_gdiag<<<kUtBlocks, 256, 0, s>>>(n, lmpos, Sdiag, g, part, flag);
  k_sum_parts<<<1, 32, 0, s>>>(kUtBlocks, part, scal + 1);
  return cudaGetLastError();
}

size_t aafn_part_doubles(int k, int R) { return (size_t)kUtBlocks * k * R + 1024; }

cudaError_t launch_aafn_uinv(long long n, int k, int R, const int* lm, const int* lmpos, const double* Linv,
                             const double* Phi, const double* g, const double* T, double* y1, double* out,
                             cudaStream_t s) {
  k_lm_solve<<<(k * R + 255) / 256, 256, 0, s>>>(k, R, lm, Linv, T, y1);
  const size_t smem = sizeof(double) * k * R;
  static std::atomic<unsigned long long> attr{0};
  if (!optin_done(attr)) {
    cudaError_t e = cudaFuncSetAttribute(k_uinv_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    optin_mark(attr);
  }
  k_uinv_rows<<<148 * 4, 256, smem, s>>>(n, k, R, lmpos, Phi, g, y1, T, out);
  return cudaGetLastError();
}

cudaError_t launch_aafn_uinvT(long long n, int k, int R, const int* lm, const int* lmpos, const double* Linv,
                              const double* Phi, const double* g, const double* Y, double* part, double* tmp,
                              double* out, cudaStream_t s) {
  k_uinvT_rows<<<kUtBlocks, 256, sizeof(double) * 32 * R, s>>>(n, k, R, lmpos, Phi, g, Y, out, part);
  k_ut_reduce<<<(k * R + 127) / 128, 128, 0, s>>>(k, R, kUtBlocks, lm, Y, part, tmp);
  k_lm_solveT<<<(k * R + 127) / 128, 128, 0, s>>>(k, R, lm, Linv, tmp, out);
  return cudaGetLastError();
}

__global__ void k_lmpos(long long n, int k, const int* __restrict__ lm, int* __restrict__ lmpos) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    lmpos[i] = -1;
}
__global__ void k_lmpos_set(int k, const int* __restrict__ lm, int* __restrict__ lmpos) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) lmpos[lm[j]] = j;
}
cudaError_t launch_lmpos(long long n, int k, const int* lm, int* lmpos, cudaStream_t s) {
  k_lmpos<<<1184, 256, 0, s>>>(n, k, lm, lmpos);
  k_lmpos_set<<<(k + 255) / 256, 256, 0, s>>>(k, lm, lmpos);
  return cudaGetLastError();
}

}  // namespace akm

namespace akm {
// ||y - Kx||^2 and ||y||^2 (blocks in a fixed order) -> out[0], out[1]
__global__ void k_resid_part(long long n, const double* __restrict__ y, const double* __restrict__ Kx,
                             double* __restrict__ part) {
  __shared__ double s0[256], s1[256];
  double a = 0.0, b = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double r = y[i] - Kx[i];
    a = fma(r, r, a);
    b = fma(y[i], y[i], b);
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double p = 0.0, q = 0.0;
    for (int t = 0; t < blockDim.x; ++t) { p += s0[t]; q += s1[t]; }
    part[2 * blockIdx.x] = p;
    part[2 * blockIdx.x + 1] = q;
  }
}
__global__ void k_resid_final(int nblk, const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x < 2) {
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += part[2 * b + threadIdx.x];
    out[threadIdx.x] = acc;
  }
}
cudaError_t launch_resid_norms(long long n, const double* y, const double* Kx, double* part, double* out, cudaStream_t s) {
  k_resid_part<<<kUtBlocks, 256, 0, s>>>(n, y, Kx, part);
  k_resid_final<<<1, 32, 0, s>>>(kUtBlocks, part, out);
  return cudaGetLastError();
}
}  // namespace akm
