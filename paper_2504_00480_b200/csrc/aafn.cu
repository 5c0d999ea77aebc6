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

// logdet of the landmark block: 2 sum log L_jj (one warp, fixed order)
__global__ void k_logdiag(int k, const double* __restrict__ L, double* __restrict__ out) {
  double s = 0.0;
  for (int j = threadIdx.x; j < k; j += 32) s += log(L[(long long)j * k + j]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *out = 2.0 * s;
}

// ---------------------------------------------------------------- dense FP64 building blocks (setup)
// C[m][n] = beta C[m][n] + alpha sum_q A[m][q] Bop[q][n] on 64 x 64 tiles (256 threads, 4 x 4 per
// thread, K staged 16 at a time).  BT: B is N x K row-major (Bop[q][n] = B[n][q]), else K x N.
// tri != 0: Bop[q][n] = 0 for q > n (B lower triangular when BT), so a tile stops at q < n0 + 64.
// lower != 0: tiles strictly above the diagonal (n0 > m0 + 63) are skipped (symmetric updates).
constexpr int kGT = 64, kGK = 16;
template <bool BT>
__global__ void __launch_bounds__(256) k_gemm(int M, int N, int K, double alpha, const double* __restrict__ A,
                                              long long lda, const double* __restrict__ B, long long ldb, double beta,
                                              double* __restrict__ C, long long ldc, int tri, int lower) {
  __shared__ double As[kGK][kGT + 1];
  __shared__ double Bs[kGK][kGT + 1];
  const int m0 = blockIdx.y * kGT, n0 = blockIdx.x * kGT;
  if (lower && n0 > m0 + kGT - 1) return;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int kend = tri ? min(K, n0 + kGT) : K;
  for (int k0 = 0; k0 < kend; k0 += kGK) {
    for (int idx = threadIdx.x; idx < kGT * kGK; idx += 256) {
      const int r = idx / kGK, q = idx % kGK;
      const int m = m0 + r, kk = k0 + q;
      As[q][r] = (m < M && kk < kend) ? A[(long long)m * lda + kk] : 0.0;
      const int nn = n0 + r;
      double b = 0.0;
      if (nn < N && kk < kend) b = BT ? B[(long long)nn * ldb + kk] : B[(long long)kk * ldb + nn];
      Bs[q][r] = b;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kGK; ++q) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[q][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[q][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int nn = n0 + tx * 4 + j;
      if (nn >= N) continue;
      double* c = C + (long long)m * ldc + nn;
      *c = (beta == 0.0 ? 0.0 : beta * *c) + alpha * acc[i][j];
    }
  }
}

static cudaError_t gemm(bool bt, int M, int N, int K, double alpha, const double* A, long long lda, const double* B,
                        long long ldb, double beta, double* C, long long ldc, int tri, int lower, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT);
  if (bt)
    k_gemm<true><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, tri, lower);
  else
    k_gemm<false><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, tri, lower);
  return cudaGetLastError();
}

// The same product C = alpha A B^T (+ beta C) for large M on the FP64 tensor cores (m8n8k4 DMMA):
// 128 x 64 tiles, 8 warps of 32 x 32 (4 x 4 accumulator tiles), K staged 16 at a time in shared memory
// (row stride 20 = 4 mod 16: a fragment's 8 rows x 4 k-columns fall on distinct banks).  B is N x K
// row-major; tri != 0 means B[n][q] = 0 for q > n (the tile's K range ends at n0 + 64).
constexpr int kMT = 128, kNT = 64, kKT = 16, kLD = kKT + 4;
__global__ void __launch_bounds__(256) k_gemm_mma(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                  long long lda, const double* __restrict__ B, long long ldb,
                                                  double beta, double* __restrict__ C, long long ldc, int tri) {
  __shared__ double As[kMT * kLD];
  __shared__ double Bs[kNT * kLD];
  const long long m0 = (long long)blockIdx.y * kMT;
  const int n0 = blockIdx.x * kNT;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wm = (wid >> 1) * 32, wn = (wid & 1) * 32;
  const int ar = lane >> 2, ac = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int kend = tri ? min(K, n0 + kNT) : K;
  for (int k0 = 0; k0 < kend; k0 += kKT) {
    for (int idx = threadIdx.x; idx < kMT * kKT; idx += 256) {
      const int r = idx / kKT, q = idx % kKT;
      const long long m = m0 + r;
      As[r * kLD + q] = (m < M && k0 + q < kend) ? A[m * lda + k0 + q] : 0.0;
    }
    for (int idx = threadIdx.x; idx < kNT * kKT; idx += 256) {
      const int r = idx / kKT, q = idx % kKT;
      const int nn = n0 + r;
      Bs[r * kLD + q] = (nn < N && k0 + q < kend) ? B[(long long)nn * ldb + k0 + q] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKT; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[(wm + i * 8 + ar) * kLD + kk + ac];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[(wn + j * 8 + ar) * kLD + kk + ac];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long m = m0 + wm + i * 8 + ar;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int nn = n0 + wn + j * 8 + 2 * ac + h;
        if (nn >= N) continue;
        double* c = C + m * ldc + nn;
        *c = (beta == 0.0 ? 0.0 : beta * *c) + alpha * acc[i][j][h];
      }
  }
}

static cudaError_t gemm_mma(long long M, int N, int K, double alpha, const double* A, long long lda, const double* B,
                            long long ldb, double beta, double* C, long long ldc, int tri, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const dim3 grid((N + kNT - 1) / kNT, (unsigned)((M + kMT - 1) / kMT));
  k_gemm_mma<<<grid, 256, 0, s>>>((int)M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, tri);
  return cudaGetLastError();
}

// Blocked right-looking Cholesky, panel width kNb: diagonal block (one CTA, shared memory), the panel
// below it (one thread per row, forward substitution against the diagonal block), trailing update
// A22 -= L21 L21^T (k_gemm, lower tiles).  flag = 1 on a non-positive pivot.
constexpr int kNb = 32;
__global__ void k_chol_diag(int k, int p, double* __restrict__ A, double jitter, int* __restrict__ flag) {
  __shared__ double D[kNb][kNb + 1];
  const int nb = min(kNb, k - p);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, j = idx % nb;
    D[i][j] = A[(long long)(p + i) * k + p + j] + (i == j ? jitter : 0.0);
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (threadIdx.x == 0) {
      double v = D[j][j];
      if (!(v > 0.0)) {
        *flag = 1;
        v = 1.0;
      }
      D[j][j] = sqrt(v);
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) D[i][j] /= D[j][j];
    __syncthreads();
    for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
      const int i = idx / nb, c = idx % nb;
      if (i > j && c > j && c <= i) D[i][c] -= D[i][j] * D[c][j];
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, j = idx % nb;
    A[(long long)(p + i) * k + p + j] = (j <= i) ? D[i][j] : 0.0;
  }
}

__global__ void k_chol_panel(int k, int p, double* __restrict__ A) {
  __shared__ double D[kNb][kNb + 1];
  const int nb = min(kNb, k - p);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) D[idx / nb][idx % nb] = A[(long long)(p + idx / nb) * k + p + idx % nb];
  __syncthreads();
  for (int i = p + nb + blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
    double x[kNb];
#pragma unroll
    for (int j = 0; j < kNb; ++j) x[j] = (j < nb) ? A[(long long)i * k + p + j] : 0.0;
#pragma unroll
    for (int j = 0; j < kNb; ++j) {
      if (j < nb) {
        double v = x[j];
        for (int q = 0; q < j; ++q) v -= x[q] * D[j][q];
        x[j] = v / D[j][j];
      }
    }
#pragma unroll
    for (int j = 0; j < kNb; ++j)
      if (j < nb) A[(long long)i * k + p + j] = x[j];
  }
}

static cudaError_t cholesky_blocked(int k, double* A, double jitter, int* flag, cudaStream_t s) {
  for (int p = 0; p < k; p += kNb) {
    const int nb = std::min(kNb, k - p);
    k_chol_diag<<<1, 256, 0, s>>>(k, p, A, jitter, flag);
    const int rest = k - p - nb;
    if (rest <= 0) break;
    k_chol_panel<<<(rest + 127) / 128, 128, 0, s>>>(k, p, A);
    // A[p+nb:, p+nb:] -= L21 L21^T  (L21 = A[p+nb:, p:p+nb])
    const double* L21 = A + (long long)(p + nb) * k + p;
    cudaError_t e = gemm_mma(rest, rest, nb, -1.0, L21, k, L21, k, 1.0, A + (long long)(p + nb) * k + p + nb, k, 0, s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// X = L^{-1} by block rows: X[P, :] = L_PP^{-1} (I[P, :] - L[P, 0:p] X[0:p, :]); X[0:p, :] is lower
// triangular, so the product only runs over columns < p (k_gemm with B = X, K x N row-major).
__global__ void k_inv_rows(int k, int p, const double* __restrict__ L, double* __restrict__ X) {
  // rows P = [p, p + nb): X[P][c] = L_PP^{-1} (e_c restricted to P  - X[P][c] as already accumulated)
  __shared__ double D[kNb][kNb + 1];
  const int nb = min(kNb, k - p);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) D[idx / nb][idx % nb] = L[(long long)(p + idx / nb) * k + p + idx % nb];
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p + nb; c += gridDim.x * blockDim.x) {
    double x[kNb];
#pragma unroll
    for (int j = 0; j < kNb; ++j) x[j] = (j < nb) ? ((p + j == c ? 1.0 : 0.0) - X[(long long)(p + j) * k + c]) : 0.0;
#pragma unroll
    for (int j = 0; j < kNb; ++j) {
      if (j < nb) {
        double v = x[j];
        for (int q = 0; q < j; ++q) v -= D[j][q] * x[q];
        x[j] = v / D[j][j];
      }
    }
#pragma unroll
    for (int j = 0; j < kNb; ++j)
      if (j < nb) X[(long long)(p + j) * k + c] = x[j];
  }
}

static cudaError_t tri_inverse_blocked(int k, const double* L, double* X, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(X, 0, sizeof(double) * k * k, s);
  if (e != cudaSuccess) return e;
  for (int p = 0; p < k; p += kNb) {
    const int nb = std::min(kNb, k - p);
    if (p > 0) {  // X[P][0:p] = L[P][0:p] X[0:p][0:p]  (kept as the subtrahend)
      e = gemm(false, nb, p, p, 1.0, L + (long long)p * k, k, X, k, 0.0, X + (long long)p * k, k, 0, 0, s);
      if (e != cudaSuccess) return e;
    }
    k_inv_rows<<<(p + nb + 127) / 128, 128, 0, s>>>(k, p, L, X);
  }
  return cudaGetLastError();
}

// K21 rows (every row; landmark rows left zero): K[i][q] = Khat(i, lm[q])
__global__ void k_khat_rows(const double* __restrict__ Xc, KhatArgs a, long long n, const int* __restrict__ lm,
                            const int* __restrict__ lmpos, int k, double* __restrict__ K) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * k;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / k;
    const int q = (int)(idx % k);
    K[idx] = (lmpos[i] < 0) ? khat_entry(Xc, a, i, lm[q]) : 0.0;
  }
}

// S_aa = Khat_aa - ||Phi_a||^2 (diagonal FSAI); one warp per row
__global__ void k_schur_diag(const double* __restrict__ Xc, KhatArgs a, long long n, const int* __restrict__ lmpos,
                             int k, const double* __restrict__ Phi, double* __restrict__ Sdiag) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n; row += warps) {
    double s = 0.0;
    for (int j = threadIdx.x & 31; j < k; j += 32) s = fma(Phi[row * k + j], Phi[row * k + j], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) Sdiag[row] = (lmpos[row] < 0) ? khat_entry(Xc, a, row, row) - s : 1.0;
  }
}

// ---------------------------------------------------------------- G and log det
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
// Phi y1 on the FP64 tensor cores: per landmark tile (grid.y, kUiJ landmarks, y1 tile staged in
// shared memory once) every warp takes 16 rows at a time and runs K = the tile's landmarks through
// m8n8k4 DMMAs (A fragments straight from Phi in HBM: 8 rows x 4 consecutive landmarks = 8 full
// 32-byte sectors per load; B fragments from the staged y1).  Phi is read exactly once.  Per-tile row
// sums go to part[tile][row][c]; k_uinv_finish adds the tiles in a fixed order.
constexpr int kUiJ = 512;
template <int NT>  // n-tiles of 8 columns (R <= 8 NT)
__global__ void __launch_bounds__(256) k_uinv_mma(long long n, int k, int R, const double* __restrict__ Phi,
                                                  const double* __restrict__ y1, double* __restrict__ part) {
  extern __shared__ double ys[];  // [kUiJ][LDY]
  constexpr int LDY = NT * 8 + 4;  // = 4 mod 8: the 4 k-rows x 8 columns of a B fragment hit distinct banks
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j0 = blockIdx.y * kUiJ;
  const int jc = min(kUiJ, k - j0);
  for (int idx = threadIdx.x; idx < kUiJ * NT * 8; idx += blockDim.x) {
    const int j = idx / (NT * 8), c = idx % (NT * 8);
    ys[j * LDY + c] = (j < jc && c < R) ? y1[(long long)(j0 + j) * R + c] : 0.0;
  }
  __syncthreads();
  const int ar = lane >> 2, ac = lane & 3;
  for (long long r0 = ((long long)blockIdx.x * nw + wid) * 16; r0 < n; r0 += (long long)gridDim.x * nw * 16) {
    double acc[2][NT][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    const long long ra = min(r0 + ar, n - 1), rb = min(r0 + 8 + ar, n - 1);
    const double* pa = Phi + ra * k + j0 + ac;
    const double* pb = Phi + rb * k + j0 + ac;
    for (int kk = 0; kk < jc; kk += 32) {
      double fa[8], fb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = kk + 4 * u + ac < jc;
        fa[u] = ok ? __ldg(pa + kk + 4 * u) : 0.0;
        fb[u] = ok ? __ldg(pb + kk + 4 * u) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double* yrow = ys + (kk + 4 * u + ac) * LDY + ar;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double b = yrow[nt * 8];
          dmma(acc[0][nt][0], acc[0][nt][1], fa[u], b);
          dmma(acc[1][nt][0], acc[1][nt][1], fb[u], b);
        }
      }
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const long long row = r0 + mt * 8 + ar;
      if (row >= n) continue;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = nt * 8 + 2 * ac + h;
          if (c < R) part[((long long)blockIdx.y * n + row) * R + c] = acc[mt][nt][h];
        }
    }
  }
}

__global__ void k_uinv_finish(long long n, int R, int ntiles, const int* __restrict__ lmpos, const double* __restrict__ g,
                              const double* __restrict__ y1, const double* __restrict__ T,
                              const double* __restrict__ part, double* __restrict__ out) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * R;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long row = idx / R;
    const int c = (int)(idx - row * R);
    const int lp = lmpos[row];
    if (lp >= 0) {
      out[idx] = y1[(long long)lp * R + c];
      continue;
    }
    double v = 0.0;
    for (int t = 0; t < ntiles; ++t) v += part[(long long)t * n * R + idx];
    out[idx] = g[row] * (T[idx] - v);
  }
}

// U^{-T}: w2_a = g_a Y_a written to out (non-landmark rows), and per-block partials of Phi^T w2 (k x R)
// on the FP64 tensor cores: M = landmarks (each warp 32 of them, 4 m-tiles), N = R, K = the block's
// rows in steps of 32 (w2 staged in shared memory).  A fragment = Phi[4 rows][8 consecutive landmarks]:
// 4 x 64 contiguous bytes per load; Phi is read exactly once over the grid.
constexpr int kUtBlocks = 296;
constexpr int kUtWarps = 4;
// w2 = g Y on the non-landmark rows (0 on the landmark rows), also written to out (k_w2 below; the
// landmark tiles of k_uinvT_mma re-read it from L2 instead of re-forming it per tile)
__global__ void k_w2(long long n, int R, const int* __restrict__ lmpos, const double* __restrict__ g,
                     const double* __restrict__ Y, double* __restrict__ W2, double* __restrict__ out) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * R;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long row = idx / R;
    const bool rest = lmpos[row] < 0;
    const double w = rest ? g[row] * Y[idx] : 0.0;
    W2[idx] = w;
    if (rest) out[idx] = w;
  }
}

template <int NT>
__global__ void __launch_bounds__(128) k_uinvT_mma(long long n, int k, int R, const double* __restrict__ Phi,
                                                   const double* __restrict__ W2, double* __restrict__ part) {
  constexpr int LDW = NT * 8 + 4;
  __shared__ double ws[32 * LDW];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long a0 = (long long)blockIdx.x * per, a1 = min(n, a0 + per);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int jw = (blockIdx.y * kUtWarps + wid) * 32;  // this warp's 32 landmarks
  double acc[4][NT][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  int jj[4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) jj[mt] = min(jw + mt * 8 + ar, k - 1);
  for (long long b0 = a0; b0 < a1; b0 += 32) {
    const int cnt = (int)min((long long)32, a1 - b0);
    // the chunk's Phi fragments first (independent of w2): their latency overlaps the staging below
    double fa[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int rr = 4 * u + ac;
      const long long row = b0 + min(rr, cnt - 1);
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) fa[u][mt] = (rr < cnt && jw < k) ? __ldg(Phi + row * k + jj[mt]) : 0.0;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 32 * NT * 8; idx += blockDim.x) {
      const int rr = idx / (NT * 8), c = idx % (NT * 8);
      ws[rr * LDW + c] = (rr < cnt && c < R) ? W2[(b0 + rr) * R + c] : 0.0;
    }
    __syncthreads();
    if (jw >= k) continue;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double* wrow = ws + (4 * u + ac) * LDW + ar;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double b = wrow[nt * 8];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], fa[u][mt], b);
      }
    }
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int j = jw + mt * 8 + ar;
    if (j >= k) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = nt * 8 + 2 * ac + h;
        if (c < R) part[((long long)blockIdx.x * k + j) * R + c] = acc[mt][nt][h];
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

// t1 = T[lm] (k x R);  out[lm[j]] = w1[j];  LinvT = Linv^T
__global__ void k_lm_gather(int k, int R, const int* __restrict__ lm, const double* __restrict__ T, double* __restrict__ t1) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < k * R; idx += gridDim.x * blockDim.x)
    t1[idx] = T[(long long)lm[idx / R] * R + idx % R];
}
__global__ void k_lm_scatter(int k, int R, const int* __restrict__ lm, const double* __restrict__ w1, double* __restrict__ out) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < k * R; idx += gridDim.x * blockDim.x)
    out[(long long)lm[idx / R] * R + idx % R] = w1[idx];
}
__global__ void k_transpose(int k, const double* __restrict__ A, double* __restrict__ At) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)k * k;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / k, j = idx % k;
    At[j * k + i] = A[idx];
  }
}

// out = sum over tiles of part[tile][row][c] (fixed order)
__global__ void k_tile_sum(long long m, int R, int ntiles, const double* __restrict__ part, double* __restrict__ out) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < m * R;
       idx += (long long)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int t = 0; t < ntiles; ++t) v += part[(long long)t * m * R + idx];
    out[idx] = v;
  }
}

// C (m x R) = A (m x K, row-major) B (K x R) through k_uinv_mma's tiles + k_tile_sum
static cudaError_t launch_tall_mma(long long m, int K, int R, const double* A, const double* B, double* part, double* C,
                                   cudaStream_t s);

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
                               double* LinvT, double* Phi, double* K21, double* Sdiag, double* g,
                               double* scal /* [0] logdet L, [1] sum log S */, double* part, int* flag, double jitter,
                               cudaStream_t s) {
  const KhatArgs a = make_khat_args(tab, nf, family, sf, ell, se);
  k_khat_lm<<<(int)std::min<long long>(((long long)k * k + 255) / 256, 1184), 256, 0, s>>>(Xc, a, lm, k, L);
  cudaError_t e = cholesky_blocked(k, L, jitter, flag, s);
  if (e != cudaSuccess) return e;
  e = tri_inverse_blocked(k, L, Linv, s);
  if (e != cudaSuccess) return e;
  k_transpose<<<(int)std::min<long long>(((long long)k * k + 255) / 256, 4096), 256, 0, s>>>(k, Linv, LinvT);
  k_logdiag<<<1, 32, 0, s>>>(k, L, scal);
  k_khat_rows<<<148 * 16, 256, 0, s>>>(Xc, a, n, lm, lmpos, k, K21);
  // Phi = K21 Linv^T  (Linv lower: Bop[q][j] = Linv[j][q] = 0 for q > j)
  e = gemm_mma(n, k, k, 1.0, K21, k, Linv, k, 0.0, Phi, k, 1, s);
  if (e != cudaSuccess) return e;
  k_schur_diag<<<148 * 8, 256, 0, s>>>(Xc, a, n, lmpos, k, Phi, Sdiag);
  k_gdiag<<<kUtBlocks, 256, 0, s>>>(n, lmpos, Sdiag, g, part, flag);
  k_sum_parts<<<1, 32, 0, s>>>(kUtBlocks, part, scal + 1);
  return cudaGetLastError();
}

size_t aafn_part_doubles(long long n, int k, int R) {
  const size_t a = (size_t)kUtBlocks * k * R + 1024;
  const size_t b = (size_t)((k + kUiJ - 1) / kUiJ) * n * R;
  return a > b ? a : b;
}

static cudaError_t launch_uinv_tiles(long long n, int k, int R, const double* Phi, const double* y1, double* part,
                                     cudaStream_t s);

cudaError_t launch_aafn_uinv(long long n, int k, int R, const int* lm, const int* lmpos, const double* Linv,
                             const double* Phi, const double* g, const double* T, double* y1, double* tmp,
                             double* part, double* out, cudaStream_t s) {
  // y1 = L11^{-1} T[lm]
  k_lm_gather<<<(k * R + 255) / 256, 256, 0, s>>>(k, R, lm, T, tmp);
  cudaError_t e0 = launch_tall_mma(k, k, R, Linv, tmp, part, y1, s);
  if (e0 != cudaSuccess) return e0;
  cudaError_t e = launch_uinv_tiles(n, k, R, Phi, y1, part, s);
  if (e != cudaSuccess) return e;
  k_uinv_finish<<<148 * 8, 256, 0, s>>>(n, R, (k + kUiJ - 1) / kUiJ, lmpos, g, y1, T, part, out);
  return cudaGetLastError();
}

static cudaError_t launch_uinv_tiles(long long n, int k, int R, const double* Phi, const double* y1, double* part,
                                     cudaStream_t s) {
  const dim3 grid(148 * 2, (k + kUiJ - 1) / kUiJ);
  cudaError_t e;
#define AKM_UI(NT)                                                                                        \
  {                                                                                                       \
    const size_t smem = sizeof(double) * kUiJ * (NT * 8 + 4);                                             \
    static std::atomic<unsigned long long> attr{0};                                                       \
    if (!optin_done(attr)) {                                                                              \
      e = cudaFuncSetAttribute(k_uinv_mma<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
      if (e != cudaSuccess) return e;                                                                     \
      optin_mark(attr);                                                                                   \
    }                                                                                                     \
    k_uinv_mma<NT><<<grid, 256, smem, s>>>(n, k, R, Phi, y1, part);                                       \
  }
  if (R <= 8) AKM_UI(1) else if (R <= 16) AKM_UI(2) else AKM_UI(4)
#undef AKM_UI
  return cudaGetLastError();
}

static cudaError_t launch_tall_mma(long long m, int K, int R, const double* A, const double* B, double* part, double* C,
                                   cudaStream_t s) {
  cudaError_t e = launch_uinv_tiles(m, K, R, A, B, part, s);
  if (e != cudaSuccess) return e;
  k_tile_sum<<<(int)std::min<long long>((m * R + 255) / 256, 1184), 256, 0, s>>>(m, R, (K + kUiJ - 1) / kUiJ, part, C);
  return cudaGetLastError();
}

cudaError_t launch_aafn_uinvT(long long n, int k, int R, const int* lm, const int* lmpos, const double* LinvT,
                              const double* Phi, const double* g, const double* Y, double* part, double* tmp,
                              double* w1, double* w2buf, double* out, cudaStream_t s) {
  const dim3 grid(kUtBlocks, (k + 32 * kUtWarps - 1) / (32 * kUtWarps));
  double* W2 = w2buf;
  k_w2<<<(int)std::min<long long>((n * R + 255) / 256, 148 * 8), 256, 0, s>>>(n, R, lmpos, g, Y, W2, out);
  if (R <= 8)
    k_uinvT_mma<1><<<grid, 32 * kUtWarps, 0, s>>>(n, k, R, Phi, W2, part);
  else if (R <= 16)
    k_uinvT_mma<2><<<grid, 32 * kUtWarps, 0, s>>>(n, k, R, Phi, W2, part);
  else
    k_uinvT_mma<4><<<grid, 32 * kUtWarps, 0, s>>>(n, k, R, Phi, W2, part);
  k_ut_reduce<<<(k * R + 127) / 128, 128, 0, s>>>(k, R, kUtBlocks, lm, Y, part, tmp);
  cudaError_t e0 = launch_tall_mma(k, k, R, LinvT, tmp, part, w1, s);  // w1 = L11^{-T} tmp
  if (e0 != cudaSuccess) return e0;
  k_lm_scatter<<<(k * R + 255) / 256, 256, 0, s>>>(k, R, lm, w1, out);
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
