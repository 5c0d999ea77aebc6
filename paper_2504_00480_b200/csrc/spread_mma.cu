// spread_mma.cu -- adjoint NFFT gridding on the FP64 tensor pipe (App. A,
// P:1201-1211; inner sums of eq. 3.3):
//
//   g^{w,c}_l = sum_j V[j,c] phi~(x~_j^w - l/n_g)
//
// Per work item (a chunk of points of one bin of B^d cells) the bin's footprint accumulator is
//   C[(o0,o1), (o2,c)] = sum_p (w0_p[o0] w1_p[o1]) * (w2_p[o2] v_p[c])   = A'^T B,
// a GEMM with K = points.  It runs on DMMA (mma.sync.m8n8k4.f64): on B200 DMMA and DFMA share
// one FP64 pipe (35 TFLOP/s either way, profiles/r01_fp64_peaks.txt) but one DMMA instruction
// carries 256 FMAs, so operand delivery and issue stop limiting and the accumulator tile lives in
// MMA fragments (2 doubles per thread per 8x8 tile).  Each warp owns MB x NB tiles of C; the two
// factor matrices of a batch of PB points are staged in shared memory with row strides = 4 mod 16
// doubles (conflict-free fragment loads).  Window weights: Horner polynomials (window_taps).
// The footprint is written once per work item with RED.ADD.F64.
#include "akm_internal.cuh"

namespace akm {

template <int MB, int NB>
__global__ void __launch_bounds__(288) k_spread_mma(const WinTable* __restrict__ tabp,
                                                    const WorkItem* __restrict__ items,
                                                    const double* __restrict__ u_sorted, const int* __restrict__ perm,
                                                    const double* __restrict__ V, long long ldv, long long n, int r0,
                                                    int rc, int r_total, double* __restrict__ grid, int PB, int WN) {
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const int F0 = g.F[0], F1 = g.F[1], F2 = g.F[2];
  const int Fmax = max(F0, max(F1, F2));
  const int M = F0 * F1, Nn = F2 * rc;
  const int TMt = (M + 7) / 8, TNt = (Nn + 7) / 8;
  const int lda = mma_ld(TMt * 8), ldb = mma_ld(TNt * 8);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int taps = 2 * tab.m;

  extern __shared__ double smem[];
  double* poly = smem;                         // [2m][kPolyLen]
  double* As = poly + kMaxTaps * kPolyLen;     // [PB][lda]  w0 (x) w1
  double* Bs = As + (size_t)PB * lda;          // [PB][ldb]  w2 (x) v
  double* Ws = Bs + (size_t)PB * ldb;          // [PB][3][Fmax]
  double* Vs = Ws + (size_t)PB * 3 * Fmax;     // [PB][rc]

  int org[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) org[a] = g.box_lo[a] + it.bin[a] * g.B;
  for (int idx = tid; idx < taps * kPolyLen; idx += blockDim.x) poly[idx] = tab.poly[idx];

  double acc[MB][NB][2];
#pragma unroll
  for (int i = 0; i < MB; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const long long ptbase = (long long)it.win * n + it.start;
  for (int p0 = 0; p0 < it.count; p0 += PB) {
    const int pb = min(PB, it.count - p0);
    const int pb4 = (pb + 3) & ~3;
    __syncthreads();  // poly visible / previous batch consumed
    // (1) window weights: one thread per (point, axis); Horner polynomials, no divisions
    for (int pa = tid; pa < pb * 3; pa += blockDim.x) {
      const int p = pa / 3, a = pa - 3 * p;
      double* wrow = Ws + (size_t)pa * Fmax;
      if (a < 3 - g.d) {
        for (int o = 0; o < Fmax; ++o) wrow[o] = (o == 0) ? 1.0 : 0.0;
      } else {
        const double u = u_sorted[((long long)it.win * 3 + a) * n + it.start + p0 + p];
        const double fl = floor(u);
        const int s0 = (int)fl - tab.m + 1 - org[a];  // footprint position of the point's tap 0
        const double x = 2.0 * (u - fl) - 1.0;
        for (int o = 0; o < Fmax; ++o) {
          const int tap = o - s0;
          wrow[o] = (tap >= 0 && tap < taps && o < g.F[a]) ? window_tap(poly, tap, x) : 0.0;
        }
      }
    }
    for (int pc = tid; pc < pb * rc; pc += blockDim.x) {
      const int p = pc / rc, c = pc - p * rc;
      Vs[pc] = V[(long long)perm[ptbase + p0 + p] * ldv + r0 + c];
    }
    __syncthreads();
    // (2) factor matrices; each thread owns whole columns (index math once per column)
    for (int row = tid; row < lda; row += blockDim.x) {
      const bool ok = row < M;
      const int o0 = ok ? row / F1 : 0, o1 = ok ? row - (row / F1) * F1 : 0;
      for (int p = 0; p < pb4; ++p)
        As[(size_t)p * lda + row] = (ok && p < pb) ? Ws[(p * 3 + 0) * Fmax + o0] * Ws[(p * 3 + 1) * Fmax + o1] : 0.0;
    }
    for (int col = tid; col < ldb; col += blockDim.x) {
      const bool ok = col < Nn;
      const int o2 = ok ? col / rc : 0, c = ok ? col - (col / rc) * rc : 0;
      for (int p = 0; p < pb4; ++p)
        Bs[(size_t)p * ldb + col] = (ok && p < pb) ? Ws[(p * 3 + 2) * Fmax + o2] * Vs[p * rc + c] : 0.0;
    }
    __syncthreads();
    // C += A'^T B over this batch, 4 points per MMA k-step
    const double* ap = As + (lane & 3) * lda + (wm * MB) * 8 + (lane >> 2);
    const double* bp = Bs + (lane & 3) * ldb + (wn * NB) * 8 + (lane >> 2);
    for (int k = 0; k < pb4; k += 4) {
      double a[MB], b[NB];
#pragma unroll
      for (int i = 0; i < MB; ++i) a[i] = ap[(size_t)k * lda + i * 8];
#pragma unroll
      for (int j = 0; j < NB; ++j) b[j] = bp[(size_t)k * ldb + j * 8];
#pragma unroll
      for (int i = 0; i < MB; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }

  // flush: fragment (row = lane>>2, cols 2*(lane&3) + {0,1}) of each owned tile
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int row = (wm * MB + i) * 8 + (lane >> 2);
    if (row >= M) continue;
    const long long l0 = org[0] - g.box_lo[0] + row / F1;
    const long long l1 = org[1] - g.box_lo[1] + row % F1;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = (wn * NB + j) * 8 + 2 * (lane & 3) + h;
        const double v = acc[i][j][h];
        if (col >= Nn || v == 0.0) continue;
        const long long l2 = org[2] - g.box_lo[2] + col / rc;
        const long long tap = (l0 * g.L[1] + l1) * g.L[2] + l2;
        atomicAdd(grid + (g.tap_off + tap) * r_total + r0 + col % rc, v);
      }
    }
  }
}

#define AKM_MMA_TILES(X) X(2, 2) X(3, 2) X(4, 2) X(2, 3) X(3, 3) X(4, 3) X(2, 4) X(3, 4) X(4, 4) X(6, 3) X(3, 6) X(6, 6)

bool spread_mma_choose(int M, int Nn, int& MB, int& NB, int& WM, int& WN) {
  static const int cand[][2] = {{2, 2}, {3, 2}, {4, 2}, {2, 3}, {3, 3}, {4, 3}, {2, 4}, {3, 4}, {4, 4}, {6, 3}, {3, 6}, {6, 6}};
  const int TMt = (M + 7) / 8, TNt = (Nn + 7) / 8;
  double best = 1e300;
  bool found = false;
  for (auto& c : cand) {
    const int mb = c[0], nb = c[1];
    const int wm = (TMt + mb - 1) / mb, wn = (TNt + nb - 1) / nb;
    const int warps = wm * wn;
    if (warps > 9) continue;  // __launch_bounds__(288)
    // cost: tile slots issued (incl. empty ones) + operand loads per k-step; prefer >= 4 warps
    const double slots = (double)warps * mb * nb;
    const double loads = (double)warps * (mb + nb) * 0.25;
    double score = slots + loads;
    if (warps < 4) score *= 1.0 + 0.15 * (4 - warps);
    if (score < best) {
      best = score;
      MB = mb;
      NB = nb;
      WM = wm;
      WN = wn;
      found = true;
    }
  }
  return found;
}

size_t spread_mma_smem(int PB, int M, int Nn, int Fmax, int rc) {
  const int TMt = (M + 7) / 8, TNt = (Nn + 7) / 8;
  return sizeof(double) * ((size_t)kMaxTaps * kPolyLen +
                           (size_t)PB * (mma_ld(TMt * 8) + mma_ld(TNt * 8) + 3 * Fmax + rc));
}

cudaError_t launch_spread_mma(const WinTable* dtab, const WorkItem* items, int n_items, const double* u_sorted,
                              const int* perm, const double* V, long long ldv, long long n, int r0, int rc,
                              int r_total, double* grid, int MB, int NB, int WM, int WN, int PB, size_t smem,
                              cudaStream_t s) {
  if (n_items <= 0) return cudaSuccess;
  const int threads = 32 * WM * WN;
#define AKM_CASE(a, b)                                                                                         \
  if (MB == a && NB == b) {                                                                                    \
    static bool attr_set = false;                                                                              \
    if (!attr_set) {                                                                                           \
      cudaError_t e = cudaFuncSetAttribute(k_spread_mma<a, b>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                           200 * 1024);                                                        \
      if (e != cudaSuccess) return e;                                                                          \
      attr_set = true;                                                                                         \
    }                                                                                                          \
    k_spread_mma<a, b><<<n_items, threads, smem, s>>>(dtab, items, u_sorted, perm, V, ldv, n, r0, rc, r_total, \
                                                      grid, PB, WN);                                           \
    return cudaGetLastError();                                                                                 \
  }
  AKM_MMA_TILES(AKM_CASE)
#undef AKM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace akm
