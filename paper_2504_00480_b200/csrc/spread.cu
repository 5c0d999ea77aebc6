// spread.cu -- adjoint NFFT gridding (App. A; eq. 3.3 inner sums).
//
//   g^{w,c}_l = sum_j V[j,c] phi~(x~_j^w - l/n_g),  phi~ = tensor-product Kaiser-Bessel window
//
// Design (B200, FP64-FMA bound):
//   * Points are bin-sorted (setup_kernels.cu); one CTA takes one work item = a chunk of points
//     of one bin of B^d cells.  Every point of the bin touches only the bin's footprint of
//     F^d = (B + 2m - 1)^d grid nodes, so the CTA accumulates the whole footprint x RC
//     right-hand sides in REGISTERS and writes it once with RED.ADD.F64 at the end.
//   * Per point the contribution is a rank-1 update of the (F^{d-1}) x (F*RC) footprint matrix
//       acc[(o0,o1), (o2,c)] += (w0[o0] w1[o1]) * (w2[o2] v[c]),
//     i.e. a small GEMM over the chunk's points.  Each thread owns an MT x NT register tile;
//     the two factor vectors of a batch of PB points are staged in shared memory (window
//     weights evaluated on the fly, once per point and axis), so every FMA of the inner loop
//     is useful work and shared-memory traffic is (MT+NT)/(MT*NT) of the FMA count.
//   * Window support handling: w_a[o] = phi(u_a - node) is evaluated for all F footprint
//     nodes and is exactly zero outside |delta| < m, so a bin of B > 1 cells needs no masks.
#include "akm_internal.cuh"

namespace akm {

template <int MT, int NT>
__global__ void __launch_bounds__(256) k_spread(const WinTable* __restrict__ tabp, const WorkItem* __restrict__ items,
                                                 const double* __restrict__ u_sorted, const int* __restrict__ perm,
                                                 const double* __restrict__ V, long long ldv, long long n, int r0,
                                                 int rc, int r_total, double* __restrict__ grid, double beta, int PB) {
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const double mm = (double)tab.m;
  const int F0 = g.F[0], F1 = g.F[1], F2 = g.F[2];
  const int Fmax = max(F0, max(F1, F2));
  const int M = F0 * F1;
  const int Nn = F2 * rc;
  const int TN = (Nn + NT - 1) / NT;
  const int TM = (M + MT - 1) / MT;
  const int Mpad = TM * MT, Npad = TN * NT;
  const int tid = threadIdx.x;
  const int tn = tid % TN, tm = tid / TN;
  const bool active = tm < TM;

  extern __shared__ double smem[];
  double* poly = smem;                        // [2m][kPolyLen] window polynomials
  double* As = poly + kMaxTaps * kPolyLen;    // [PB][Mpad]  w0 (x) w1
  double* Bs = As + (size_t)PB * Mpad;        // [PB][Npad]  w2 (x) v
  double* Ws = Bs + (size_t)PB * Npad;        // [PB][3][Fmax] window weights
  double* Vs = Ws + (size_t)PB * 3 * Fmax;    // [PB][rc]

  // footprint origin (global grid node) per padded axis
  int org[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) org[a] = g.box_lo[a] + it.bin[a] * g.B;

  const int taps = 2 * tab.m;
  for (int idx = tid; idx < taps * kPolyLen; idx += blockDim.x) poly[idx] = tab.poly[idx];
  __syncthreads();

  double acc[MT][NT];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j] = 0.0;

  const long long ptbase = (long long)it.win * n + it.start;
  for (int p0 = 0; p0 < it.count; p0 += PB) {
    const int pb = min(PB, it.count - p0);
    // (1) window weights and RHS values of the batch
    for (int idx = tid; idx < pb * 3 * Fmax; idx += blockDim.x) {
      const int p = idx / (3 * Fmax);
      const int a = (idx / Fmax) % 3;
      const int o = idx % Fmax;
      double wv = 0.0;
      if (a < 3 - g.d) {
        wv = (o == 0) ? 1.0 : 0.0;  // singleton axis
      } else if (o < g.F[a]) {
        const double u = u_sorted[((long long)it.win * 3 + a) * n + it.start + p0 + p];
        const double fl = floor(u);
        const int tap = o - ((int)fl - tab.m + 1 - org[a]);  // tap index of footprint node o
        if (tap >= 0 && tap < taps) wv = window_tap(poly, tap, 2.0 * (u - fl) - 1.0);
      }
      Ws[idx] = wv;
    }
    for (int idx = tid; idx < pb * rc; idx += blockDim.x) {
      const int p = idx / rc, c = idx % rc;
      const long long i = perm[ptbase + p0 + p];
      Vs[idx] = V[i * ldv + r0 + c];
    }
    __syncthreads();
    // (2) the two factors of each point's rank-1 update
    for (int idx = tid; idx < pb * Mpad; idx += blockDim.x) {
      const int p = idx / Mpad, row = idx % Mpad;
      double v = 0.0;
      if (row < M) {
        const int o0 = row / F1, o1 = row % F1;
        v = Ws[(p * 3 + 0) * Fmax + o0] * Ws[(p * 3 + 1) * Fmax + o1];
      }
      As[idx] = v;
    }
    for (int idx = tid; idx < pb * Npad; idx += blockDim.x) {
      const int p = idx / Npad, col = idx % Npad;
      double v = 0.0;
      if (col < Nn) {
        const int o2 = col / rc, c = col % rc;
        v = Ws[(p * 3 + 2) * Fmax + o2] * Vs[p * rc + c];
      }
      Bs[idx] = v;
    }
    __syncthreads();
    // (3) rank-1 updates in registers
    if (active) {
      const double* ap = As + tm * MT;
      const double* bp = Bs + tn * NT;
      for (int p = 0; p < pb; ++p) {
        double av[MT], bv[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) av[i] = ap[(size_t)p * Mpad + i];
#pragma unroll
        for (int j = 0; j < NT; ++j) bv[j] = bp[(size_t)p * Npad + j];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
    }
    __syncthreads();
  }

  // (4) one RED.ADD.F64 per touched footprint value
  if (active) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int row = tm * MT + i;
      if (row >= M) continue;
      const int o0 = row / F1, o1 = row % F1;
      const long long l0 = org[0] - g.box_lo[0] + o0;
      const long long l1 = org[1] - g.box_lo[1] + o1;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int col = tn * NT + j;
        if (col >= Nn || acc[i][j] == 0.0) continue;
        const int o2 = col / rc, c = col % rc;
        const long long l2 = org[2] - g.box_lo[2] + o2;
        const long long tap = (l0 * g.L[1] + l1) * g.L[2] + l2;
        atomicAdd(grid + (g.tap_off + tap) * r_total + r0 + c, acc[i][j]);
      }
    }
  }
}

#define AKM_SPREAD_TILES(X) X(2, 8) X(2, 16) X(4, 4) X(4, 6) X(4, 8) X(4, 11) X(4, 12) X(4, 16) X(8, 4) X(8, 6) X(8, 8) X(8, 11) X(8, 12)

bool spread_tile_supported(int MT, int NT) {
#define AKM_CASE(a, b) if (MT == a && NT == b) return true;
  AKM_SPREAD_TILES(AKM_CASE)
#undef AKM_CASE
  return false;
}

size_t spread_smem_bytes(int PB, int Mpad, int Npad, int Fmax, int rc) {
  return sizeof(double) * ((size_t)PB * (size_t)(Mpad + Npad + 3 * Fmax + rc) + kMaxTaps * kPolyLen);
}

cudaError_t launch_spread(const WinTable* dtab, const WorkItem* items, int n_items, const double* u_sorted,
                          const int* perm, const double* V, long long ldv, long long n, int r0, int rc, int r_total,
                          double* grid, int MT, int NT, int threads, int PB, size_t smem, double beta, cudaStream_t s) {
  if (n_items <= 0) return cudaSuccess;
#define AKM_CASE(a, b)                                                                                          \
  if (MT == a && NT == b) {                                                                                     \
    static bool attr_set = false;                                                                               \
    if (!attr_set) {                                                                                            \
      cudaError_t e = cudaFuncSetAttribute(k_spread<a, b>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
      if (e != cudaSuccess) return e;                                                                           \
      attr_set = true;                                                                                          \
    }                                                                                                           \
    k_spread<a, b><<<n_items, threads, smem, s>>>(dtab, items, u_sorted, perm, V, ldv, n, r0, rc, r_total, grid, \
                                                  beta, PB);                                                    \
    return cudaGetLastError();                                                                                  \
  }
  AKM_SPREAD_TILES(AKM_CASE)
#undef AKM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace akm
