// interp_impl.cuh -- the interpolation kernel template (NFFT step 3, App. A; outer sums of
// eq. 3.3).  Instantiated per (D, TAPS) in interp_d<D>_t<TAPS>.cu so the builds run in parallel;
// dispatched from interp.cu.
//
// Design: one CTA per work item (a chunk of <= 128 points of one bin),
// one thread per point.  The bin's grid footprint (F^{d-1} nodes x OPS x RC values per plane
// for d = 3; the whole footprint for d <= 2) is staged in shared memory; a point's 2m window
// weights per axis live in registers, and the tap loop does OPS*RC FMAs per weight product.
// Points of a bin with B = 1 all read the same shared-memory words (broadcast).
#pragma once
#include "akm_internal.cuh"

namespace akm {

template <int D, int TAPS, int OPS, int RC>
__global__ void __launch_bounds__(128) k_interp(const WinTable* __restrict__ tabp, const WorkItem* __restrict__ items,
                                                const double* __restrict__ u_sorted, const int* __restrict__ perm,
                                                const double* __restrict__ H, int r, int r0,
                                                double* __restrict__ part, long long n, double beta) {
  constexpr int VALS = OPS * RC;
  constexpr int VP = (VALS + 1) & ~1;  // padded to an even count (16-byte rows)
  constexpr int T0 = (D >= 3) ? TAPS : 1;
  constexpr int T1 = (D >= 2) ? TAPS : 1;
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const double mm = (double)tab.m;
  const int F0 = g.F[0], F1 = g.F[1], F2 = g.F[2];
  const int slab = F1 * F2;
  extern __shared__ double sm[];  // [slab][VP]

  int org[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) org[a] = g.box_lo[a] + it.bin[a] * g.B;

  const int tid = threadIdx.x;
  const bool has = tid < it.count;
  const long long pidx = (long long)it.start + (has ? tid : 0);
  double u[3] = {0.0, 0.0, 0.0};
  int s[3] = {0, 0, 0};  // offset of the point's first tap inside the footprint
#pragma unroll
  for (int a = 3 - D; a < 3; ++a) {
    u[a] = u_sorted[((long long)it.win * 3 + a) * n + pidx];
    s[a] = (int)floor(u[a]) - tab.m + 1 - org[a];
  }
  double w1[T1], w2[TAPS];
#pragma unroll
  for (int o = 0; o < TAPS; ++o) w2[o] = kb_window(u[2] - (double)(org[2] + s[2] + o), mm, beta);
#pragma unroll
  for (int o = 0; o < T1; ++o) w1[o] = (D >= 2) ? kb_window(u[1] - (double)(org[1] + s[1] + o), mm, beta) : 1.0;

  double acc[OPS][RC];
#pragma unroll
  for (int q = 0; q < OPS; ++q)
#pragma unroll
    for (int c = 0; c < RC; ++c) acc[q][c] = 0.0;

  const int row_vals = OPS * r;  // values per node in H
  for (int q0 = 0; q0 < F0; ++q0) {
    __syncthreads();
    const long long l0 = org[0] - g.box_lo[0] + q0;
    for (int idx = tid; idx < slab * VALS; idx += blockDim.x) {
      const int t = idx / VALS, v = idx % VALS;
      const int op = v / RC, c = v % RC;
      const int q1 = t / F2, q2 = t % F2;
      const long long l1 = org[1] - g.box_lo[1] + q1;
      const long long l2 = org[2] - g.box_lo[2] + q2;
      const long long tap = (l0 * g.L[1] + l1) * g.L[2] + l2;
      sm[t * VP + v] = H[(g.tap_off + tap) * row_vals + op * r + r0 + c];
    }
    __syncthreads();
    const int o0 = q0 - s[0];
    if (has && o0 >= 0 && o0 < T0) {
      const double wa = (D >= 3) ? kb_window(u[0] - (double)(org[0] + q0), mm, beta) : 1.0;
#pragma unroll
      for (int o1 = 0; o1 < T1; ++o1) {
        const double w01 = wa * w1[o1];
        const double* rowp = sm + ((s[1] + o1) * F2 + s[2]) * VP;
#pragma unroll
        for (int o2 = 0; o2 < TAPS; ++o2) {
          const double wt = w01 * w2[o2];
          const double* hp = rowp + o2 * VP;
#pragma unroll
          for (int q = 0; q < OPS; ++q)
#pragma unroll
            for (int c = 0; c < RC; ++c) acc[q][c] = fma(wt, hp[q * RC + c], acc[q][c]);
        }
      }
    }
  }
  if (has) {
    const long long i = perm[(long long)it.win * n + pidx];
    double* out = part + (((long long)it.win * n + i) * OPS) * r + r0;
#pragma unroll
    for (int q = 0; q < OPS; ++q)
#pragma unroll
      for (int c = 0; c < RC; ++c) out[(long long)q * r + c] = acc[q][c];
  }
}


template <int D, int T>
cudaError_t launch_interp_dt(const WinTable* dtab, const WorkItem* items, int n_items, const double* u_sorted,
                             const int* perm, const double* H, int ops, int r, int r0, int rc, double* part,
                             long long n, double beta, size_t smem, cudaStream_t s) {
#define AKM_CASE(O, R)                                                                                              \
  if (ops == O && rc == R) {                                                                                        \
    static bool attr_set = false;                                                                                   \
    if (!attr_set) {                                                                                                \
      cudaError_t e = cudaFuncSetAttribute(k_interp<D, T, O, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                           200 * 1024);                                                             \
      if (e != cudaSuccess) return e;                                                                               \
      attr_set = true;                                                                                              \
    }                                                                                                               \
    k_interp<D, T, O, R><<<n_items, 128, smem, s>>>(dtab, items, u_sorted, perm, H, r, r0, part, n, beta);         \
    return cudaGetLastError();                                                                                      \
  }
  AKM_CASE(1, 1) AKM_CASE(1, 2) AKM_CASE(1, 4) AKM_CASE(1, 11)
  AKM_CASE(2, 1) AKM_CASE(2, 2) AKM_CASE(2, 4) AKM_CASE(2, 11)
#undef AKM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace akm
