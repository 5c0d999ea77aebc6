// interp_impl.cuh -- the interpolation kernel template (NFFT step 3, App. A; outer sums of
// eq. 3.3).  Instantiated per (D, TAPS) in interp_d<D>_t<TAPS>.cu so the builds run in parallel;
// dispatched from interp.cu.
//
// Design: one CTA of 128 threads per work item = a chunk of <= 256 points of
// ONE grid cell, two points per thread.  All points of a cell share the footprint of (2m)^d
// nodes, which is staged in shared memory (whole, or one o0-plane at a time when it exceeds
// 48 KB); every tap's OPS x RC values are then read once per warp as broadcasts and feed
// 2 * OPS * RC FMAs.  Window weights come from the Horner polynomials of the window
// (window_taps).  For OPS*RC <= 10 the tap loop is sum-factorised over the last axis.
#pragma once
#include "akm_internal.cuh"

namespace akm {

template <int D, int TAPS, int OPS, int RC, int PPT>
__global__ void __launch_bounds__(64) k_interp(const WinTable* __restrict__ tabp, const WorkItem* __restrict__ items,
                                                const double* __restrict__ u_sorted, const int* __restrict__ perm,
                                                const double* __restrict__ H, int r, int r0,
                                                double* __restrict__ part, long long n) {
  constexpr int V = OPS * RC;           // values per grid node used by this CTA
  constexpr int VP = (V + 1) & ~1;      // padded to an even count (16-byte rows)
  constexpr int T0 = (D >= 3) ? TAPS : 1;
  constexpr int T1 = (D >= 2) ? TAPS : 1;
  constexpr int SLAB = T1 * TAPS;       // nodes of one o0-plane of the cell footprint
  constexpr bool FULL = (size_t)T0 * SLAB * VP * sizeof(double) <= 48 * 1024;
  constexpr int NPL = FULL ? T0 : 1;    // planes staged per pass
  constexpr bool SUMF = V <= 10;        // sum-factorised tap loop (fewer weight products)
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  __shared__ double poly[TAPS * kPolyLen];
  extern __shared__ double sm[];        // [NPL * SLAB][VP]

  const int tid = threadIdx.x;
  for (int idx = tid; idx < TAPS * kPolyLen; idx += blockDim.x) poly[idx] = tab.poly[idx];
  __syncthreads();

  // points of this thread (strided so a warp holds consecutive points of the cell)
  bool has[PPT];
  long long pidx[PPT];
  double x0[PPT], w1[PPT][T1], w2[PPT][TAPS];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int q = tid + k * blockDim.x;
    has[k] = q < it.count;
    pidx[k] = (long long)it.start + (has[k] ? q : 0);
    double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 3 - D; a < 3; ++a) {
      const double u = u_sorted[((long long)it.win * 3 + a) * n + pidx[k]];
      x[a] = 2.0 * (u - floor(u)) - 1.0;
    }
    x0[k] = x[0];
    window_taps<TAPS>(poly, x[2], w2[k]);
    if (D >= 2) {
      window_taps<T1>(poly, x[1], w1[k]);
    } else {
#pragma unroll
      for (int o = 0; o < T1; ++o) w1[k][o] = 1.0;
    }
  }

  double acc[PPT][V];
#pragma unroll
  for (int k = 0; k < PPT; ++k)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[k][v] = 0.0;

  const int cell0 = it.bin[0], cell1 = it.bin[1], cell2 = it.bin[2];
  const long long row_vals = (long long)OPS * r;  // values per node in H
  for (int pg = 0; pg < T0; pg += NPL) {
    __syncthreads();
    for (int idx = tid; idx < NPL * SLAB * V; idx += blockDim.x) {
      const int t = idx / V, v = idx % V;
      const int op = v / RC, c = v % RC;
      const int o0 = pg + t / SLAB;
      const int o1 = (t % SLAB) / TAPS, o2 = t % TAPS;
      const long long tap = ((long long)(cell0 + o0) * g.L[1] + (cell1 + o1)) * g.L[2] + (cell2 + o2);
      sm[t * VP + v] = H[(g.tap_off + tap) * row_vals + op * r + r0 + c];
    }
    __syncthreads();
#pragma unroll 1
    for (int pl = 0; pl < NPL; ++pl) {
      double wa[PPT];
#pragma unroll
      for (int k = 0; k < PPT; ++k) wa[k] = (D >= 3) ? window_tap(poly, pg + pl, x0[k]) : 1.0;
      const double* plane = sm + pl * SLAB * VP;
#pragma unroll
      for (int o1 = 0; o1 < T1; ++o1) {
        const double* rowp = plane + o1 * TAPS * VP;
        double w01[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) w01[k] = wa[k] * w1[k][o1];
        if (SUMF) {
          double t[PPT][V];
#pragma unroll
          for (int k = 0; k < PPT; ++k)
#pragma unroll
            for (int v = 0; v < V; ++v) t[k][v] = 0.0;
#pragma unroll
          for (int o2 = 0; o2 < TAPS; ++o2) {
            double h[V];
#pragma unroll
            for (int v = 0; v < V; ++v) h[v] = rowp[o2 * VP + v];
#pragma unroll
            for (int k = 0; k < PPT; ++k)
#pragma unroll
              for (int v = 0; v < V; ++v) t[k][v] = fma(w2[k][o2], h[v], t[k][v]);
          }
#pragma unroll
          for (int k = 0; k < PPT; ++k)
#pragma unroll
            for (int v = 0; v < V; ++v) acc[k][v] = fma(w01[k], t[k][v], acc[k][v]);
        } else {
#pragma unroll
          for (int o2 = 0; o2 < TAPS; ++o2) {
            double h[V];
#pragma unroll
            for (int v = 0; v < V; ++v) h[v] = rowp[o2 * VP + v];
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
              const double wt = w01[k] * w2[k][o2];
#pragma unroll
              for (int v = 0; v < V; ++v) acc[k][v] = fma(wt, h[v], acc[k][v]);
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    if (!has[k]) continue;
    const long long i = perm[(long long)it.win * n + pidx[k]];
    double* out = part + (((long long)it.win * n + i) * OPS) * r + r0;
#pragma unroll
    for (int q = 0; q < OPS; ++q)
#pragma unroll
      for (int c = 0; c < RC; ++c) out[(long long)q * r + c] = acc[k][q * RC + c];
  }
}

// dynamic shared memory of k_interp<D, TAPS, OPS, RC, *>
inline size_t interp_smem(int D, int TAPS, int OPS, int RC) {
  const int V = OPS * RC, VP = (V + 1) & ~1;
  const int T0 = (D >= 3) ? TAPS : 1, T1 = (D >= 2) ? TAPS : 1;
  const size_t slab = (size_t)T1 * TAPS;
  const bool full = (size_t)T0 * slab * VP * sizeof(double) <= 48 * 1024;
  return (full ? T0 : 1) * slab * VP * sizeof(double);
}


// ---------------------------------------------------------------- FP64 tensor-core variant
// For OPS*RC >= 8 values per node: per o0-plane of the cell footprint, S[p][v] += sum over the
// plane's taps t of W[p][t] H[t][v] is a GEMM (M = points, N = values, K = taps) on DMMA.  The
// A fragment W[p][t] = (w0 w1)[p] * w2[p][t] is one multiply per thread per k-step; B fragments
// come from the staged plane (row stride = 4 mod 16 doubles).  Planes are double-buffered with
// cp.async so staging overlaps the MMAs.  8 warps x 16 points = 128 points per work item.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int D, int TAPS, int OPS, int RC>
__global__ void __launch_bounds__(256) k_interp_mma(const WinTable* __restrict__ tabp,
                                                    const WorkItem* __restrict__ items,
                                                    const double* __restrict__ u_sorted, const int* __restrict__ perm,
                                                    const double* __restrict__ H, int r, int r0,
                                                    double* __restrict__ part, long long n) {
  constexpr int V = OPS * RC;
  constexpr int NT = (V + 7) / 8;
  constexpr int LDH = mma_ld(NT * 8);
  constexpr int T0 = (D >= 3) ? TAPS : 1;
  constexpr int T1 = (D >= 2) ? TAPS : 1;
  constexpr int SLAB = T1 * TAPS;
  constexpr int KQ = TAPS / 4;
  constexpr int MT = 2;
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  __shared__ double poly[TAPS * kPolyLen];
  extern __shared__ double sm[];  // [2][SLAB][LDH]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < TAPS * kPolyLen; idx += blockDim.x) poly[idx] = tab.poly[idx];

  const int cell0 = it.bin[0], cell1 = it.bin[1], cell2 = it.bin[2];
  const long long row_vals = (long long)OPS * r;
  auto stage = [&](int o0, double* buf) {
    for (int idx = tid; idx < SLAB * V; idx += blockDim.x) {
      const int t = idx / V, v = idx % V;
      const int op = v / RC, c = v % RC;
      const int o1 = t / TAPS, o2 = t % TAPS;
      const long long tap = ((long long)(cell0 + o0) * g.L[1] + (cell1 + o1)) * g.L[2] + (cell2 + o2);
      cp_async8(buf + t * LDH + v, H + (g.tap_off + tap) * row_vals + op * r + r0 + c);
    }
    cp_async_commit();
  };
  stage(0, sm);
  __syncthreads();  // poly

  __shared__ double w1s[8 * MT * 8][T1];  // [point of the CTA][o1]
  bool has[MT];
  long long pidx[MT];
  double x0[MT], w2[MT][KQ];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int q = warp * 16 + mt * 8 + (lane >> 2);
    has[mt] = q < it.count;
    pidx[mt] = (long long)it.start + (has[mt] ? q : 0);
    double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 3 - D; a < 3; ++a) {
      const double u = u_sorted[((long long)it.win * 3 + a) * n + pidx[mt]];
      x[a] = 2.0 * (u - floor(u)) - 1.0;
    }
    x0[mt] = x[0];
    // the 4 lanes of a quad share a point: lane&3 evaluates taps {lane&3, +4, +8, ...}
#pragma unroll
    for (int kq = 0; kq < (T1 + 3) / 4; ++kq) {
      const int o = kq * 4 + (lane & 3);
      if (o < T1) w1s[q][o] = (D >= 2) ? window_tap(poly, o, x[1]) : 1.0;
    }
#pragma unroll
    for (int kq = 0; kq < KQ; ++kq) w2[mt][kq] = has[mt] ? window_tap(poly, kq * 4 + (lane & 3), x[2]) : 0.0;
  }
  __syncwarp();

  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

  for (int o0 = 0; o0 < T0; ++o0) {
    double* cur = sm + (o0 & 1) * SLAB * LDH;
    if (o0 + 1 < T0) {
      stage(o0 + 1, sm + ((o0 + 1) & 1) * SLAB * LDH);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    double wa[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) wa[mt] = (D >= 3) ? window_tap(poly, o0, x0[mt]) : 1.0;
    const double* bbase = cur + (lane & 3) * LDH + (lane >> 2);
#pragma unroll 1
    for (int o1 = 0; o1 < T1; ++o1) {
      double w01[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) w01[mt] = wa[mt] * w1s[warp * 16 + mt * 8 + (lane >> 2)][o1];
#pragma unroll
      for (int kq = 0; kq < KQ; ++kq) {
        const double* bp = bbase + (o1 * TAPS + kq * 4) * LDH;
        double b[NT], a[MT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = bp[nt * 8];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) a[mt] = w01[mt] * w2[mt][kq];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
      }
    }
    __syncthreads();  // buffer `cur` is re-filled two planes later
  }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    if (!has[mt]) continue;
    const long long i = perm[(long long)it.win * n + pidx[mt]];
    double* out = part + (((long long)it.win * n + i) * OPS) * r + r0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int v = nt * 8 + 2 * (lane & 3) + h;
        if (v < V) out[(long long)(v / RC) * r + (v % RC)] = acc[mt][nt][h];
      }
  }
}

inline size_t interp_mma_smem(int D, int TAPS, int OPS, int RC) {
  const int V = OPS * RC, NT = (V + 7) / 8;
  const int T1 = (D >= 2) ? TAPS : 1;
  return 2 * (size_t)T1 * TAPS * mma_ld(NT * 8) * sizeof(double);
}

template <int D, int T>
cudaError_t launch_interp_dt(const WinTable* dtab, const WorkItem* items, int n_items, const double* u_sorted,
                             const int* perm, const double* H, int ops, int r, int r0, int rc, double* part,
                             long long n, cudaStream_t s) {
  constexpr int PPT = 2;
#define AKM_CASE(O, R)                                                                                              \
  if (ops == O && rc == R) {                                                                                        \
    if constexpr (O * R >= 8) {                                                                                     \
      const size_t smem = interp_mma_smem(D, T, O, R);                                                              \
      static bool attr_set = false;                                                                                 \
      if (!attr_set) {                                                                                              \
        cudaError_t e = cudaFuncSetAttribute(k_interp_mma<D, T, O, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)smem);                                                            \
        if (e != cudaSuccess) return e;                                                                             \
        attr_set = true;                                                                                            \
      }                                                                                                             \
      k_interp_mma<D, T, O, R><<<n_items, 256, smem, s>>>(dtab, items, u_sorted, perm, H, r, r0, part, n);         \
    } else {                                                                                                        \
      const size_t smem = interp_smem(D, T, O, R);                                                                  \
      static bool attr_set = false;                                                                                 \
      if (!attr_set) {                                                                                              \
        cudaError_t e = cudaFuncSetAttribute(k_interp<D, T, O, R, PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,\
                                             (int)smem);                                                            \
        if (e != cudaSuccess) return e;                                                                             \
        attr_set = true;                                                                                            \
      }                                                                                                             \
      k_interp<D, T, O, R, PPT><<<n_items, 64, smem, s>>>(dtab, items, u_sorted, perm, H, r, r0, part, n);         \
    }                                                                                                               \
    return cudaGetLastError();                                                                                      \
  }
  AKM_CASE(1, 1) AKM_CASE(1, 2) AKM_CASE(1, 4) AKM_CASE(1, 11)
  AKM_CASE(2, 1) AKM_CASE(2, 2) AKM_CASE(2, 4) AKM_CASE(2, 11)
#undef AKM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace akm
