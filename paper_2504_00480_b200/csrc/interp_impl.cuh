// interp_impl.cuh -- the interpolation kernel template (NFFT step 3, App. A; outer sums of
// eq. 3.3).  Instantiated per (D, TAPS) in interp_d<D>_t<TAPS>.cu so the builds run in parallel;
// dispatched from interp.cu.
//
// Two kernels: k_interp_mma (OPS*RC >= 8 values per node: per-cell work items,
// the tap contraction as a GEMM on DMMA) and k_interp_bin (fewer values: per-bin work items,
// scalar FP64 with the last axis sum-factorised).  Window weights come from the Chebyshev
// polynomials of the window (window_taps / window_taps_estrin).
#pragma once
#include <cuda.h>

#include "akm_internal.cuh"

namespace akm {

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

// TMA staging (TMA = true): every footprint plane [o1][o2][v] is ONE cp.async.bulk.tensor.3d of the
// window's tensor map (dims: values per node, axis-2 nodes, (axis-0, axis-1) rows; 16-byte node
// pitch needs an even number of values per node), box [LDH][TAPS][T1]: the values past V fall
// outside the tensor and arrive as zeros, which is exactly the padded plane layout of the cp.async
// path.  One elected thread issues the copy; the plane's mbarrier (expect_tx) signals its arrival.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned phase) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
  return ok != 0;
}

template <int D, int TAPS, int OPS, int RC, bool TMA = false>
__global__ void __launch_bounds__(256, 2) k_interp_mma(const WinTable* __restrict__ tabp,
                                                    const WorkItem* __restrict__ items,
                                                    const double* __restrict__ u_sorted, const int* __restrict__ perm,
                                                    const double* __restrict__ H, int r, int r0,
                                                    double* __restrict__ part, long long n,
                                                    const __grid_constant__ TmaMaps maps) {
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
  __shared__ __align__(8) unsigned long long pbar[2];  // TMA: "full" mbarrier per plane buffer
  __shared__ __align__(8) unsigned long long ebar[2];  // TMA: "empty" mbarrier per plane buffer (8 warp arrivals)
  extern __shared__ __align__(128) double sm[];  // [2][SLAB][LDH]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < TAPS * kPolyLen; idx += blockDim.x) poly[idx] = tab.poly[idx];
  if (TMA && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&pbar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&pbar[1])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;\n" ::"r"(smem_u32(&ebar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;\n" ::"r"(smem_u32(&ebar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  unsigned pphase[2] = {0u, 0u}, ephase[2] = {0u, 0u};

  const int cell0 = it.bin[0], cell1 = it.bin[1], cell2 = it.bin[2];
  const long long row_vals = (long long)OPS * r;
  const bool contiguous = (RC == r && r0 == 0);  // all V values of a node adjacent in H
  const long long L1g = g.L[1], L2g = g.L[2], toff = g.tap_off;
  auto stage = [&](int o0, double* buf) {
    if constexpr (TMA) {
      if (tid == 0) {
        const int slot = (buf == sm) ? 0 : 1;
        constexpr unsigned bytes = (unsigned)(SLAB * LDH * sizeof(double));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads of buf -> async write
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&pbar[slot])),
                     "r"(bytes) : "memory");
        const int row = (int)((cell0 + o0) * L1g + cell1);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
            ::"r"(smem_u32(buf)), "l"(&maps.m[it.win]), "r"(0), "r"(cell2), "r"(row), "r"(smem_u32(&pbar[slot]))
            : "memory");
      }
      return;
    }
    if (contiguous) {
      // each footprint row (o0, o1) is one run of TAPS * V consecutive doubles of H, copied by
      // warp o1 % 8 with consecutive lanes on consecutive doubles (immediate source offsets)
      constexpr int RUN = TAPS * V, CPL = (RUN + 31) / 32;
      const int lane = tid & 31;
      const double* base = H + (toff + ((long long)(cell0 + o0) * L1g + cell1) * L2g + cell2) * row_vals + lane;
      for (int o1 = tid >> 5; o1 < T1; o1 += 8) {
        const double* src = base + o1 * L2g * row_vals;
        double* dst = buf + o1 * TAPS * LDH;
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int col = lane + 32 * j, o2 = col / V;
          if (j * 32 + 32 <= RUN || col < RUN) cp_async8(dst + o2 * LDH + (col - o2 * V), src + 32 * j);
        }
      }
    } else {
      for (int idx = tid; idx < SLAB * V; idx += blockDim.x) {
        const int t = idx / V, v = idx % V;
        const int op = v / RC, c = v % RC;
        const int o1 = t / TAPS, o2 = t % TAPS;
        const long long tap = ((long long)(cell0 + o0) * L1g + (cell1 + o1)) * L2g + (cell2 + o2);
        cp_async8(buf + t * LDH + v, H + (toff + tap) * row_vals + op * r + r0 + c);
      }
    }
    cp_async_commit();
  };
  if (TMA) __syncthreads();  // mbarriers initialised before the first copy
  stage(0, sm);
  if (TMA && T0 > 1) stage(1, sm + SLAB * LDH);  // TMA: both buffers in flight from the start
  __syncthreads();  // poly

  __shared__ double w1s[8 * MT * 8][T1];  // [point of the CTA][o1]
  __shared__ double w0s[8 * MT * 8][T0];  // [point of the CTA][o0]
  bool has[MT];
  long long pidx[MT];
  double w2[MT][KQ];
  // window weights by Estrin (independent chains: next to the other CTA's DMMA stream every
  // dependent FP64 step costs ~135 clk).  The 4 lanes of a quad share a point: lane&3 takes the
  // taps {lane&3, +4, +8, ...} of w2 and a quarter of the w0 / w1 taps for the shared tables.
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
    // lane&3 evaluates the taps {lane&3, +4, +8, ...} of each axis (KQ = TAPS / 4 of them)
    const int l4 = lane & 3;
    double wt[KQ];
    window_taps_estrin_strided<KQ>(poly, l4, 4, x[2], wt);
#pragma unroll
    for (int kq = 0; kq < KQ; ++kq) w2[mt][kq] = has[mt] ? wt[kq] : 0.0;
    if (D >= 2) {
      window_taps_estrin_strided<KQ>(poly, l4, 4, x[1], wt);
#pragma unroll
      for (int kq = 0; kq < KQ; ++kq) w1s[q][l4 + 4 * kq] = wt[kq];
    } else if (l4 == 0) {
      w1s[q][0] = 1.0;
    }
    if (D >= 3) {
      window_taps_estrin_strided<KQ>(poly, l4, 4, x[0], wt);
#pragma unroll
      for (int kq = 0; kq < KQ; ++kq) w0s[q][l4 + 4 * kq] = wt[kq];
    } else if (l4 == 0) {
      w0s[q][0] = 1.0;
    }
  }
  __syncwarp();
  const bool wact = warp * 16 < it.count;  // warp-uniform: this warp holds at least one point

  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

  for (int o0 = 0; o0 < T0; ++o0) {
    double* cur = sm + (o0 & 1) * SLAB * LDH;
    if (!TMA && o0 + 1 < T0) stage(o0 + 1, sm + ((o0 + 1) & 1) * SLAB * LDH);
    if constexpr (TMA) {
      const int slot = o0 & 1;
      while (!mbar_try_wait(smem_u32(&pbar[slot]), pphase[slot])) {
      }
      pphase[slot] ^= 1u;
    } else {
      if (o0 + 1 < T0) cp_async_wait<1>();
      else cp_async_wait<0>();
      __syncthreads();
    }
    double wa[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) wa[mt] = w0s[warp * 16 + mt * 8 + (lane >> 2)][o0];
    const double* bbase = cur + (lane & 3) * LDH + (lane >> 2);
    // rows in groups of G: first the A values of the group (DMULs), then its DMMAs.  With the
    // TMA-staged planes one row per group measures fastest (c4 interpolation G = 1 / 2 / 3 / 4 / 6:
    // 10.80 / 10.84 / 10.88 / 10.94 / 10.92 ms).  Warps without points skip the MMAs.
    constexpr int G = 1;
    if (wact) {
#pragma unroll 1
      for (int g0 = 0; g0 < T1; g0 += G) {
        double af[G][KQ][MT];
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const double w01 = wa[mt] * w1s[warp * 16 + mt * 8 + (lane >> 2)][g0 + gg];
#pragma unroll
            for (int kq = 0; kq < KQ; ++kq) af[gg][kq][mt] = w01 * w2[mt][kq];
          }
        }
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
#pragma unroll
          for (int kq = 0; kq < KQ; ++kq) {
            const double* bp = bbase + ((g0 + gg) * TAPS + kq * 4) * LDH;
            double b[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) b[nt] = bp[nt * 8];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[gg][kq][mt], b[nt]);
          }
        }
      }
    }
    if constexpr (TMA) {
      // release the buffer: each warp arrives on its "empty" barrier; thread 0 waits for all 8 and
      // refills it with plane o0 + 2 (no CTA-wide barrier per plane)
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&ebar[o0 & 1])) : "memory");
      if (tid == 0 && o0 + 2 < T0) {
        while (!mbar_try_wait(smem_u32(&ebar[o0 & 1]), ephase[o0 & 1])) {
        }
        ephase[o0 & 1] ^= 1u;
        stage(o0 + 2, cur);
      }
    } else {
      __syncthreads();  // buffer `cur` is re-filled two planes later
    }
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


// ---------------------------------------------------------------- bin-based scalar variant
// For few values per node (OPS*RC < 8) and sparse cells: one CTA of 128 threads per work item = a
// chunk of <= 128 points of ONE BIN (B^d cells, the spreading bins), one point per thread.  The
// bin footprint (F = B + 2m - 1 nodes per axis) streams through shared memory one o0-plane at a
// time (double-buffered); each thread reads its own 2m x 2m window of the plane at its cell's
// offset inside the bin.  Points are sorted by cell inside a bin, so the lanes of a warp mostly
// read the same addresses (broadcasts).  FP64 FMAs per point and value: (2m)^d + (2m)^(d-1).
template <int D, int TAPS, int OPS, int RC>
__global__ void __launch_bounds__(128, (OPS * RC == 2) ? 6 : ((OPS * RC >= 8 && OPS * RC <= 12) ? 4 : 1)) k_interp_bin(const WinTable* __restrict__ tabp,
                                                    const WorkItem* __restrict__ items,
                                                    const double* __restrict__ u_sorted, const int* __restrict__ perm,
                                                    const double* __restrict__ H, int r, int r0,
                                                    double* __restrict__ part, long long n, int whole) {
  constexpr int V = OPS * RC;
  constexpr int VP = (V + 1) & ~1;
  constexpr int T1 = (D >= 2) ? TAPS : 1;
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const int F0 = g.F[0], F1 = g.F[1], F2 = g.F[2], B = g.B;
  const int plane = F1 * F2;
  __shared__ double poly[TAPS * kPolyLen];
  extern __shared__ double sm[];  // whole ? [F0][F1*F2][VP] : [2][F1*F2][VP]
  const int tid = threadIdx.x;
  for (int idx = tid; idx < TAPS * kPolyLen; idx += blockDim.x) poly[idx] = tab.poly[idx];

  int org[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) org[a] = g.box_lo[a] + it.bin[a] * (a < 3 - D ? 0 : B);
  const long long row_vals = (long long)OPS * r;
  const long long tap0 = g.tap_off + ((long long)(org[0] - g.box_lo[0]) * g.L[1] + (org[1] - g.box_lo[1])) * g.L[2] +
                         (org[2] - g.box_lo[2]);
  auto stage = [&](int P, double* buf) {  // footprint plane P of the bin
    for (int idx = tid; idx < plane * V; idx += blockDim.x) {
      const int t = idx / V, v = idx - t * V;
      const int op = v / RC, c = v - op * RC;
      const int q1 = t / F2, q2 = t - q1 * F2;
      const long long tap = tap0 + ((long long)P * g.L[1] + q1) * g.L[2] + q2;
      cp_async8(buf + t * VP + v, H + tap * row_vals + op * r + r0 + c);
    }
    cp_async_commit();
  };
  // the whole bin footprint when it fits (one barrier), else planes double-buffered
  const int nstage = whole ? F0 : 1;
  for (int P = 0; P < nstage; ++P) stage(P, sm + P * plane * VP);
  cp_async_wait<0>();
  __syncthreads();  // poly, staged planes

  const bool has = tid < it.count;
  const long long pidx = (long long)it.start + (has ? tid : 0);
  int s[3] = {0, 0, 0};  // the point's cell offset inside the bin (= its footprint offset)
  double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 3 - D; a < 3; ++a) {
    const double u = u_sorted[((long long)it.win * 3 + a) * n + pidx];
    const double fl = floor(u);
    x[a] = 2.0 * (u - fl) - 1.0;
    s[a] = (int)fl - tab.m + 1 - org[a];
  }
  double w1[T1], w2[TAPS];
  window_taps_estrin<TAPS>(poly, x[2], w2);
  if (D >= 2) {
    window_taps_estrin<T1>(poly, x[1], w1);
  } else {
#pragma unroll
    for (int o = 0; o < T1; ++o) w1[o] = 1.0;
  }
  double acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.0;

  for (int P = 0; P < F0; ++P) {
    double* cur = whole ? sm + P * plane * VP : sm + (P & 1) * plane * VP;
    if (!whole && P + 1 < F0) stage(P + 1, sm + ((P + 1) & 1) * plane * VP);
    const int o0 = P - s[0];
    if (has && o0 >= 0 && o0 < ((D >= 3) ? TAPS : 1)) {
      const double wa = (D >= 3) ? window_tap(poly, o0, x[0]) : 1.0;
      const double* base = cur + (s[1] * F2 + s[2]) * VP;
      if constexpr (T1 * V <= 32) {
        // sum-factorised over o2 with T1 * V independent accumulator chains (ILP for the FP64 pipe)
        double t[T1][V];
#pragma unroll
        for (int o1 = 0; o1 < T1; ++o1)
#pragma unroll
          for (int v = 0; v < V; ++v) t[o1][v] = 0.0;
#pragma unroll
        for (int o2 = 0; o2 < TAPS; ++o2) {
#pragma unroll
          for (int o1 = 0; o1 < T1; ++o1) {
            const double* hp = base + (o1 * F2 + o2) * VP;
#pragma unroll
            for (int v = 0; v < V; ++v) t[o1][v] = fma(w2[o2], hp[v], t[o1][v]);
          }
        }
#pragma unroll
        for (int o1 = 0; o1 < T1; ++o1) {
          const double w01 = wa * w1[o1];
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v] = fma(w01, t[o1][v], acc[v]);
        }
      } else {
        // many values per node: V independent chains per row already
#pragma unroll 2
        for (int o1 = 0; o1 < T1; ++o1) {
          const double* rowp = base + o1 * F2 * VP;
          double t[V];
#pragma unroll
          for (int v = 0; v < V; ++v) t[v] = 0.0;
#pragma unroll
          for (int o2 = 0; o2 < TAPS; ++o2) {
#pragma unroll
            for (int v = 0; v < V; ++v) t[v] = fma(w2[o2], rowp[o2 * VP + v], t[v]);
          }
          const double w01 = wa * w1[o1];
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v] = fma(w01, t[v], acc[v]);
        }
      }
    }
    if (!whole) {
      cp_async_wait<0>();
      __syncthreads();  // plane P consumed; plane P+1 staged
    }
  }
  if (!has) return;
  const long long i = perm[(long long)it.win * n + pidx];
  double* out = part + (((long long)it.win * n + i) * OPS) * r + r0;
#pragma unroll
  for (int q = 0; q < OPS; ++q)
#pragma unroll
    for (int c = 0; c < RC; ++c) out[(long long)q * r + c] = acc[q * RC + c];
}

inline size_t interp_bin_smem(int V, int F0, int F1, int F2, int& whole) {
  const size_t planeb = (size_t)F1 * F2 * ((V + 1) & ~1) * sizeof(double);
  whole = (size_t)F0 * planeb <= 96 * 1024;
  return whole ? F0 * planeb : 2 * planeb;
}

template <int D, int T>
cudaError_t launch_interp_dt(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                             int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                             const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                             const void* tma, cudaStream_t s) {
#define AKM_CASE(O, R)                                                                                              \
  if (ops == O && rc == R) {                                                                                        \
    if (O * R >= 8 && !sparse) {                                                                                    \
      const size_t smem = interp_mma_smem(D, T, O, R);                                                              \
      static std::atomic<unsigned long long> attr_set{0};                                                                                 \
      if (!optin_done(attr_set)) {                                                                                              \
        cudaError_t e = cudaFuncSetAttribute(k_interp_mma<D, T, O, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)smem);                                                            \
        if (e != cudaSuccess) return e;                                                                             \
        optin_mark(attr_set);                                                                                            \
      }                                                                                                             \
      if constexpr (D == 3 && T == 12 && O == 2 && R == 11) {                                                     \
        if (tma && rc == r && r0 == 0) {                                                                            \
          static std::atomic<unsigned long long> attr_tma{0};                                                       \
          if (!optin_done(attr_tma)) {                                                                              \
            cudaError_t e = cudaFuncSetAttribute(k_interp_mma<D, T, O, R, true>,                                    \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 128);     \
            if (e != cudaSuccess) return e;                                                                         \
            optin_mark(attr_tma);                                                                                   \
          }                                                                                                         \
          k_interp_mma<D, T, O, R, true><<<n_items, 256, smem, s>>>(dtab, items, u_sorted, perm, H, r, r0, part, n, \
                                                                   *static_cast<const TmaMaps*>(tma));              \
          return cudaGetLastError();                                                                                \
        }                                                                                                           \
      }                                                                                                             \
      k_interp_mma<D, T, O, R><<<n_items, 256, smem, s>>>(dtab, items, u_sorted, perm, H, r, r0, part, n,         \
                                                         TmaMaps{});                                               \
    } else {                                                                                                        \
      if (n_items_bin <= 0) return cudaSuccess;                                                                     \
      int whole = 0;                                                                                                \
      const size_t smem = interp_bin_smem(O * R, D >= 3 ? Fb2 : 1, Fb1, Fb2, whole);                                \
      static std::atomic<unsigned long long> attr_set{0};                                                                                 \
      if (!optin_done(attr_set)) {                                                                                              \
        cudaError_t e = cudaFuncSetAttribute(k_interp_bin<D, T, O, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             200 * 1024);                                                           \
        if (e != cudaSuccess) return e;                                                                             \
        optin_mark(attr_set);                                                                                            \
      }                                                                                                             \
      k_interp_bin<D, T, O, R><<<n_items_bin, 128, smem, s>>>(dtab, items_bin, u_sorted, perm, H, r, r0, part, n,  \
                                                              whole);                                               \
    }                                                                                                               \
    return cudaGetLastError();                                                                                      \
  }
  AKM_CASE(1, 1) AKM_CASE(1, 2) AKM_CASE(1, 4) AKM_CASE(1, 11)
  AKM_CASE(2, 1) AKM_CASE(2, 2) AKM_CASE(2, 4) AKM_CASE(2, 11)
#undef AKM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace akm
