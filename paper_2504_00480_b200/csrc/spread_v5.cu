// spread_v5.cu -- adjoint NFFT gridding (NFFT step 1 transposed, App. A), the kernel
// for 3-D window groups (plan.cu; 2-D groups take k_spread_strip in spread_strip.cu unless
// AKM_SPREAD_STRIP=0, 1-D windows k_spread_mma, or all windows under AKM_SPREAD_V5=0).
//
// Same GEMM as spread_mma.cu (C[(o0,o1),(o2,c)] = sum_p (w0 w1)[p] (w2 v)[p] on DMMA), but:
//   * 4 MMA warps per CTA (two CTAs per SM at <= 255 registers: one or two MMA warps per SM
//     sub-partition), so each warp can hold up to 9 x 5 DMMA accumulator tiles (tools/microbench/dmma_occupancy.cu: one warp
//     per sub-partition keeps the DMMA pipe busy);
//   * fragments are formed on the fly (A = W0 * W1, B = W2 * V: one independent DMUL each) from
//     the per-point weight rows, so there are no operand panels and no staging phase for them;
//   * the window weights of a batch are a small DMMA product (powers of x times the polynomial
//     coefficients), evaluated for batch b+1 right after the MMAs of batch b (double-buffered);
//     raw inputs stream through a 5-deep cp.async ring;
//   * with small register tiles (few RHS) a warp-specialised variant adds 4 helper warps that run
//     the weights and the ring while the MMA warps stream (named-barrier handshake per batch).
// AKM_SPREAD_V5=0/1 and AKM_V5_WS=0/1 force the kernel choices (A/B measurements).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "akm_internal.cuh"

namespace akm {

namespace {
constexpr int kV5PB = 32;
constexpr int kV5Warps = 4;
constexpr int kV5Threads = 32 * kV5Warps;
constexpr int kV5Ring = 5;
constexpr int kV5LdC = 24;  // coefficient table row stride: rows k, k+1 land 16 banks apart

__device__ __forceinline__ void v5_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void v5_cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void v5_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void v5_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void v5_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void v5_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Row strides of the per-point tables read as fragments.  A half-warp reads 4 points (lane & 3) x 4
// consecutive columns (lane >> 2): a stride of 4 (mod 16) doubles puts the 4 point rows 4 banks
// apart, so the 16 reads hit 16 distinct 8-byte banks (the earlier 8 (mod 16) collided rows p and
// p + 2: 2x the ideal shared-memory wavefronts at c4, ncu).
__host__ __device__ constexpr int v5_ldw(int fmax) { return ((fmax + 1 + 11) / 16) * 16 + 4; }  // 4 mod 16, > fmax
__host__ __device__ constexpr int v5_vld(int rc) { return rc <= 12 ? 12 : ((rc + 11) / 16) * 16 + 4; }  // RHS row
}  // namespace

template <int MB, int NB, bool WS, bool DET>
__global__ void __launch_bounds__(WS ? 2 * kV5Threads : kV5Threads, 1) k_spread_v5(const WinTable* __restrict__ tabp,
                                                             const WorkItem* __restrict__ items,
                                                             const double* __restrict__ u_sorted,
                                                             const int* __restrict__ perm, const double* __restrict__ V,
                                                             long long ldv, long long n, int r0, int rc, int r_total,
                                                             double* __restrict__ grid, int WN,
                                                             const __grid_constant__ PolyParam pp, const DetAcc da) {
  constexpr int PB = kV5PB;
  constexpr int NT = kV5Threads;
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const int d = g.d;
  const int F1 = g.F[1];
  const int Fmax = max(g.F[0], max(F1, g.F[2]));
  const int LDW = v5_ldw(Fmax);
  const int VLD = v5_vld(rc);      // ring row stride of a point's RHS values
  const int VS = PB * VLD + 1;  // ring slot of RHS values + one zero
  const int M = g.F[0] * F1, Nn = g.F[2] * rc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // WS: warps 0-3 run the MMAs, warps 4-7 ("helpers") the weights and the input ring; otherwise
  // the same 4 warps do both, phase after phase
  const int ltid = WS ? (tid & (NT - 1)) : tid, lwarp = WS ? (warp & (kV5Warps - 1)) : warp;
  const int taps = 2 * tab.m;
  const int nbatch = (it.count + PB - 1) / PB;
  const float inv_rc = 1.0f / rc;

  extern __shared__ double smem[];
  double* Wb = smem;                                    // [2][3][PB][LDW] weights (zero slot LDW-1)
  double* Vring = Wb + 2 * 3 * PB * LDW;                // [R][PB*rc + 1]
  double* Uring = Vring + kV5Ring * VS;                 // [R][3][PB]
  double* Cs = Uring + kV5Ring * 3 * PB;                // [16 powers][kV5LdC] window coefficients
  int* Pring = reinterpret_cast<int*>(Cs + 16 * kV5LdC);  // [R][PB]
  const int wm = warp / WN, wn = warp % WN;

  int org[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) org[a] = g.box_lo[a] + it.bin[a] * g.B;
  constexpr int NALL = WS ? 2 * NT : NT;
  for (int idx = tid; idx < 2 * 3 * PB * LDW; idx += NALL) Wb[idx] = 0.0;
  for (int s = tid; s < kV5Ring; s += NALL) Vring[s * VS + PB * VLD] = 0.0;
  for (int idx = tid; idx < 16 * kV5LdC; idx += NALL) {
    const int k = idx / kV5LdC, q = idx - k * kV5LdC;
    Cs[idx] = (k < kPolyLen && q < taps) ? pp.c[q * kPolyLen + k] : 0.0;
  }

  const long long ptbase = (long long)it.win * n + it.start;
  const double* ubase = u_sorted + (long long)it.win * 3 * n + it.start;
  auto issue_perm = [&](int b) {
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    if (ltid < pb) v5_cp4(Pring + (b % kV5Ring) * PB + ltid, perm + ptbase + q0 + ltid);
  };
  auto issue_u = [&](int b) {
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    for (int j = ltid; j < 3 * PB; j += NT) {
      const int a = j / PB, p = j - a * PB;
      if (a >= 3 - d && p < pb) v5_cp8(Uring + ((b % kV5Ring) * 3 + a) * PB + p, ubase + (long long)a * n + q0 + p);
    }
  };
  auto issue_v = [&](int b) {  // needs Pring[b] visible
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    double* Vs = Vring + (b % kV5Ring) * VS;
    const int* pr = Pring + (b % kV5Ring) * PB;
    for (int j = ltid; j < PB * rc; j += NT) {
      const int p = fdiv(j, inv_rc), c = j - p * rc;
      double* dst = Vs + p * VLD + c;
      if (p < pb) v5_cp8(dst, V + (long long)pr[p] * ldv + r0 + c);
      else *dst = 0.0;
    }
  };
  // weights of batch b into Wb[b&1], on the tensor core: for the 3*PB (axis, point) rows,
  // W[(a,p)][q] = sum_k x_{a,p}^k c[q][k] is a (96 x 16) x (16 x 16) product (powers x taps), so
  // the window polynomials cost 24 DMMAs per warp and a handful of DMULs instead of a scalar FP64
  // phase (scalar FP64 next to a DMMA stream is starved).  Warp w owns row
  // tiles 3w..3w+2; each lane writes the taps of its own row at nodes s0 + q and zeroes the rest.
  // NTL of the warp's three row tiles at a time (interleaved for latency; fewer with big register
  // tiles, where the accumulators leave no room)
  auto wtiles = [&](int b, int t0, auto ntl) {
    constexpr int NTL = decltype(ntl)::value;
    const int pb = min(PB, it.count - b * PB);
    const double* U = Uring + (b % kV5Ring) * 3 * PB;
    double* W = Wb + (b & 1) * 3 * PB * LDW;
    const int j4 = lane & 3;
    double xp[NTL], x4[NTL], c0[NTL][2], c1[NTL][2];
    int s0[NTL];
#pragma unroll
    for (int t = 0; t < NTL; ++t) {
      const int R = (lwarp * 3 + t0 + t) * 8 + (lane >> 2), a = R / PB, p = R - a * PB;
      const bool real = p < pb && a >= 3 - d;
      const double u = real ? U[a * PB + p] : 0.5;
      const double fl = floor(u);
      s0[t] = (int)fl - tab.m + 1 - org[a];
      const double x = 2.0 * (u - fl) - 1.0;
      const double x2 = x * x;
      x4[t] = x2 * x2;
      xp[t] = j4 == 0 ? 1.0 : (j4 == 1 ? x : (j4 == 2 ? x2 : x2 * x));
      c0[t][0] = c0[t][1] = c1[t][0] = c1[t][1] = 0.0;
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const double* cr = Cs + (4 * kk + j4) * kV5LdC + (lane >> 2);
      const double b0 = cr[0], b1 = cr[8];
#pragma unroll
      for (int t = 0; t < NTL; ++t) {
        dmma(c0[t][0], c0[t][1], xp[t], b0);
        dmma(c1[t][0], c1[t][1], xp[t], b1);
      }
#pragma unroll
      for (int t = 0; t < NTL; ++t) xp[t] *= x4[t];
    }
#pragma unroll
    for (int t = 0; t < NTL; ++t) {
      const int R = (lwarp * 3 + t0 + t) * 8 + (lane >> 2), a = R / PB, p = R - a * PB;
      const bool live = p < pb, real = live && a >= 3 - d;
      double* wrow = W + (a * PB + p) * LDW;
      const int Fa = g.F[a], s = s0[t];
      if (real) {
        const int q0 = 2 * j4;
        if (s + q0 < Fa) wrow[s + q0] = c0[t][0];
        if (s + q0 + 1 < Fa) wrow[s + q0 + 1] = c0[t][1];
        if (s + q0 + 8 < Fa) wrow[s + q0 + 8] = c1[t][0];
        if (s + q0 + 9 < Fa) wrow[s + q0 + 9] = c1[t][1];
        for (int o = j4; o < s; o += 4) wrow[o] = 0.0;
        for (int o = s + 16 + j4; o < Fa; o += 4) wrow[o] = 0.0;
      } else {
        const double fill = (live && a < 3 - d) ? 1.0 : 0.0;
        for (int o = j4; o < Fa; o += 4) wrow[o] = fill;
      }
    }
  };
  auto wgemm = [&](int b) {
    if constexpr (WS) {  // helpers hold no accumulators: all three tiles interleaved
      wtiles(b, 0, std::integral_constant<int, 3>{});
    } else if constexpr (MB * NB >= 45) {
#pragma unroll 1
      for (int t = 0; t < 3; ++t) wtiles(b, t, std::integral_constant<int, 1>{});
    } else if constexpr (MB * NB >= 36) {
      wtiles(b, 0, std::integral_constant<int, 2>{});
      wtiles(b, 2, std::integral_constant<int, 1>{});
    } else {
      wtiles(b, 0, std::integral_constant<int, 3>{});
    }
  };

  if constexpr (WS) {
    __syncthreads();  // initialised tables
    if (warp >= kV5Warps) {
      // helpers: per batch b, wait until the MMA warps released W[b&1] (batch b-2), evaluate the
      // weights of b, issue the loads of later batches, then hand W[b&1] and V(b) over
      for (int b = 0; b < 4; ++b) issue_perm(b);
      for (int b = 0; b < 3; ++b) issue_u(b);
      v5_commit();
      v5_wait_all();
      v5_bar_sync(5, NT);
      for (int b = 0; b < 3; ++b) issue_v(b);
      v5_commit();
      for (int b = 0; b < nbatch; ++b) {
        if (b >= 2) v5_bar_sync(3 + (b & 1), 2 * NT);  // FREE: batch b-2 consumed
        v5_wait_all();
        v5_bar_sync(5, NT);  // every helper's copies visible to all helpers
        wgemm(b);
        issue_perm(b + 4);
        issue_u(b + 3);
        issue_v(b + 3);
        v5_commit();
        v5_bar_arrive(1 + (b & 1), 2 * NT);  // READY: W(b), V(b)
      }
      for (int b = max(nbatch, 2); b < nbatch + 2; ++b) v5_bar_sync(3 + (b & 1), 2 * NT);
      v5_wait_all();
      return;
    }
  } else {
    // prologue: perm 0..3, u 0..2, then V 0..2 and the weights of batch 0
    for (int b = 0; b < 4; ++b) issue_perm(b);
    for (int b = 0; b < 3; ++b) issue_u(b);
    v5_commit();
    v5_wait_all();
    __syncthreads();
    for (int b = 0; b < 3; ++b) issue_v(b);
    v5_commit();
    wgemm(0);
    v5_wait_all();
    __syncthreads();
  }

  // fragment coordinates (invalid rows / columns point at the zero weight slot)
  unsigned ai[MB], bi[NB];  // (w0 row | w1 row << 16), (w2 row | rhs << 16)
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int row = (wm * MB + i) * 8 + (lane >> 2);
    const bool ok = row < M;
    ai[i] = ok ? (unsigned)(row / F1) | ((unsigned)(row - (row / F1) * F1) << 16) : (unsigned)(LDW - 1) * 0x10001u;
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int col = (wn * NB + j) * 8 + (lane >> 2);
    const bool ok = col < Nn;
    bi[j] = ok ? (unsigned)(col / rc) | ((unsigned)(col - (col / rc) * rc) << 16) : (unsigned)(LDW - 1);
  }

  double acc[MB][NB][2];
#pragma unroll
  for (int i = 0; i < MB; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int b = 0; b < nbatch; ++b) {
    if constexpr (WS) v5_bar_sync(1 + (b & 1), 2 * NT);  // READY
    const double* W0 = Wb + (b & 1) * 3 * PB * LDW;
    const double* W1 = W0 + PB * LDW;
    const double* W2 = W1 + PB * LDW;
    const double* Vs = Vring + (b % kV5Ring) * VS;
    const int ksteps = (min(PB, it.count - b * PB) + 3) >> 2;
#pragma unroll 1
    for (int ks = 0; ks < ksteps; ++ks) {
      const int p = ks * 4 + (lane & 3);
      const double* w0 = W0 + p * LDW;
      const double* w1 = W1 + p * LDW;
      const double* w2 = W2 + p * LDW;
      const double* vs = Vs + p * VLD;
      double af[MB], bf[NB];
#pragma unroll
      for (int i = 0; i < MB; ++i) af[i] = w0[ai[i] & 0xffff] * w1[ai[i] >> 16];
#pragma unroll
      for (int j = 0; j < NB; ++j) bf[j] = w2[bi[j] & 0xffff] * vs[bi[j] >> 16];
#pragma unroll
      for (int i = 0; i < MB; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if constexpr (WS) {
      v5_bar_arrive(3 + (b & 1), 2 * NT);  // FREE
    } else {
      if (b + 1 < nbatch) wgemm(b + 1);  // the next batch's weights (its coordinates have landed)
      v5_wait_all();                     // V(b+1..), u(b+2..), perm(b+3..) issued earlier
      __syncthreads();
      issue_perm(b + 4);
      issue_u(b + 3);
      issue_v(b + 3);
      v5_commit();
    }
  }

  // flush
  const long long L1 = g.L[1], L2 = g.L[2], toff = g.tap_off;
  const int c0 = org[0] - g.box_lo[0], c1 = org[1] - g.box_lo[1], c2 = org[2] - g.box_lo[2];
  const float inv_F1 = 1.0f / F1;
  double* gbase = grid + r0;
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int row = (wm * MB + i) * 8 + (lane >> 2);
    if (row >= M) continue;
    const int o0 = fdiv(row, inv_F1);
    const long long line = ((long long)(c0 + o0) * L1 + (c1 + row - o0 * F1)) * L2 + c2;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = (wn * NB + j) * 8 + 2 * (lane & 3) + h;
        const double v = acc[i][j][h];
        if (col >= Nn || v == 0.0) continue;
        const int o2 = fdiv(col, inv_rc);
        if constexpr (DET) det_add(da, it.win, (toff + line + o2) * r_total + r0 + (col - o2 * rc), r0 + (col - o2 * rc), v);
        else atomicAdd(gbase + (toff + line + o2) * r_total + (col - o2 * rc), v);
      }
    }
  }
}

#define AKM_V5_TILES(X) X(9, 5) X(5, 9) X(9, 4) X(4, 9) X(6, 6) X(6, 3) X(3, 6) X(3, 7) X(3, 4) X(6, 2) X(3, 2) X(2, 2) X(1, 2)

bool spread_v5_choose(int M, int Nn, int& MB, int& NB, int& WN) {
  static const int cand[][2] = {
#define AKM_PAIR(a, b) {a, b},
      AKM_V5_TILES(AKM_PAIR)
#undef AKM_PAIR
  };
  const int TMt = (M + 7) / 8, TNt = (Nn + 7) / 8;
  double best = 1e300;
  bool found = false;
  for (auto& c : cand) {
    const int mb = c[0], nb = c[1];
    for (int wm = 1; wm <= kV5Warps; wm *= 2) {
      const int wn = kV5Warps / wm;
      if (wm * mb < TMt || wn * nb < TNt) continue;
      const double score = (double)mb * nb * (1.0 + 0.5 * (double)(mb + nb) / (mb * nb));
      if (score < best) {
        best = score;
        MB = mb;
        NB = nb;
        WN = wn;
        found = true;
      }
    }
  }
  return found;
}

size_t spread_v5_smem(int Fmax, int rc, int MB, int NB, int WN) {
  (void)MB, (void)NB, (void)WN;
  return sizeof(double) * (2 * 3 * (size_t)kV5PB * v5_ldw(Fmax) + (size_t)kV5Ring * (kV5PB * v5_vld(rc) + 1) +
                           (size_t)kV5Ring * 3 * kV5PB + 16 * kV5LdC) +
         sizeof(int) * (size_t)kV5Ring * kV5PB;
}

cudaError_t launch_spread_v5(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                             const double* u_sorted, const int* perm, const double* V, long long ldv, long long n,
                             int r0, int rc, int r_total, double* grid, int MB, int NB, int WN, size_t smem,
                             cudaStream_t s, const DetAcc& da) {
  if (n_items <= 0) return cudaSuccess;
  // warp-specialised variant for small register tiles (few RHS, e.g. c2: the helpers' latency-bound
  // weight and ring work overlaps the MMAs) and for launches with fewer than 2 x 148 work items
  // (c1: nothing to hide behind); with big tiles and many items the helpers' scalar FP64 on the same
  // SM sub-partitions slows the DMMA stream more than it hides
  static const int ws_env = getenv("AKM_V5_WS") ? atoi(getenv("AKM_V5_WS")) : -1;
  const bool ws = ws_env >= 0 ? ws_env != 0 : (MB * NB <= 12 || n_items < 2 * 148);
// DET (deterministic integer-limb flush) is a template parameter: a runtime branch in the flush
// changed the register allocation of the MMA loop (c4 spreading 6.97 -> 7.27 ms)
#define AKM_CASE2(a, b, o, det)                                                                                \
  if (MB == a && NB == b && ws == o && (da.limbs != nullptr) == det) {                                         \
    static std::atomic<unsigned long long> attr_set{0};                                                         \
    if (!optin_done(attr_set)) {                                                                                \
      cudaError_t e = cudaFuncSetAttribute(k_spread_v5<a, b, o, det>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           227 * 1024);                                                         \
      if (e != cudaSuccess) return e;                                                                           \
      optin_mark(attr_set);                                                                                     \
    }                                                                                                           \
    k_spread_v5<a, b, o, det><<<n_items, o ? 2 * kV5Threads : kV5Threads, smem, s>>>(                           \
        dtab, items, u_sorted, perm, V, ldv, n, r0, rc, r_total, grid, WN, pp, da);                              \
    return cudaGetLastError();                                                                                  \
  }
#define AKM_CASE1(a, b, o) AKM_CASE2(a, b, o, false) AKM_CASE2(a, b, o, true)
#define AKM_CASE(a, b) AKM_CASE1(a, b, true) AKM_CASE1(a, b, false)
  AKM_V5_TILES(AKM_CASE)
#undef AKM_CASE
#undef AKM_CASE1
#undef AKM_CASE2
  return cudaErrorInvalidValue;
}

}  // namespace akm
