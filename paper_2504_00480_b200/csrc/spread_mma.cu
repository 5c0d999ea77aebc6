// spread_mma.cu -- adjoint NFFT gridding on the FP64 tensor pipe (App. A,
// P:1201-1211; inner sums of eq. 3.3):
//
//   g^{w,c}_l = sum_j V[j,c] phi~(x~_j^w - l/n_g)
//
// Per work item (a chunk of points of one bin of B^d cells) the bin's footprint accumulator is
//   C[(o0,o1), (c,o2)] = sum_p (w0_p[o0] w1_p[o1]) * (v_p[c] w2_p[o2])   = A^T B,
// a GEMM with K = points, run on DMMA (mma.sync.m8n8k4.f64): on B200 DMMA and DFMA share one FP64
// pipe (37 TFLOP/s, profiles/r01_fp64_peaks.txt) but one DMMA instruction carries 256 FMAs, so
// operand delivery and issue stop limiting and the accumulator lives in MMA fragments.
//
// Phased design.  Measured on B200 (tools/microbench/dmma_occupancy.cu and the
// round-1 ncu captures): while one warp streams DMMAs, a DFMA/DMUL of ANOTHER warp on the same SM
// sub-partition is granted the FP64 pipe only every ~34 clk.  Any scalar FP64 work overlapped with
// DMMAs of other warps (on-the-fly fragment products, producer warps building panels) therefore
// starves and stalls the MMAs behind it.  So every batch of PB points runs in two phases, all
// 8 warps (2 per sub-partition) together:
//   STAGE  window weights (Estrin polynomials, independent chains) and the two factor panels
//          A[p][(o0,o1)] = w0 w1, B[p][(o2,c)] = w2 v in shared memory -- no DMMA in flight;
//   MMA    C += A^T B: fragments are single conflict-free LDS.64 (panel row stride = 4 mod 16
//          doubles) straight into DMMA -- no scalar FP64 in flight.
// Raw inputs (grid coordinates, permutation, RHS values gathered through it) stream in through a
// cp.async ring a few batches ahead, so neither phase waits on global memory.  The footprint is
// written once per work item with RED.ADD.F64.
#include <algorithm>

#include "akm_internal.cuh"

namespace akm {

// points per batch: 64 (16 MMA k-steps) for large register tiles; 32 for small tiles (MB*NB <= 12,
// the small-RHS footprints), whose CTAs are then capped at 128 registers and half the shared
// memory so that two CTAs share an SM and one's staging overlaps the other's DMMAs
__host__ __device__ constexpr int spread_pb(int mb, int nb) { return mb * nb <= 12 ? 32 : 64; }
__host__ __device__ constexpr int spread_minb(int mb, int nb) { return mb * nb <= 12 ? 2 : 1; }
constexpr int kSpreadWarps = 8;      // two per SM sub-partition
constexpr int kSpreadThreads = 32 * kSpreadWarps;
constexpr int kRing = 4;             // cp.async ring depth (batches)

__device__ __forceinline__ void cpasync8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cpasync4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__host__ __device__ constexpr int spread_ldf(int f) { return (f + 2) & ~1; }  // weight row: even, > f

template <int MB, int NB, bool DET>
__global__ void __launch_bounds__(kSpreadThreads, spread_minb(MB, NB)) k_spread_mma(const WinTable* __restrict__ tabp,
                                                                  const WorkItem* __restrict__ items,
                                                                  const double* __restrict__ u_sorted,
                                                                  const int* __restrict__ perm,
                                                                  const double* __restrict__ V, long long ldv,
                                                                  long long n, int r0, int rc, int r_total,
                                                                  double* __restrict__ grid, int WN,
                                                                  const __grid_constant__ PolyParam pp,
                                                                  const DetAcc da) {
  constexpr int PB = spread_pb(MB, NB);
  constexpr int NT = kSpreadThreads;
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const int d = g.d;
  const int F1 = g.F[1];
  const int Fmax = max(g.F[0], max(F1, g.F[2]));
  const int LDF = spread_ldf(Fmax);
  const int M = g.F[0] * F1, Nn = g.F[2] * rc;
  const int WM = kSpreadWarps / WN;
  const int lda = mma_ld(WM * MB * 8), ldb = mma_ld(WN * NB * 8);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int taps = 2 * tab.m;
  const int nbatch = (it.count + PB - 1) / PB;
  const float inv_rc = 1.0f / rc, inv_F1 = 1.0f / F1, inv_F2 = 1.0f / g.F[2];

  extern __shared__ double smem[];
  double* As = smem;                               // [PB][lda]
  double* Bs = As + PB * lda;                      // [PB][ldb]
  double* Ws = Bs + PB * ldb;                      // [3][PB][LDF]  weights on the footprint
  double* Vring = Ws + 3 * PB * LDF;               // [R][PB][rc]   RHS values        (cp.async ring)
  double* Uring = Vring + kRing * PB * rc;         // [R][3][PB]    grid coordinates  (cp.async ring)
  int* Pring = reinterpret_cast<int*>(Uring + kRing * 3 * PB);  // [R][PB] permutation (cp.async ring)

  int org[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) org[a] = g.box_lo[a] + it.bin[a] * g.B;
  // panels: the padding rows / columns (>= M, >= Nn) are never written and stay zero
  for (int idx = tid; idx < PB * (lda + ldb); idx += NT) As[idx] = 0.0;

  const long long ptbase = (long long)it.win * n + it.start;
  const double* ubase = u_sorted + (long long)it.win * 3 * n + it.start;
  // ring schedule: at batch b the permutation of b+3, the coordinates of b+2 and the RHS values of
  // b+1 (gathered through the permutation, which landed a batch earlier) are issued
  auto issue_perm = [&](int b) {
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    if (tid < pb) cpasync4(Pring + (b % kRing) * PB + tid, perm + ptbase + q0 + tid);
  };
  auto issue_u = [&](int b) {
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    for (int j = tid; j < 3 * PB; j += NT) {
      const int a = j / PB, p = j - a * PB;
      if (a >= 3 - d && p < pb) cpasync8(Uring + ((b % kRing) * 3 + a) * PB + p, ubase + (long long)a * n + q0 + p);
    }
  };
  auto issue_v = [&](int b) {  // needs Pring[b] visible to all threads
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    double* Vs = Vring + (b % kRing) * PB * rc;
    const int* pr = Pring + (b % kRing) * PB;
    for (int j = tid; j < PB * rc; j += NT) {
      const int p = fdiv(j, inv_rc), c = j - p * rc;
      if (p < pb) cpasync8(Vs + j, V + (long long)pr[p] * ldv + r0 + c);
      else Vs[j] = 0.0;  // absent points: zero (0 * a stale NaN would poison the panel)
    }
  };
  for (int b = 0; b < 3; ++b) issue_perm(b);
  for (int b = 0; b < 2; ++b) issue_u(b);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  issue_v(0);
  cp_async_commit();

  const int wm = warp / WN, wn = warp % WN;
  double acc[MB][NB][2];
#pragma unroll
  for (int i = 0; i < MB; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int aoff = (lane & 3) * lda + wm * MB * 8 + (lane >> 2);
  const int boff = (lane & 3) * ldb + wn * NB * 8 + (lane >> 2);

  for (int b = 0; b < nbatch; ++b) {
    const int pb = min(PB, it.count - b * PB);
    const double* Vc = Vring + (b % kRing) * PB * rc;
    const double* U = Uring + (b % kRing) * 3 * PB;
    // ---- STAGE.  u(b), V(b) and perm(b+1) have landed (issued >= 1 batch ago); the previous
    //      batch's MMAs are done (panels free)
    cp_async_wait<0>();
    __syncthreads();
    issue_perm(b + 3);
    issue_u(b + 2);
    issue_v(b + 1);
    cp_async_commit();
    // window weights: one job per (point, axis) (PB * 3 <= 256 threads), all 2m taps by Estrin
    // (independent chains of depth 4; coefficients are constant-bank operands)
    for (int job = tid; job < PB * 3; job += NT) {
      const int p = job / 3, a = job - 3 * p;
      double* wrow = Ws + (a * PB + p) * LDF;
      const int Fa = g.F[a];
      if (p >= pb || a < 3 - d) {
        const double fill = (p < pb) ? 1.0 : 0.0;  // singleton axis: F = 1, weight 1
        for (int o = 0; o < Fa; ++o) wrow[o] = fill;
        continue;
      }
      const double u = U[a * PB + p];
      const double fl = floor(u);
      const int s0 = (int)fl - tab.m + 1 - org[a];  // footprint position of the point's tap 0
      const double x = 2.0 * (u - fl) - 1.0;
      for (int o = 0; o < s0; ++o) wrow[o] = 0.0;
      for (int o = s0 + taps; o < Fa; ++o) wrow[o] = 0.0;
      double wv[kMaxTaps];
      if (taps == 12) window_taps_estrin<12>(pp.c, x, wv);
      else if (taps == 8) window_taps_estrin<8>(pp.c, x, wv);
      else window_taps_estrin<16>(pp.c, x, wv);
#pragma unroll
      for (int q = 0; q < kMaxTaps; ++q)
        if (q < taps) wrow[s0 + q] = wv[q];
    }
    __syncthreads();
    // factor panels.  A[p][o0*F1 + o1] = w0[o0] w1[o1]: one job per (point, o0) writes F1
    // consecutive doubles; B[p][c*F2 + o2] = v[c] w2[o2] (columns ordered (c, o2)): one job per
    // (point, c) writes F2 consecutive doubles.  Even runs go as 16-byte vectors (weight rows and
    // panel rows are 16-byte aligned: LDF, lda, ldb even); consecutive threads take consecutive
    // points (row strides = 4 mod 16 doubles spread the stores over the banks).
    {
      const double* W0 = Ws;
      const double* W1 = Ws + PB * LDF;
      const double* W2 = Ws + 2 * PB * LDF;
      const int F0 = g.F[0], F2 = g.F[2];
      if ((F1 & 1) == 0) {  // one job per (point, o0, pair of o1): enough jobs when F0 = 1 (d = 2)
        const int H1 = F1 >> 1;
        for (int job = tid; job < PB * F0 * H1; job += NT) {
          const int po = job / H1, h = job - po * H1;
          const int o0 = po / PB, p = po - o0 * PB;
          const double w0 = W0[p * LDF + o0];
          const double2 t = *reinterpret_cast<const double2*>(W1 + p * LDF + 2 * h);
          *reinterpret_cast<double2*>(As + p * lda + o0 * F1 + 2 * h) = make_double2(w0 * t.x, w0 * t.y);
        }
      } else {
        for (int job = tid; job < PB * F0; job += NT) {
          const int o0 = job / PB, p = job - o0 * PB;
          const double w0 = W0[p * LDF + o0];
          const double* w1 = W1 + p * LDF;
          double* dst = As + p * lda + o0 * F1;
          for (int o = 0; o < F1; ++o) dst[o] = w0 * w1[o];
        }
      }
      for (int job = tid; job < PB * rc; job += NT) {
        const int c = job / PB, p = job - c * PB;
        const double v = Vc[p * rc + c];
        const double* w2 = W2 + p * LDF;
        double* dst = Bs + p * ldb + c * F2;
        if ((F2 & 1) == 0) {
          for (int o = 0; o < F2; o += 2) {
            const double2 t = *reinterpret_cast<const double2*>(w2 + o);
            *reinterpret_cast<double2*>(dst + o) = make_double2(v * t.x, v * t.y);
          }
        } else {
          for (int o = 0; o < F2; ++o) dst[o] = v * w2[o];
        }
      }
    }
    __syncthreads();
    // ---- MMA
    const double* ap = As + aoff;
    const double* bp = Bs + boff;
    const int ksteps = (pb + 3) >> 2;
#pragma unroll 1
    for (int ks = 0; ks < ksteps; ++ks) {
      double af[MB];
#pragma unroll
      for (int i = 0; i < MB; ++i) af[i] = ap[i * 8];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const double bfj = bp[j * 8];
#pragma unroll
        for (int i = 0; i < MB; ++i) dmma(acc[i][j][0], acc[i][j][1], af[i], bfj);
      }
      ap += 4 * lda;
      bp += 4 * ldb;
    }
  }

  // flush: fragment (row = lane>>2, cols 2*(lane&3) + {0,1}) of each owned tile; table fields are
  // read once (the atomics would otherwise force re-loads of the global table)
  const long long L1 = g.L[1], L2 = g.L[2], toff = g.tap_off;
  const int b0 = org[0] - g.box_lo[0], b1 = org[1] - g.box_lo[1], b2 = org[2] - g.box_lo[2];
  double* gbase = grid + r0;
  const int F2 = g.F[2];
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int row = (wm * MB + i) * 8 + (lane >> 2);
    if (row >= M) continue;
    const int o0 = fdiv(row, inv_F1);
    const long long line = ((long long)(b0 + o0) * L1 + (b1 + row - o0 * F1)) * L2 + b2;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = (wn * NB + j) * 8 + 2 * (lane & 3) + h;
        const double v = acc[i][j][h];
        if (col >= Nn || v == 0.0) continue;
        const int c = fdiv(col, inv_F2), o2 = col - c * F2;  // B columns are ordered (c, o2)
        if constexpr (DET) det_add(da, it.win, (toff + line + o2) * r_total + r0 + c, r0 + c, v);
        else atomicAdd(gbase + (toff + line + o2) * r_total + c, v);
      }
    }
  }
}

// (MB, NB) register tiles of the 8 warps (WM x WN = 8); an 8x8 f64 accumulator tile costs 4
// registers per thread, MB x NB <= 45 keeps a thread under the 255-register cap
#define AKM_MMA_TILES(X)                                                                                      \
  X(9, 5) X(5, 9) X(9, 4) X(4, 9) X(6, 6) X(9, 3) X(3, 9) X(6, 3) X(3, 6) X(3, 7) X(7, 3) X(12, 2) X(2, 12) X(3, 4)  \
  X(6, 2) X(2, 6) X(4, 4) X(3, 3) X(4, 2) X(2, 4) X(3, 2) X(2, 3) X(2, 2) X(1, 6) X(1, 3) X(1, 2)

static size_t spread_smem_for(int lda, int ldb, int Fmax, int rc, int PB) {
  return sizeof(double) * ((size_t)PB * (lda + ldb) + 3 * (size_t)PB * spread_ldf(Fmax) + (size_t)kRing * PB * (rc + 3)) +
         sizeof(int) * (size_t)kRing * PB;
}

bool spread_mma_choose(int M, int Nn, int Fmax, int rc, int& MB, int& NB, int& WM, int& WN) {
  static const int cand[][2] = {
#define AKM_PAIR(a, b) {a, b},
      AKM_MMA_TILES(AKM_PAIR)
#undef AKM_PAIR
  };
  const int TMt = (M + 7) / 8, TNt = (Nn + 7) / 8;
  double best = 1e300;
  bool found = false;
  for (auto& c : cand) {
    const int mb = c[0], nb = c[1];
    for (int wm = 1; wm <= kSpreadWarps; wm *= 2) {
      const int wn = kSpreadWarps / wm;
      if (wm * mb < TMt || wn * nb < TNt) continue;
      // panels (and the worst-case scratch) must fit the 227 KB of a CTA
      if (spread_smem_for(mma_ld(wm * mb * 8), mma_ld(wn * nb * 8), Fmax, rc, spread_pb(mb, nb)) > 224 * 1024) continue;
      // time ~ DMMA slots per sub-partition (incl. padding tiles) + fragment loads per k-step
      const double slots = (double)mb * nb;
      const double score = slots * (1.0 + 0.25 * (double)(mb + nb) / (mb * nb));
      if (score < best) {
        best = score;
        MB = mb;
        NB = nb;
        WM = wm;
        WN = wn;
        found = true;
      }
    }
  }
  return found;
}

size_t spread_mma_smem(int /*PB*/, int M, int Nn, int Fmax, int rc) {
  int MB, NB, WM, WN;
  if (!spread_mma_choose(M, Nn, Fmax, rc, MB, NB, WM, WN)) return 0;
  return spread_smem_for(mma_ld(WM * MB * 8), mma_ld(WN * NB * 8), Fmax, rc, spread_pb(MB, NB));
}

cudaError_t launch_spread_mma(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                              const double* u_sorted, const int* perm, const double* V, long long ldv, long long n,
                              int r0, int rc, int r_total, double* grid, int MB, int NB, int /*WM*/, int WN,
                              int /*PB*/, size_t smem, cudaStream_t s, const DetAcc& da) {
  if (n_items <= 0) return cudaSuccess;
#define AKM_CASE1(a, b, det)                                                                                   \
  if (MB == a && NB == b && (da.limbs != nullptr) == det) {                                                    \
    static std::atomic<unsigned long long> attr_set{0};                                                         \
    if (!optin_done(attr_set)) {                                                                                \
      cudaError_t e = cudaFuncSetAttribute(k_spread_mma<a, b, det>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           227 * 1024);                                                         \
      if (e != cudaSuccess) return e;                                                                           \
      optin_mark(attr_set);                                                                                     \
    }                                                                                                           \
    k_spread_mma<a, b, det><<<n_items, kSpreadThreads, smem, s>>>(dtab, items, u_sorted, perm, V, ldv, n, r0, rc, \
                                                                  r_total, grid, WN, pp, da);                   \
    return cudaGetLastError();                                                                                  \
  }
#define AKM_CASE(a, b) AKM_CASE1(a, b, false) AKM_CASE1(a, b, true)
  AKM_MMA_TILES(AKM_CASE)
#undef AKM_CASE
#undef AKM_CASE1
  return cudaErrorInvalidValue;
}

}  // namespace akm
