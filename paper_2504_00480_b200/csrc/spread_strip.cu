// spread_strip.cu -- adjoint NFFT gridding (NFFT step 1 transposed, App. A) for 2-D
// windows, one DMMA GEMM per strip of cells:
//
//   C_s[i][(o2, c)] = sum_{p in strip s} w1[p][i] (w2 v)[p][(o2, c)]      i = 0 .. 2m-1 (exact)
//   footprint[s + i][(o2, c)] += C_s[i][(o2, c)]                          (shared memory)
//
// A work item is a chunk of the points of one bin (B x B cells; k_spread_v5's items); inside a bin
// the points are sorted by cell, axis 1 major (binsort.cu slot_key), so the points of one cell row
// s (a strip of 1 x B cells) are consecutive and their axis-1 taps are exactly footprint rows
// s .. s + 2m - 1.  Rows relative to the strip make the GEMM's M dimension the 2m taps (2 DMMA row
// tiles at m = 8) instead of the F = B + 2m - 1 footprint rows padded to 8 (c3: 24 rows for 16
// taps); at a strip change each warp adds its register tiles into the shared-memory footprint at
// row offset s (warps own disjoint columns: no races) and restarts from zero.  A k-step whose four
// points straddle a strip change runs once per strip with the other points masked.  The footprint
// leaves the CTA once per item with RED.ADD.F64, as in k_spread_v5.
//
// Everything else follows k_spread_v5 (4 warps, fragments formed on the fly, window weights of the
// next batch on DMMA, 5-deep cp.async ring of the raw inputs); B = w2 * v (one DMUL), A = w1 (no
// multiply: axis 0 is a singleton).  AKM_SPREAD_STRIP=0 keeps k_spread_v5 (A/B).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "akm_internal.cuh"

namespace akm {

namespace {
constexpr int kSsPB = 32;
static_assert(kSsPB == 32, "k_spread_strip reads one point's strip per lane (S1[lane]) and ballots over a batch");
constexpr int kSsWarps = 4;
constexpr int kSsThreads = 32 * kSsWarps;
constexpr int kSsRing = 5;
constexpr int kSsLdC = 24;

__device__ __forceinline__ void ss_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void ss_cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void ss_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void ss_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// table row strides = 4 (mod 16) doubles: the 4 points of a half-warp's fragment reads land 4 banks
// apart (spread_v5.cu v5_ldw)
__host__ __device__ constexpr int ss_ldw(int fmax) { return ((fmax + 1 + 11) / 16) * 16 + 4; }  // 4 mod 16, > fmax
__host__ __device__ constexpr int ss_vld(int rc) { return rc <= 12 ? 12 : ((rc + 11) / 16) * 16 + 4; }
__host__ __device__ constexpr int ss_ldc(int nb) { return ((4 * nb * 8 + 15) / 16) * 16 + 8; }  // 8 mod 16

struct SsLayout {
  size_t wb, vring, uring, cs, pring, s1b, cacc, total;  // byte offsets
};
__host__ __device__ inline SsLayout ss_layout(int F, int rc, int NB) {
  SsLayout l;
  const int LDW = ss_ldw(F);
  l.wb = 0;
  l.vring = l.wb + sizeof(double) * 2 * 3 * kSsPB * LDW;
  l.uring = (l.vring + sizeof(double) * kSsRing * (kSsPB * ss_vld(rc) + 1) + 15) & ~(size_t)15;
  l.cs = l.uring + sizeof(double) * kSsRing * 3 * kSsPB;
  l.cacc = (l.cs + sizeof(double) * 16 * kSsLdC + 15) & ~(size_t)15;  // double2 accesses
  l.pring = l.cacc + sizeof(double) * (size_t)F * ss_ldc(NB);
  l.s1b = l.pring + sizeof(int) * kSsRing * kSsPB;
  l.total = l.s1b + sizeof(int) * 2 * kSsPB;
  return l;
}
}  // namespace

template <int TAPS, int NB, bool DET>
__global__ void __launch_bounds__(kSsThreads, 2) k_spread_strip(const WinTable* __restrict__ tabp,
                                                               const WorkItem* __restrict__ items,
                                                               const double* __restrict__ u_sorted,
                                                               const int* __restrict__ perm,
                                                               const double* __restrict__ V, long long ldv,
                                                               long long n, int r0, int rc, int r_total,
                                                               double* __restrict__ grid,
                                                               const __grid_constant__ PolyParam pp,
                                                               const DetAcc da) {
  constexpr int PB = kSsPB;
  constexpr int NT = kSsThreads;
  constexpr int MT = (TAPS + 7) / 8;  // row tiles: the strip's 2m axis-1 taps
  constexpr int LDC = ss_ldc(NB);
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const int F1 = g.F[1], F2 = g.F[2];
  const int LDW = ss_ldw(max(F1, F2));
  const int VLD = ss_vld(rc);  // ring row stride of a point's RHS values
  const int VS = PB * VLD + 1;
  const int Nn = F2 * rc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nbatch = (it.count + PB - 1) / PB;
  const float inv_rc = 1.0f / rc;

  extern __shared__ __align__(16) unsigned char ss_smem[];
  const SsLayout SL = ss_layout(max(F1, F2), rc, NB);
  double* Wb = reinterpret_cast<double*>(ss_smem + SL.wb);        // [2][3][PB][LDW]
  double* Vring = reinterpret_cast<double*>(ss_smem + SL.vring);  // [R][PB*rc + 1]
  double* Uring = reinterpret_cast<double*>(ss_smem + SL.uring);  // [R][3][PB]
  double* Cs = reinterpret_cast<double*>(ss_smem + SL.cs);        // [16][kSsLdC]
  double* Cacc = reinterpret_cast<double*>(ss_smem + SL.cacc);    // [F1][LDC] footprint accumulator
  int* Pring = reinterpret_cast<int*>(ss_smem + SL.pring);        // [R][PB]
  int* S1b = reinterpret_cast<int*>(ss_smem + SL.s1b);            // [2][PB] strip (axis-1 offset) per point

  int org[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) org[a] = g.box_lo[a] + it.bin[a] * g.B;
  for (int idx = tid; idx < 2 * 3 * PB * LDW; idx += NT) Wb[idx] = 0.0;
  for (int s = tid; s < kSsRing; s += NT) Vring[s * VS + PB * VLD] = 0.0;
  for (int idx = tid; idx < 16 * kSsLdC; idx += NT) {
    const int k = idx / kSsLdC, q = idx - k * kSsLdC;
    Cs[idx] = (k < kPolyLen && q < TAPS) ? pp.c[q * kPolyLen + k] : 0.0;
  }
  for (int idx = tid; idx < F1 * LDC; idx += NT) Cacc[idx] = 0.0;

  const long long ptbase = (long long)it.win * n + it.start;
  const double* ubase = u_sorted + (long long)it.win * 3 * n + it.start;
  auto issue_perm = [&](int b) {
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    if (tid < pb) ss_cp4(Pring + (b % kSsRing) * PB + tid, perm + ptbase + q0 + tid);
  };
  auto issue_u = [&](int b) {  // axes 1 and 2
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    for (int j = tid; j < 2 * PB; j += NT) {
      const int a = 1 + j / PB, p = j % PB;
      if (p < pb) ss_cp8(Uring + ((b % kSsRing) * 3 + a) * PB + p, ubase + (long long)a * n + q0 + p);
    }
  };
  auto issue_v = [&](int b) {  // needs Pring[b] visible
    if (b >= nbatch) return;
    const int q0 = b * PB, pb = min(PB, it.count - q0);
    double* Vs = Vring + (b % kSsRing) * VS;
    const int* pr = Pring + (b % kSsRing) * PB;
    for (int j = tid; j < PB * rc; j += NT) {
      const int p = fdiv(j, inv_rc), c = j - p * rc;
      if (p < pb) ss_cp8(Vs + p * VLD + c, V + (long long)pr[p] * ldv + r0 + c);
      else Vs[p * VLD + c] = 0.0;
    }
  };
  // weights of batch b on the tensor core (as k_spread_v5): rows (axis a in {1, 2}, point p) =
  // row tiles 4 .. 11 (two per warp); W[(a,p)][q] = sum_k x^k c[q][k]; the taps land at footprint
  // nodes s + q with zeros elsewhere; S1b gets the point's strip s (axis 1), -1 for no point
  auto wgemm = [&](int b) {
    const int pb = min(PB, it.count - b * PB);
    const double* U = Uring + (b % kSsRing) * 3 * PB;
    double* W = Wb + (b & 1) * 3 * PB * LDW;
    const int j4 = lane & 3;
    double xp[2], x4[2], c0[2][2], c1[2][2];
    int s0[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int R = (4 + warp * 2 + t) * 8 + (lane >> 2), a = R / PB, p = R - a * PB;
      const bool real = p < pb;
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
      const double* cr = Cs + (4 * kk + j4) * kSsLdC + (lane >> 2);
      const double b0 = cr[0], b1 = cr[8];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        dmma(c0[t][0], c0[t][1], xp[t], b0);
        dmma(c1[t][0], c1[t][1], xp[t], b1);
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) xp[t] *= x4[t];
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int R = (4 + warp * 2 + t) * 8 + (lane >> 2), a = R / PB, p = R - a * PB;
      const bool real = p < pb;
      double* wrow = W + (a * PB + p) * LDW;
      const int Fa = g.F[a], s = s0[t];
      if (a == 1 && j4 == 0) S1b[(b & 1) * PB + p] = real ? s : -1;
      if (real) {
        const int q0 = 2 * j4;
        if (q0 < TAPS) wrow[s + q0] = c0[t][0];
        if (q0 + 1 < TAPS) wrow[s + q0 + 1] = c0[t][1];
        if (q0 + 8 < TAPS) wrow[s + q0 + 8] = c1[t][0];
        if (q0 + 9 < TAPS) wrow[s + q0 + 9] = c1[t][1];
        if (a == 2) {  // axis 1 rows are read only at the point's own taps (rows relative to its strip)
          for (int o = j4; o < s; o += 4) wrow[o] = 0.0;
          for (int o = s + TAPS + j4; o < Fa; o += 4) wrow[o] = 0.0;
        }
      } else {
        for (int o = j4; o < Fa; o += 4) wrow[o] = 0.0;
      }
    }
  };

  // prologue: perm 0..3, u 0..2, then V 0..2 and the weights of batch 0
  __syncthreads();  // tables initialised
  for (int b = 0; b < 4; ++b) issue_perm(b);
  for (int b = 0; b < 3; ++b) issue_u(b);
  ss_commit();
  ss_wait_all();
  __syncthreads();
  for (int b = 0; b < 3; ++b) issue_v(b);
  ss_commit();
  wgemm(0);
  ss_wait_all();
  __syncthreads();

  // fragment coordinates: A rows are the strip's taps i (rows >= TAPS read nothing); B columns
  // (o2, c) = (w2 row | rhs << 16), invalid columns at the zero weight slot
  unsigned bi[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int col = (warp * NB + j) * 8 + (lane >> 2);
    bi[j] = col < Nn ? (unsigned)(col / rc) | ((unsigned)(col - (col / rc) * rc) << 16) : (unsigned)(LDW - 1);
  }
  double acc[MT][NB][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // the register tiles of strip cs into the shared footprint (rows cs + i), then zero
  auto spill = [&](int cs) {
    if (cs >= 0) {
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int row = i * 8 + (lane >> 2);
        if (row >= TAPS) continue;
        double* crow = Cacc + (cs + row) * LDC + warp * NB * 8 + 2 * (lane & 3);
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          double2* c2 = reinterpret_cast<double2*>(crow + j * 8);
          double2 v = *c2;
          v.x += acc[i][j][0];
          v.y += acc[i][j][1];
          *c2 = v;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  };

  int cs = -1;  // current strip (-1: none yet)
  for (int b = 0; b < nbatch; ++b) {
    const double* W1 = Wb + (b & 1) * 3 * PB * LDW + PB * LDW;
    const double* W2 = W1 + PB * LDW;
    const double* Vs = Vring + (b % kSsRing) * VS;
    const int* S1 = S1b + (b & 1) * PB;
    const int ksteps = (min(PB, it.count - b * PB) + 3) >> 2;
    // the batch's k-steps in runs inside the current strip (straight-line DMMA streams, two k-steps
    // in flight) and single k-steps at strip changes
    const int my_s = S1[lane];  // PB == 32: lane = point of the batch
    auto fast = [&](int ks) {  // every point of k-step ks in strip cs (or padding: zero weights)
      const int p = ks * 4 + (lane & 3);
      const double* w1 = W1 + p * LDW + cs;
      const double* w2 = W2 + p * LDW;
      const double* vs = Vs + p * VLD;
      double bf[NB], af[MT];
#pragma unroll
      for (int j = 0; j < NB; ++j) bf[j] = w2[bi[j] & 0xffff] * vs[bi[j] >> 16];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int row = i * 8 + (lane >> 2);
        af[i] = (TAPS % 8 == 0 || row < TAPS) ? w1[row] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    };
    auto slow = [&](int ks) {  // a strip change inside k-step ks: once per strip, the others masked
      const int p = ks * 4 + (lane & 3);
      const double* w1 = W1 + p * LDW;
      const double* w2 = W2 + p * LDW;
      const double* vs = Vs + p * VLD;
      const int sq = S1[p];
      double bf[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) bf[j] = w2[bi[j] & 0xffff] * vs[bi[j] >> 16];
      bool pending = sq >= 0;
#pragma unroll
      for (int rep = 0; rep < 5; ++rep) {
        const bool mine = pending && sq == cs;
        if (__any_sync(0xffffffffu, mine)) {
          double af[MT];
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const int row = i * 8 + (lane >> 2);
            af[i] = (mine && row < TAPS) ? w1[sq + row] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NB; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
          pending = pending && !mine;
        }
        if (rep < 4 && __any_sync(0xffffffffu, pending)) {
          int nxt = pending ? sq : INT_MAX;  // the next strip: the smallest pending one
          nxt = min(nxt, __shfl_xor_sync(0xffffffffu, nxt, 1));
          nxt = min(nxt, __shfl_xor_sync(0xffffffffu, nxt, 2));
          spill(cs);
          cs = nxt;
        }
      }
    };
    for (int ks = 0; ks < ksteps;) {
      const unsigned bad = ~__ballot_sync(0xffffffffu, my_s == cs || my_s < 0) & (0xffffffffu << (4 * ks));
      const int ke = bad ? min(ksteps, (__ffs(bad) - 1) >> 2) : ksteps;
#pragma unroll 2
      for (int k = ks; k < ke; ++k) fast(k);
      if (ke >= ksteps) break;
      slow(ke);
      ks = ke + 1;
    }
    if (b + 1 < nbatch) wgemm(b + 1);
    ss_wait_all();
    __syncthreads();
    issue_perm(b + 4);
    issue_u(b + 3);
    issue_v(b + 3);
    ss_commit();
  }
  spill(cs);
  __syncthreads();

  // flush the footprint: F1 x Nn values (row o1, column (o2, c))
  const long long L2 = g.L[2], toff = g.tap_off;
  const int c1 = org[1] - g.box_lo[1], c2 = org[2] - g.box_lo[2];
  double* gbase = grid + r0;
  for (int idx = tid; idx < F1 * Nn; idx += NT) {
    const int row = idx / Nn, col = idx - row * Nn;
    const double v = Cacc[row * LDC + col];
    if (v == 0.0) continue;
    const int o2 = fdiv(col, inv_rc), c = col - o2 * rc;
    const long long node = toff + (long long)(c1 + row) * L2 + c2 + o2;
    if constexpr (DET) det_add(da, it.win, node * r_total + r0 + c, r0 + c, v);
    else atomicAdd(gbase + node * r_total + c, v);
  }
}

#define AKM_SS_INSTANCES(X) X(16, 7) X(16, 8) X(16, 6) X(16, 5) X(16, 4) X(16, 3) X(16, 2) X(16, 1) \
  X(8, 6) X(8, 5) X(8, 4) X(8, 3) X(8, 2) X(8, 1) X(12, 7) X(12, 6) X(12, 5) X(12, 4) X(12, 3) X(12, 2) X(12, 1)

namespace {
constexpr size_t kSsSmemMax = 113 * 1024;  // two CTAs per SM
bool ss_has(int taps, int nb) {
#define AKM_SS_HAS(T, N) \
  if (taps == T && nb == N) return true;
  AKM_SS_INSTANCES(AKM_SS_HAS)
#undef AKM_SS_HAS
  return false;
}
}  // namespace

// n-tiles per warp for a footprint of F nodes per axis and rc RHS columns; 0 = unsupported
int spread_strip_nb(int d, int taps, int F, int rc) {
  static const int mode = getenv("AKM_SPREAD_STRIP") ? atoi(getenv("AKM_SPREAD_STRIP")) : -1;
  if (mode == 0 || d != 2 || F < taps || F - taps + 1 > 8) return 0;
  const int nb = ((F * rc + 7) / 8 + kSsWarps - 1) / kSsWarps;
  if (!ss_has(taps, nb)) return 0;
  if (ss_layout(F, rc, nb).total > kSsSmemMax) return 0;
  return nb;
}

size_t spread_strip_smem(int F, int rc, int nb) { return ss_layout(F, rc, nb).total; }

cudaError_t launch_spread_strip(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                                const double* u_sorted, const int* perm, const double* V, long long ldv, long long n,
                                int r0, int rc, int r_total, double* grid, int taps, int F, int nb, cudaStream_t s,
                                const DetAcc& da) {
  if (n_items <= 0) return cudaSuccess;
  const size_t smem = spread_strip_smem(F, rc, nb);
#define AKM_SS_CASE1(T, N, det)                                                                                 \
  if (taps == T && nb == N && (da.limbs != nullptr) == det) {                                                    \
    static std::atomic<unsigned long long> attr_set{0};                                                         \
    if (!optin_done(attr_set)) {                                                                                \
      cudaError_t e = cudaFuncSetAttribute(k_spread_strip<T, N, det>,                                          \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSsSmemMax);       \
      if (e != cudaSuccess) return e;                                                                           \
      optin_mark(attr_set);                                                                                     \
    }                                                                                                           \
    k_spread_strip<T, N, det><<<n_items, kSsThreads, smem, s>>>(dtab, items, u_sorted, perm, V, ldv, n, r0, rc, \
                                                                r_total, grid, pp, da);                         \
    return cudaGetLastError();                                                                                  \
  }
#define AKM_SS_CASE(T, N) AKM_SS_CASE1(T, N, false) AKM_SS_CASE1(T, N, true)
  AKM_SS_INSTANCES(AKM_SS_CASE)
#undef AKM_SS_CASE
#undef AKM_SS_CASE1
  return cudaErrorInvalidValue;
}

}  // namespace akm
