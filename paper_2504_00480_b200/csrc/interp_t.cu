// interp_t.cu -- NFFT interpolation (App. A; the outer sums of eq. 3.3) for 3-D windows
// with many values per node, as a GEMM over the first two tap axes:
//
//   T[p][(o2, v)] = sum_{(o0, o1)} (w0 w1)[p][(o0, o1)] H[(o0, o1)][(o2, v)]     (DMMA)
//   out[p][v]     = sum_{o2} w2[p][o2] T[p][(o2, v)]                            (epilogue)
//
// for the points p of one bin (all sharing one FP^3 footprint).  Compared with the per-plane
// GEMM of interp_impl.cuh (N = V values, K = taps) the N dimension is TAPS * V, so V = 11 pads to
// 136 instead of 16 columns (97% instead of 69% useful MMA work), each A value (one DMUL) feeds
// NTW DMMAs instead of NT, and a footprint row (o0, o1) is one contiguous run of H.
#include <algorithm>

#include "akm_internal.cuh"

namespace akm {

namespace {
__device__ __forceinline__ void it_cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void it_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void it_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int kItWarps = 4;  // two CTAs per SM: one's barriers and epilogue hide under the other's MMAs
constexpr int kItPS = 1;              // o0-planes per pipeline step (one CTA barrier per step)
constexpr int kItRing = 3 * kItPS;    // ring slots: steps s (computing), s+1, s+2 (in flight)

template <int FP, int V, int MT, int WN>
struct ItShape {
  static constexpr int KQF = (FP + 3) / 4;            // k-steps per footprint plane
  static constexpr int KR = 4 * KQF;                  // staged rows per plane (zero-padded)
  static constexpr int N = FP * V;                    // GEMM columns (o2, v)
  static constexpr int NTT = (N + 7) / 8;             // column tiles
  static constexpr int NTW = (NTT + WN - 1) / WN;     // column tiles per warp
  static constexpr int LDB = mma_ld(WN * NTW * 8);    // staged row stride (= 4 mod 16)
  static constexpr int PPC = (kItWarps / WN) * MT * 8;  // points per pass
  static constexpr int LDT = WN * NTW * 8 + 2;        // epilogue row stride
  static constexpr size_t ring_bytes = (size_t)kItRing * KR * LDB * sizeof(double);
  static constexpr size_t t_bytes = (size_t)PPC * LDT * sizeof(double);
  static constexpr size_t w_bytes = 3 * (size_t)PPC * KR * sizeof(double);  // w0s, w1s, w2s
  static constexpr size_t smem = (ring_bytes > t_bytes ? ring_bytes : t_bytes) + w_bytes;
};
}  // namespace

// One CTA per work item = up to 128 points of ONE BIN (B^3 cells; the footprint is FP = B + 2m - 1
// nodes per axis).  A point's weights are zero outside its own 2m taps, so all points of the bin
// share the staged footprint planes and the GEMM shape; for B = 1 (c4, c5: a bin is a cell) no
// work is padded.
template <int TAPS, int FP, int OPS, int RC, int MT, int WN>
__global__ void __launch_bounds__(32 * kItWarps, (OPS * RC <= 2) ? 4 : 2) k_interp_t(const WinTable* __restrict__ tabp,
                                                               const WorkItem* __restrict__ items,
                                                               const double* __restrict__ u_sorted,
                                                               const int* __restrict__ perm,
                                                               const double* __restrict__ H, int r, int r0,
                                                               double* __restrict__ part, long long n,
                                                               const __grid_constant__ PolyParam pp, int bscale) {
  constexpr int V = OPS * RC;
  using S = ItShape<FP, V, MT, WN>;
  constexpr int N = S::N, NTW = S::NTW, LDB = S::LDB, PPC = S::PPC, LDT = S::LDT, KQF = S::KQF, KR = S::KR;
  constexpr int KQ = TAPS / 4;
  constexpr int NT = 32 * kItWarps;
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN, j4 = lane & 3;

  extern __shared__ double sm[];
  double* ring = sm;  // [kItRing][KR][LDB]; later T [PPC][LDT]
  double* w0s = sm + (S::ring_bytes > S::t_bytes ? S::ring_bytes : S::t_bytes) / sizeof(double);  // [PPC][KR]
  double* w1s = w0s + PPC * KR;
  double* w2s = w1s + PPC * KR;

  const long long row_vals = (long long)OPS * r;
  const bool contiguous = (RC == r && r0 == 0);
  const long long L1g = g.L[1], L2g = g.L[2], toff = g.tap_off;
  // box-local footprint origin: bin items (bscale = B) or per-cell items (bscale = 1, FP = TAPS)
  const int ob0 = it.bin[0] * bscale, ob1 = it.bin[1] * bscale, ob2 = it.bin[2] * bscale;
  // staging of footprint plane o0 into ring slot slot_of(o0): footprint row o1 by warp
  // o1 % kItWarps, consecutive lanes on consecutive columns (contiguous H: a row (o0, o1) is one
  // run of N doubles of H; otherwise a gather per element)
  int plane_ctr = 0;  // planes staged in earlier passes
  auto slot_of = [&](int o0) { return (plane_ctr + o0) % kItRing; };
  // contiguous H: the warp's rows (o1 = warp + kItWarps * i) start at fixed offsets from the
  // footprint origin; a plane step adds L1 * L2 nodes.  Unrolled, each copy is one cp.async with
  // an immediate offset.
  constexpr int RPW = (FP + kItWarps - 1) / kItWarps, CPL = (N + 31) / 32;
  const double* src0 = H + (toff + ((long long)ob0 * L1g + ob1 + warp) * L2g + ob2) * row_vals + lane;
  const long long plane_stride = L1g * L2g * row_vals, row_stride = kItWarps * L2g * row_vals;
  auto stage = [&](int o0) {
    double* buf = ring + slot_of(o0) * KR * LDB;
    if (contiguous) {
      const double* src = src0 + o0 * plane_stride;
      double* dst = buf + warp * LDB + lane;
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        if (FP % kItWarps == 0 || warp + i * kItWarps < FP) {
#pragma unroll
          for (int j = 0; j < CPL; ++j)
            if (j * 32 + 32 <= N || j * 32 + lane < N) it_cp8(dst + j * 32, src + j * 32);
        }
        src += row_stride;
        dst += kItWarps * LDB;
      }
      return;
    }
    const long long tap_row = toff + ((long long)(ob0 + o0) * L1g + ob1) * L2g + ob2;
    for (int o1 = warp; o1 < FP; o1 += kItWarps) {
      const long long trow = tap_row + o1 * L2g;
      double* dst = buf + o1 * LDB;
      for (int col = lane; col < N; col += 32) {
        const int o2 = col / V, v = col - o2 * V, op = v / RC, c = v - op * RC;
        it_cp8(dst + col, H + (trow + o2) * row_vals + op * r + r0 + c);
      }
    }
  };
  auto stage_step = [&](int st) {  // planes st*kItPS .. +kItPS-1 as one cp.async group
#pragma unroll
    for (int k = 0; k < kItPS; ++k)
      if (st * kItPS + k < FP) stage(st * kItPS + k);
    it_commit();
  };

  // padding rows and columns of the ring (never staged): zeros, not uninitialised (NaN) bits
  for (int idx = tid; idx < kItRing * KR * LDB; idx += NT) {
    const int row = idx / LDB, c = idx - row * LDB;
    if (row % KR >= FP || c >= N) ring[idx] = 0.0;
  }

  for (int pbase = 0; pbase < it.count; pbase += PPC) {
    const int cnt = min(PPC, it.count - pbase);
    // stage the first two steps while the weights are evaluated
    stage_step(0);
    stage_step(1);

    // weights: per point and axis a row of KR footprint nodes, the 2m taps at the point's offset
    // s inside the bin and zeros elsewhere.  The quad of lanes sharing a point row takes taps
    // {j4, j4+4, ...} (and the zero-fill of nodes {j4, j4+4, ...}).
    double w1r[MT][KQF];
    if constexpr (FP == TAPS) {
      // B = 1: every point's taps start at footprint node 0; w1 straight into registers
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int q = (wm * MT + mt) * 8 + (lane >> 2);
        const bool has = q < cnt;
        const long long pidx = (long long)it.start + pbase + (has ? q : 0);
        double x[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double u = u_sorted[((long long)it.win * 3 + a) * n + pidx];
          x[a] = 2.0 * (u - floor(u)) - 1.0;
        }
        double wt[KQ];
        window_taps_estrin_strided<KQ>(pp.c, j4, 4, x[1], wt);
#pragma unroll
        for (int k = 0; k < KQ; ++k) w1r[mt][k] = has ? wt[k] : 0.0;
        if (wn == 0) {
          window_taps_estrin_strided<KQ>(pp.c, j4, 4, x[0], wt);
#pragma unroll
          for (int k = 0; k < KQ; ++k) w0s[q * KR + j4 + 4 * k] = has ? wt[k] : 0.0;
          window_taps_estrin_strided<KQ>(pp.c, j4, 4, x[2], wt);
#pragma unroll
          for (int k = 0; k < KQ; ++k) w2s[q * KR + j4 + 4 * k] = wt[k];
        }
      }
    } else {
      if (wn == 0) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int q = (wm * MT + mt) * 8 + (lane >> 2);
          const bool has = q < cnt;
          const long long pidx = (long long)it.start + pbase + (has ? q : 0);
          double* wrow[3] = {w0s + q * KR, w1s + q * KR, w2s + q * KR};
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < KQF; ++k) wrow[a][j4 + 4 * k] = 0.0;
          __syncwarp();
          if (has) {
            const int ob[3] = {ob0, ob1, ob2};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const double u = u_sorted[((long long)it.win * 3 + a) * n + pidx];
              const double fl = floor(u);
              const int s = (int)fl - tab.m + 1 - (g.box_lo[a] + ob[a]);
              double wt[KQ];
              window_taps_estrin_strided<KQ>(pp.c, j4, 4, 2.0 * (u - fl) - 1.0, wt);
#pragma unroll
              for (int k = 0; k < KQ; ++k) wrow[a][s + j4 + 4 * k] = wt[k];
            }
          }
        }
      }
      if constexpr (WN == 1) __syncwarp();  // a warp reads only its own points' tables
      else __syncthreads();
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int k = 0; k < KQF; ++k) w1r[mt][k] = w1s[((wm * MT + mt) * 8 + (lane >> 2)) * KR + 4 * k + j4];
    }
    const bool wact = wm * MT * 8 < cnt;

    double acc[MT][NTW][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

    const int boff = j4 * LDB + wn * NTW * 8 + (lane >> 2);
    constexpr int NSTEP = (FP + kItPS - 1) / kItPS;
    for (int st = 0; st < NSTEP; ++st) {
      if (st + 1 < NSTEP) it_wait<1>();
      else it_wait<0>();
      __syncthreads();  // step st visible to all; step st-1's slots free
      stage_step(st + 2);
      if (!wact) continue;
#pragma unroll 1
      for (int o0 = st * kItPS; o0 < min(FP, st * kItPS + kItPS); ++o0) {
        const double* bp = ring + slot_of(o0) * KR * LDB + boff;
        double w0c[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) w0c[mt] = w0s[((wm * MT + mt) * 8 + (lane >> 2)) * KR + o0];
#pragma unroll
        for (int k = 0; k < KQF; ++k) {
          double af[MT];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) af[mt] = w0c[mt] * w1r[mt][k];
          const double* bk = bp + 4 * k * LDB;
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) {
            const double b = bk[nt * 8];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], b);
          }
        }
      }
    }
    it_wait<0>();
    plane_ctr += FP;
    __syncthreads();  // all planes consumed: the ring becomes T

    // T -> shared, then out[p][v] = sum_o2 w2[p][o2] T[p][o2 * V + v]
    double* T = ring;
    if (wact) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int q = (wm * MT + mt) * 8 + (lane >> 2);
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) {
          const int col = (wn * NTW + nt) * 8 + 2 * j4;
          *reinterpret_cast<double2*>(T + q * LDT + col) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        }
      }
    }
    __syncthreads();
    for (int job = tid; job < cnt * V; job += NT) {
      const int q = job / V, v = job - q * V;
      const double* tr = T + q * LDT + v;
      const double* w2 = w2s + q * KR;
      double s = 0.0;
#pragma unroll
      for (int o2 = 0; o2 < FP; ++o2) s = fma(w2[o2], tr[o2 * V], s);
      const long long i = perm[(long long)it.win * n + it.start + pbase + q];
      const int op = v / RC, c = v - op * RC;
      part[(((long long)it.win * n + i) * OPS + op) * r + r0 + c] = s;
    }
    __syncthreads();  // T / weights reused by the next pass.  (T overwrote the ring's padding with
                      // finite values: padded rows meet zero weights, padded columns are never read.)
  }
}

// instances: (TAPS, FP, OPS, RC) -> (MT, WN)
#define AKM_IT_INSTANCES(X) X(12, 12, 1, 11, 2, 1) X(12, 12, 2, 1, 2, 1) X(12, 12, 1, 2, 2, 1)

bool interp_t_supported(int d, int taps, int fp, int ops, int rc) {
#define AKM_IT_SUP(T, F, O, R, M, W) \
  if (d == 3 && taps == T && fp == F && ops == O && rc == R) return true;
  AKM_IT_INSTANCES(AKM_IT_SUP)
#undef AKM_IT_SUP
  return false;
}

cudaError_t launch_interp_t(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                            const double* u_sorted, const int* perm, const double* H, int taps, int fp, int ops, int r,
                            int r0, int rc, double* part, long long n, cudaStream_t s, int bscale) {
  if (n_items <= 0) return cudaSuccess;
#define AKM_IT_CASE(T, F, O, R, M, W)                                                                          \
  if (taps == T && fp == F && ops == O && rc == R) {                                                           \
    constexpr size_t smem = ItShape<F, O * R, M, W>::smem;                                                     \
    static std::atomic<unsigned long long> attr_set{0};                                                                              \
    if (!optin_done(attr_set)) {                                                                                           \
      cudaError_t e = cudaFuncSetAttribute(k_interp_t<T, F, O, R, M, W>,                                       \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
      if (e != cudaSuccess) return e;                                                                          \
      optin_mark(attr_set);                                                                                         \
    }                                                                                                          \
    k_interp_t<T, F, O, R, M, W><<<n_items, 32 * kItWarps, smem, s>>>(dtab, items, u_sorted, perm, H, r, r0,   \
                                                                      part, n, pp, bscale);                    \
    return cudaGetLastError();                                                                                 \
  }
  AKM_IT_INSTANCES(AKM_IT_CASE)
#undef AKM_IT_CASE
  return cudaErrorInvalidValue;
}

}  // namespace akm
