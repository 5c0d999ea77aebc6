// interp_pt.cu -- NFFT interpolation (App. A; the outer sums of eq. 3.3) for SMALL
// launches: one warp per point, the lanes splitting the point's (o1, o2) taps, H read straight from
// L2 (no staging), a warp reduction per value.
//
// The staged kernels (k_interp_bin / k_interp_t / k_interp_strip) stream a bin footprint through
// shared memory plane by plane; with few work items (c1: n = 2000, ~60 bins) a launch is one CTA's
// serial chain of F staged planes (25 us at c1).  Here every point is independent: the chain is one
// pass over the 2m o0-planes with ~(2m)^2/32 taps per lane, and all points run at once.  The L1/L2
// traffic is (2m)^d values per point and value, which only small launches can afford (the staged
// kernels exist because large ones cannot): plan.cu uses it below 2 x 148 per-bin items.
#include <cstdlib>

#include "akm_internal.cuh"

namespace akm {

namespace {
constexpr int kPtWarps = 8;   // warps per CTA
constexpr int kPtSplit = 4;   // CTAs per item: an item of <= 128 points takes <= 4 rounds per warp (16 measured no faster)
constexpr int kPtMaxV = 32;   // values per node handled (OPS * RC): one per lane
}  // namespace

template <int D, int TAPS>
__global__ void __launch_bounds__(32 * kPtWarps, 1) k_interp_pt(const WinTable* __restrict__ tabp,
                                                             const WorkItem* __restrict__ items,
                                                             const double* __restrict__ u_sorted,
                                                             const int* __restrict__ perm,
                                                             const double* __restrict__ H, int ops, int r, int r0,
                                                             int rc, double* __restrict__ part, long long n,
                                                             const __grid_constant__ PolyParam pp) {
  constexpr int T0 = (D >= 3) ? TAPS : 1;
  constexpr int T1 = (D >= 2) ? TAPS : 1;
  constexpr int NT = T1 * TAPS;                 // (o1, o2) taps per plane
  constexpr int TPL = (NT + 31) / 32;           // taps per lane
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double poly[TAPS * kPolyLen];  // runtime tap indices: from shared memory, not the parameter
  for (int idx = threadIdx.x; idx < TAPS * kPolyLen; idx += blockDim.x) poly[idx] = pp.c[idx];
  __syncthreads();
  const int V = ops * rc;
  const long long row_vals = (long long)ops * r;
  for (int q = blockIdx.y * kPtWarps + warp; q < it.count; q += kPtWarps * kPtSplit) {
    const long long pidx = (long long)it.start + q;
    int base[3] = {0, 0, 0};
    double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 3 - D; a < 3; ++a) {
      const double u = u_sorted[((long long)it.win * 3 + a) * n + pidx];
      const double fl = floor(u);
      x[a] = 2.0 * (u - fl) - 1.0;
      base[a] = (int)fl - tab.m + 1 - g.box_lo[a];  // box-local node of tap 0
    }
    // this lane's taps (o1, o2) and their weights w1 w2; the o0 weight per plane below
    long long toff[TPL];
    double w12[TPL];
#pragma unroll
    for (int j = 0; j < TPL; ++j) {
      const int t = lane + 32 * j;
      const bool ok = t < NT;
      const int o1 = ok ? t / TAPS : 0, o2 = ok ? t - (t / TAPS) * TAPS : 0;
      const double w1 = (D >= 2) ? window_tap(poly, o1, x[1]) : 1.0;
      w12[j] = ok ? w1 * window_tap(poly, o2, x[2]) : 0.0;
      toff[j] = ((long long)(base[1] + (D >= 2 ? o1 : 0)) * g.L[2] + base[2] + o2) * row_vals;
    }
    // lane o holds the o0 weight of tap o (handed out by shuffles); one value of the node at a time,
    // rolled loops: the kernel stays small (an unrolled value loop overflowed the instruction cache)
    const double w0l = (D >= 3 && lane < T0) ? window_tap(poly, lane, x[0]) : 1.0;
    double mine = 0.0;  // lane v keeps value v
    for (int v = 0; v < V; ++v) {
      const long long voff = (long long)(v / rc) * r + (v % rc);
      double acc = 0.0;
#pragma unroll 2
      for (int o0 = 0; o0 < T0; ++o0) {
        const double w0 = (D >= 3) ? __shfl_sync(0xffffffffu, w0l, o0) : 1.0;
        const double* hp = H + (g.tap_off + (long long)(base[0] + o0) * g.L[1] * g.L[2]) * row_vals + r0 + voff;
#pragma unroll
        for (int j = 0; j < TPL; ++j)
          if (lane + 32 * j < NT) acc = fma(w0 * w12[j], __ldg(hp + toff[j]), acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == (v & 31)) mine = acc;
    }
    const long long i = perm[(long long)it.win * n + pidx];
    double* out = part + (((long long)it.win * n + i) * ops) * r + r0;
    if (lane < V) out[(long long)(lane / rc) * r + (lane % rc)] = mine;
  }
}

// per-bin items below which a launch is latency-bound (fewer than two CTAs per SM)
bool interp_pt_choose(int d, int taps, int ops, int rc, int n_items_bin) {
  static const int mode = getenv("AKM_INTERP_PT") ? atoi(getenv("AKM_INTERP_PT")) : -1;
  if (mode == 0 || ops * rc > kPtMaxV || n_items_bin <= 0 || d < 1 || d > 3) return false;
  if (taps != 8 && taps != 12 && taps != 16) return false;
  return mode == 1 || n_items_bin < 2 * 148;
}

cudaError_t launch_interp_pt(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                             const double* u_sorted, const int* perm, const double* H, int d, int taps, int ops,
                             int r, int r0, int rc, double* part, long long n, cudaStream_t s) {
  if (n_items <= 0) return cudaSuccess;
#define AKM_PT_CASE(D, T)                                                                                  \
  if (d == D && taps == T) {                                                                               \
    k_interp_pt<D, T><<<dim3(n_items, kPtSplit), 32 * kPtWarps, 0, s>>>(dtab, items, u_sorted, perm, H, ops, r, r0, rc,    \
                                                        part, n, pp);                                      \
    return cudaGetLastError();                                                                             \
  }
  AKM_PT_CASE(1, 8) AKM_PT_CASE(1, 12) AKM_PT_CASE(1, 16)
  AKM_PT_CASE(2, 8) AKM_PT_CASE(2, 12) AKM_PT_CASE(2, 16)
  AKM_PT_CASE(3, 8) AKM_PT_CASE(3, 12) AKM_PT_CASE(3, 16)
#undef AKM_PT_CASE
  return cudaErrorInvalidValue;
}

}  // namespace akm
