// interp_strip.cu -- NFFT interpolation (App. A; the outer sums of eq. 3.3) for 2-D
// windows on the FP64 tensor cores, one GEMM per strip of cells:
//
//   T[p][(v, i)] = sum_k W2[p][k] H[(s1 + i, k)][v]          (DMMA; K = footprint nodes on axis 2)
//   out[p][v]    = sum_i w1[p][i] T[p][(v, i)]              (accumulator epilogue, no shared memory)
//
// Work item = up to 128 points of one bin (B x B cells, footprint F = B + 2m - 1 nodes per axis;
// the per-bin items of k_interp_bin).  Inside a bin the points are sorted by cell, axis 1 major
// (binsort.cu slot_key), so the points of one cell row s1 are contiguous: a STRIP of 1 x B cells
// whose axis-1 taps are exactly the 2m footprint rows s1 .. s1 + 2m - 1.  Along axis 1 nothing is
// padded (N = V x 2m columns); along axis 2 the point's 2m taps sit at its offset s2 in the
// F-node K range (zeros elsewhere), so a strip pads K by F / 2m (B = 4, m = 8: 19 -> 20 rows for 16
// taps) -- against (F / 2m)^2 for the whole-bin footprint GEMM and the scalar per-bin kernel's
// shared-memory-wavefront bound (c3).
//
// Fragment layouts (akm_internal.cuh dmma): A = W2[p = lane>>2][k = lane&3] from the per-point tap
// table; B = Hs[k = lane&3][(v, i = lane>>2)] from the staged footprint [k][v][i]; C rows are points,
// columns (v, i = 2 (lane&3) + {0,1}) -- so the epilogue is 2 FMAs per accumulator pair with the
// point's own w1 taps and a reduction over the 4 lanes of a quad.
#include <algorithm>
#include <cstdlib>

#include "akm_internal.cuh"

namespace akm {

namespace {
__device__ __forceinline__ void is_cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

constexpr int kIsThreads = 128;  // one point per thread in the prologue; 4 warps share the m-tiles
// (the per-bin items hold <= 128 points: plan.cu ch_ib, as for k_interp_bin's one point per thread)

struct IsLayout {
  int KP;   // staged K rows (axis-2 footprint nodes, rounded up to a multiple of 4; padding rows zero)
  int LDV;  // per-value stride of a staged row (axis-1 footprint nodes)
  int LDK;  // staged row stride (= 4 mod 16 doubles: conflict-free B fragments)
};
__host__ __device__ inline IsLayout is_layout(int F, int V) {
  IsLayout l;
  l.KP = (F + 3) & ~3;
  l.LDV = F;
  l.LDK = mma_ld(V * F);
  return l;
}
template <int TAPS>
__host__ __device__ constexpr int is_ldw() { return TAPS + 1; }
}  // namespace

template <int TAPS, int OPS, int RC>
__global__ void __launch_bounds__(kIsThreads, (OPS * RC * TAPS / 8 > 24) ? 2 : 3) k_interp_strip(const WinTable* __restrict__ tabp,
                                                                const WorkItem* __restrict__ items,
                                                                const double* __restrict__ u_sorted,
                                                                const int* __restrict__ perm,
                                                                const double* __restrict__ H, int r, int r0,
                                                                double* __restrict__ part, long long n, int F,
                                                                const __grid_constant__ PolyParam pp) {
  constexpr int V = OPS * RC;
  constexpr int NI = TAPS / 8;  // column tiles per value (axis-1 taps)
  constexpr int NT = V * NI;
  constexpr int LDW = is_ldw<TAPS>();
  const WinTable& tab = *tabp;
  const WorkItem it = items[blockIdx.x];
  const WinGeom& g = tab.w[it.win];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = F - TAPS + 1;
  const IsLayout L = is_layout(F, V);

  extern __shared__ __align__(16) double sm[];
  double* Hs = sm;                       // [KP][LDK]: Hs[k][v * LDV + i] = H[(o1 = i, o2 = k)][v]
  double* w1s = Hs + L.KP * L.LDK;       // [128][LDW] axis-1 taps per point
  double* w2s = w1s + kIsThreads * LDW;  // [128][LDW] axis-2 taps per point
  int* s2s = reinterpret_cast<int*>(w2s + kIsThreads * LDW);  // [128] axis-2 offset in the bin

  // ---- stage the bin footprint (rows o1 by warp, a row (o2, v) run of H by consecutive lanes)
  const long long row_vals = (long long)OPS * r;
  const int org1 = it.bin[1] * B, org2 = it.bin[2] * B;  // box-local footprint origin
  const long long L2g = g.L[2];
  const double* hrow0 = H + (g.tap_off + (long long)org1 * L2g + org2) * row_vals;
  const bool contiguous = (RC == r && r0 == 0);
  for (int i = warp; i < F; i += kIsThreads / 32) {
    const double* src = hrow0 + (long long)i * L2g * row_vals;
    double* dst = Hs + i;
    for (int j = lane; j < F * V; j += 32) {
      const int k = j / V, v = j - k * V;
      if (contiguous) {
        is_cp8(dst + k * L.LDK + v * L.LDV, src + j);
      } else {
        const int op = v / RC, c = v - op * RC;
        is_cp8(dst + k * L.LDK + v * L.LDV, src + (long long)k * row_vals + op * r + r0 + c);
      }
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  // K padding rows: zeros (their A values are zero, but 0 * NaN would not be)
  for (int idx = tid; idx < (L.KP - F) * L.LDK; idx += kIsThreads) Hs[F * L.LDK + idx] = 0.0;

  // ---- per point: cell offsets in the bin and the 2m taps per axis
  const bool has = tid < it.count;
  const long long pidx = (long long)it.start + (has ? tid : 0);
  int s1 = B;  // sentinel: no row
  {
    const double u1 = u_sorted[((long long)it.win * 3 + 1) * n + pidx];
    const double u2 = u_sorted[((long long)it.win * 3 + 2) * n + pidx];
    const double f1 = floor(u1), f2 = floor(u2);
    double w[TAPS];
    window_taps_estrin<TAPS>(pp.c, 2.0 * (u1 - f1) - 1.0, w);
#pragma unroll
    for (int o = 0; o < TAPS; ++o) w1s[tid * LDW + o] = w[o];
    window_taps_estrin<TAPS>(pp.c, 2.0 * (u2 - f2) - 1.0, w);
#pragma unroll
    for (int o = 0; o < TAPS; ++o) w2s[tid * LDW + o] = w[o];
    if (has) {
      s1 = (int)f1 - tab.m + 1 - (g.box_lo[1] + org1);
      s2s[tid] = (int)f2 - tab.m + 1 - (g.box_lo[2] + org2);
    } else {
      s2s[tid] = 0;
    }
  }
  // rows of the bin: points sorted by s1, so row b is the contiguous range [start_b, start_b + cnt_b)
  int cnt[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) cnt[b] = (b < B) ? __syncthreads_count(s1 == b) : 0;
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  // ---- m-tiles (8 points of one row), round-robin over the warps
  int ntiles = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) ntiles += (cnt[b] + 7) >> 3;
  const int q = lane & 3, pr = lane >> 2;
  for (int t = warp; t < ntiles; t += kIsThreads / 32) {
    int b = 0, tt = t, rs = 0;
#pragma unroll
    for (int bb = 0; bb < 8; ++bb) {  // row of tile t and its first point
      const int nt = (cnt[bb] + 7) >> 3;
      if (b == bb && tt >= nt) {
        tt -= nt;
        rs += cnt[bb];
        b = bb + 1;
      }
    }
    const int p = rs + 8 * tt + pr;
    const bool valid = p < rs + cnt[b];
    const int pp_ = valid ? p : rs;
    const int s2p = s2s[pp_];
    const double* wrow = w2s + pp_ * LDW;

    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
    const double* bbase = Hs + q * L.LDK + b + pr;
    for (int k0 = 0; k0 < L.KP; k0 += 4) {
      const int o = k0 + q - s2p;
      const double a = (valid && o >= 0 && o < TAPS) ? wrow[o] : 0.0;
      const double* bp = bbase + k0 * L.LDK;
#pragma unroll
      for (int v = 0; v < V; ++v) {
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[v * NI + ni][0], acc[v * NI + ni][1], a, bp[ni * 8]);
        bp += L.LDV;
      }
    }
    // epilogue: out[p][v] = sum_i w1[p][i] T[p][(v, i)]; this lane holds i = 8 ni + 2 q + {0, 1}
    double w1r[NI][2];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      w1r[ni][0] = w1s[pp_ * LDW + ni * 8 + 2 * q];
      w1r[ni][1] = w1s[pp_ * LDW + ni * 8 + 2 * q + 1];
    }
    const long long iout = perm[(long long)it.win * n + it.start + pp_];
    double* out = part + (((long long)it.win * n + iout) * OPS) * r + r0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      double s = 0.0;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) s = fma(w1r[ni][1], acc[v * NI + ni][1], fma(w1r[ni][0], acc[v * NI + ni][0], s));
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (valid && (v & 3) == q) out[(long long)(v / RC) * r + (v % RC)] = s;
    }
  }
}

constexpr size_t kIsSmemMax = 113 * 1024;  // two CTAs per SM at least

size_t interp_strip_smem(int taps, int F, int V) {
  const IsLayout L = is_layout(F, V);
  return sizeof(double) * ((size_t)L.KP * L.LDK + 2 * (size_t)kIsThreads * (taps + 1)) + sizeof(int) * kIsThreads;
}

#define AKM_IS_INSTANCES(X) \
  X(16, 1, 11) X(16, 2, 11) X(16, 1, 4) X(16, 2, 4) X(16, 1, 2) X(16, 2, 2) X(16, 1, 1) X(16, 2, 1) \
  X(8, 1, 11) X(8, 2, 11) X(8, 1, 4) X(8, 2, 4) X(8, 1, 2) X(8, 2, 2) X(8, 1, 1) X(8, 2, 1)

// AKM_INTERP_STRIP=0 keeps k_interp_bin for every 2-D group (A/B); =1 also for few values per node
bool interp_strip_supported(int d, int taps, int F, int ops, int rc) {
  static const int mode = getenv("AKM_INTERP_STRIP") ? atoi(getenv("AKM_INTERP_STRIP")) : -1;
  if (mode == 0 || d != 2 || F - taps + 1 > 8 || F < taps) return false;
  if (mode < 0 && ops * rc < 4) return false;  // few values per node: N too narrow for the tensor pipe
  if (interp_strip_smem(taps, F, ops * rc) > kIsSmemMax) return false;
#define AKM_IS_SUP(T, O, R) \
  if (taps == T && ops == O && rc == R) return true;
  AKM_IS_INSTANCES(AKM_IS_SUP)
#undef AKM_IS_SUP
  return false;
}

cudaError_t launch_interp_strip(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                                const double* u_sorted, const int* perm, const double* H, int taps, int F, int ops,
                                int r, int r0, int rc, double* part, long long n, cudaStream_t s) {
  if (n_items <= 0) return cudaSuccess;
  const size_t smem = interp_strip_smem(taps, F, ops * rc);
#define AKM_IS_CASE(T, O, R)                                                                                   \
  if (taps == T && ops == O && rc == R) {                                                                      \
    static std::atomic<unsigned long long> attr_set{0};                                                        \
    if (!optin_done(attr_set)) {                                                                               \
      cudaError_t e = cudaFuncSetAttribute(k_interp_strip<T, O, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           (int)kIsSmemMax);                                                  \
      if (e != cudaSuccess) return e;                                                                          \
      optin_mark(attr_set);                                                                                    \
    }                                                                                                          \
    if (smem > kIsSmemMax) return cudaErrorInvalidValue;                                                       \
    k_interp_strip<T, O, R><<<n_items, kIsThreads, smem, s>>>(dtab, items, u_sorted, perm, H, r, r0, part, n, F, \
                                                              pp);                                             \
    return cudaGetLastError();                                                                                 \
  }
  AKM_IS_INSTANCES(AKM_IS_CASE)
#undef AKM_IS_CASE
  return cudaErrorInvalidValue;
}

}  // namespace akm
