// akm_internal.cuh -- shared definitions of the CUDA implementation behind include/akm.h.
//
// Geometry conventions:
//   * Every window is handled in a "padded 3-D" form: padded axis a in {0,1,2}; the window's
//     d axes are the last d padded axes, the leading 3-d axes are singletons (length 1, k = 0).
//   * Scaled grid coordinate of point j along a real axis: u = (x - center) * n_g / c_w
//     (x~ = (x - center)/c_w in the ball of radius 1/4 - eps_B/2; u = n_g x~).
//   * Taps (App. A): the point touches grid nodes l = floor(u) - m + 1 + o,
//     o in [0, 2m).  The window is taken as zero at |u - l| >= m: the closed end of the support
//     carries weight phi(m/n_g)/phi(0) ~ 3e-11 (m = 6) and matters only for integer u
//     (reading R3).
//   * The grid "box" of a window is the range of nodes any point can touch; all grids and
//     spectra are stored box-local.  cell_t = floor(u_t) - (box_lo_t + m - 1) in [0, ncell_t).
//   * Bins are B^d blocks of cells; a bin's footprint is F = B + 2m - 1 nodes per real axis.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace akm {

constexpr int kMaxWin = 32;
constexpr int kPolyDeg = 14;              // window polynomial degree (see window_taps)
constexpr int kPolyLen = kPolyDeg + 1;
constexpr int kMaxTaps = 16;              // 2m <= 16
constexpr double kPi = 3.14159265358979323846;
constexpr int kKrMaxR = 32;               // Krylov driver: 1 CG column + <= 31 probes
constexpr int kKrMaxSteps = 64;           // Lanczos steps
constexpr int kKrMaxIters = 1024;         // CG iterations
constexpr int kRegMaxP = 8;               // regularisation order p (regularize.cu)
constexpr int kRegNfOff = 3 * kRegMaxP;   // per (window, operator): T_I (p) then T_B (2p) coefficients,
constexpr int kRegNfLen = 24;             // then the near-field series: degree (or -1), coefficients
constexpr int kRegStride = kRegNfOff + kRegNfLen;

// Per-window geometry passed (by value, inside WinTable) to kernels.
struct WinGeom {
  int d;
  int feat[3];          // feature ids of the window's axes, padded axis a -> feat[a] (a >= 3-d)
  double center[3];     // per padded axis (0 for singleton axes)
  double scale;         // n_g / c_w
  int box_lo[3];        // global grid index of box node 0 (0 for singleton axes)
  int L[3];             // box length (1 for singleton axes)
  int ncell[3];         // cells per axis (1 for singleton axes)
  int B;                // bin edge (cells)
  int F[3];             // bin footprint per axis (1 for singleton axes)
  int nbin[3];          // bins per axis
  int K[3];             // spectrum sizes: K[2] = N/2+1; K[0],K[1] = N+1 or 1 (singleton)
  long long tap_off;    // offset of this window's box in "tap" units (grids are [tap][...])
  long long ntap;       // L0*L1*L2
  long long pt_off;     // offset of this window's points in the sorted arrays (w * n)
  long long a1_off;     // offsets (complex units, per RHS) into the FFT work buffers
  long long a2_off;
  long long a3_off;     // [k0][k1][k2]
  long long c_off;      // OPS-major: [op][L0][K1][K2]
  long long c2_off;     // [op][L0][L1][K2]
  long long tw_off[3];  // offsets of twiddle tables (complex) for each padded axis: [K][L]
  long long d_off;      // offset of this window's multiplier tables [op][K0][K1][K2] (real)
  int bt_off;           // offset of this window's bin-start table (nbin0*nbin1*nbin2 + 1 entries)
};

// Window polynomial coefficients passed BY VALUE as a __grid_constant__ kernel parameter: with
// compile-time indices the FP64 FMAs read them straight from the constant bank (no smem loads).
struct PolyParam {
  double c[kMaxTaps * kPolyLen];
};

// float-reciprocal integer division for small non-negative operands (a < 2^20, b <= 2^10):
// exact because the rounding error of (a + 1/2) / b stays far below 1/(2b).
__device__ __forceinline__ int fdiv(int a, float inv_b) { return (int)(((float)a + 0.5f) * inv_b); }

struct WinTable {
  int P;
  int N, n_g, m;
  double poly[kMaxTaps * kPolyLen];  // window polynomial coefficients (see window_taps)
  WinGeom w[kMaxWin];
};

// One unit of spreading / interpolation work: a chunk of points of one bin.
struct WorkItem {
  int win;
  int bin[3];       // bin coordinates per padded axis
  int start;        // first sorted point (window-relative)
  int count;        // number of points
};

// Deterministic spreading (akm_set_deterministic; spread_det.cu): each footprint flush adds v * 2^S_c
// (S_c per RHS column, from its max |v| and n) as three signed 40-bit integer limbs with 64-bit
// integer atomics -- exact and order-independent -- and one pass converts the limb sums to float64.
struct DetAcc {
  unsigned long long* limbs = nullptr;  // [3][stride]; nullptr = float64 atomics into the grid
  const int* S = nullptr;               // [window][r_total] scale exponents
  long long stride = 0;                 // total_taps * r_total
  int r_total = 0;
};
// per-window bounds of the scale exponents (the window product W^d differs by ~1e12 per axis)
struct DetWin {
  int wbits[kMaxWin];            // ceil(d_w log2 W) + 1
  long long tap_off[kMaxWin + 1];  // window w's grid nodes: [tap_off[w], tap_off[w + 1])
  int P;
};
__device__ __forceinline__ void det_add(const DetAcc& da, int win, long long idx, int col, double v) {
  const double x = ldexp(v, da.S[win * da.r_total + col]);  // exact (power-of-two scaling)
  const double h2 = trunc(ldexp(x, -80));
  const double r1 = x - ldexp(h2, 80);        // exact: the bits of x below 2^80
  const double h1 = trunc(ldexp(r1, -40));
  const double r0 = r1 - ldexp(h1, 40);       // exact
  const double h0 = trunc(r0);                // drops the bits below one unit (2^-S)
  atomicAdd(da.limbs + idx, (unsigned long long)(long long)h0);
  atomicAdd(da.limbs + da.stride + idx, (unsigned long long)(long long)h1);
  atomicAdd(da.limbs + 2 * da.stride + idx, (unsigned long long)(long long)h2);
}

// ------------------------------------------------------------------ device helpers
// Kaiser-Bessel window (App. A) at a distance delta = n_g * x in grid cells:
//   phi = (1/pi) sinh(beta sqrt(m^2 - delta^2)) / sqrt(m^2 - delta^2) for |delta| < m,
//   0 otherwise (truncated; reading R3 for the end point).
__device__ __forceinline__ double kb_window(double delta, double m, double beta) {
  const double s = m * m - delta * delta;
  if (s > 0.0) {
    const double q = sqrt(s);
    return sinh(beta * q) / (kPi * q);
  }
  return 0.0;
}

// Window polynomials: for tap o in [0, 2m) of a point with fractional grid
// position t = u - floor(u), the weight phi(t + m - 1 - o) is an entire function of t on [0, 1]
// (sinh(beta q)/q is analytic in q^2 = m^2 - delta^2).  It is replaced by its degree-kPolyDeg
// Chebyshev interpolant on [0, 1], stored as monomial coefficients in x = 2t - 1 (Horner).
// Max error <= 2e-14 * phi(0) for m in {4,6,8}, sigma in {1.25, 2} (measured 1.2e-14 at m = 8,
// sigma = 2: rounding of the monomial form), checked against the exact sinh form by
// tests/test_gpu_parity.py::test_window_polynomials_vs_exact_kaiser_bessel via akm_get_window_poly.

// Evaluate the 2m tap weights of one axis at x = 2 frac(u) - 1 from coefficients c[o*kPolyLen + k].
template <int TAPS>
__device__ __forceinline__ void window_taps(const double* __restrict__ c, double x, double* w) {
#pragma unroll
  for (int o = 0; o < TAPS; ++o) {
    double v = c[o * kPolyLen + kPolyDeg];
#pragma unroll
    for (int k = kPolyDeg - 1; k >= 0; --k) v = fma(v, x, c[o * kPolyLen + k]);
    w[o] = v;
  }
}

// The same polynomials by Estrin's scheme: dependency depth 4 (after x^2, x^4, x^8, shared by all
// taps) instead of 14.  Used where the weights are evaluated next to DMMA traffic, which stretches
// every dependent FP64 step to ~135 clk (tools/microbench/dmma_occupancy.cu).
static_assert(kPolyDeg == 14, "Estrin layout below assumes degree 14");
template <int TAPS>
__device__ __forceinline__ void window_taps_estrin(const double* __restrict__ c, double x, double* w) {
  const double x2 = x * x, x4 = x2 * x2, x8 = x4 * x4;
#pragma unroll
  for (int o = 0; o < TAPS; ++o) {
    const double* k = c + o * kPolyLen;
    const double p0 = fma(k[1], x, k[0]), p1 = fma(k[3], x, k[2]), p2 = fma(k[5], x, k[4]);
    const double p3 = fma(k[7], x, k[6]), p4 = fma(k[9], x, k[8]), p5 = fma(k[11], x, k[10]);
    const double p6 = fma(k[13], x, k[12]), p7 = k[14];
    const double q0 = fma(p1, x2, p0), q1 = fma(p3, x2, p2), q2 = fma(p5, x2, p4), q3 = fma(p7, x2, p6);
    const double r0 = fma(q1, x4, q0), r1 = fma(q3, x4, q2);
    w[o] = fma(r1, x8, r0);
  }
}

// Estrin evaluation of the K taps first, first + stride, ... (shared x powers)
template <int K>
__device__ __forceinline__ void window_taps_estrin_strided(const double* __restrict__ c, int first, int stride,
                                                           double x, double* w) {
  const double x2 = x * x, x4 = x2 * x2, x8 = x4 * x4;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const double* k = c + (first + q * stride) * kPolyLen;
    const double p0 = fma(k[1], x, k[0]), p1 = fma(k[3], x, k[2]), p2 = fma(k[5], x, k[4]);
    const double p3 = fma(k[7], x, k[6]), p4 = fma(k[9], x, k[8]), p5 = fma(k[11], x, k[10]);
    const double p6 = fma(k[13], x, k[12]), p7 = k[14];
    const double q0 = fma(p1, x2, p0), q1 = fma(p3, x2, p2), q2 = fma(p5, x2, p4), q3 = fma(p7, x2, p6);
    const double r0 = fma(q1, x4, q0), r1 = fma(q3, x4, q2);
    w[q] = fma(r1, x8, r0);
  }
}

__device__ __forceinline__ double window_tap(const double* __restrict__ c, int o, double x) {
  double v = c[o * kPolyLen + kPolyDeg];
#pragma unroll
  for (int k = kPolyDeg - 1; k >= 0; --k) v = fma(v, x, c[o * kPolyLen + k]);
  return v;
}

// FP64 tensor-core MMA (mma.sync.m8n8k4.f64), fragment layout verified on sm_100a by
// tools/microbench/dmma_layout.cu:  A (8x4 row) a = A[lane>>2][lane&3];  B (4x8 col)
// b = B[lane&3][lane>>2];  C (8x8) c{0,1} = C[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// shared-memory row stride (doubles) of a matrix read as MMA fragments: = 4 (mod 16) makes the
// 4 k-rows x 8 columns of a fragment load hit 32 distinct banks.
__host__ __device__ constexpr int mma_ld(int cols) { return ((cols + 15) / 16) * 16 + 4; }

// Modified Bessel I0 by its power series sum_k ((x/2)^{2k} / (k!)^2); x <= ~60 here.
__host__ __device__ inline double bessel_i0(double x) {
  const double q = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 200; ++k) {
    term *= q / ((double)k * (double)k);
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}

// Tensor maps of the interpolation grids H per window (TMA staging in k_interp_mma; interp.cu builds
// them, interp_impl.cuh consumes them as a __grid_constant__ kernel parameter).
constexpr int kTmaWin = 8;
struct TmaMaps {
  CUtensorMap m[kTmaWin];
};

// Opt-ins to more than 48 KB of dynamic shared memory (cudaFuncSetAttribute) hold per device: each
// launch site keeps one bit per device.  Two threads racing on the first launch both set
// the attribute, which is idempotent.
inline bool optin_done(const std::atomic<unsigned long long>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  return (mask.load(std::memory_order_acquire) >> (dev & 63)) & 1ull;
}
inline void optin_mark(std::atomic<unsigned long long>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  mask.fetch_or(1ull << (dev & 63), std::memory_order_release);
}

}  // namespace akm

// ------------------------------------------------------------------ launchers (host side)
// `tab` is the host copy of the window table (sizes for grid dimensions), `dtab` its device copy.
namespace akm {
// setup_kernels.cu
cudaError_t launch_gather_columns(const double* X, long long n, long long ldx, const int* feat, int nf, double* Xc,
                                  cudaStream_t s);
cudaError_t launch_window_minmax(const double* X, long long n, long long ldx, const int* feat_dev, int nfeat,
                                 double* minmax_dev, cudaStream_t s);
cudaError_t launch_window_radius(const double* X, long long n, long long ldx, const WinTable& tab,
                                 const WinTable* dtab, double* r2_dev, cudaStream_t s);
cudaError_t launch_scale_and_key(const double* X, long long n, long long ldx, const WinTable& tab,
                                 const WinTable* dtab, double* u_tmp, int* key, int* hist, const long long* hist_off,
                                 int* err_flag, long long n_split, cudaStream_t s);
// binsort.cu: S0 on the device (candidate bin statistics, bin-major layout, cursors, work items)
constexpr int kBinCands = 6;  // candidate bin edges B = 1, 2, 3, 4, 6, 8
struct BinCandParam {
  long long off[kMaxWin][kBinCands];  // offset of each (window, candidate) per-bin count array
  int B[kBinCands];
  int mask[kMaxWin];                  // candidates that fit, per window
};
struct BinLayout {
  long long keybase[kMaxWin];  // first key of each window in the (group-ordered) key space
  long long binbase[kMaxWin];  // first bin of each window in the (group-ordered) bin space
};
constexpr int kItemLists = 6;  // per-cell interp (set 0, 1), spread set 0, per-bin set 0, spread set 1, per-bin set 1
struct ListScanParam {
  const int* cnt[kItemLists];
  const int* off[kItemLists];
  long long len[kItemLists];
  long long gbeg[kItemLists][kMaxWin + 1];  // index-space start of every group, then len
  int nlists;
};
cudaError_t launch_bin_costs(const WinTable& tab, const WinTable* dtab, const int* hist, const long long* hist_off,
                             const BinCandParam& cp, long long bc_total, int* bc, long long ch_s, int* stats,
                             cudaStream_t s);
cudaError_t launch_slot_keys(const WinTable& tab, const WinTable* dtab, const int* hist, const long long* hist_off,
                             const BinLayout& L, long long* key_cnt, int* i0cnt, int* i1cnt, int ch_i, cudaStream_t s);
cudaError_t launch_slot_cursor(const WinTable& tab, const WinTable* dtab, const long long* hist_off, const BinLayout& L,
                               const long long* key_cnt, const long long* key_off, int* cursor, int2* cell_tab,
                               cudaStream_t s);
cudaError_t launch_bin_pass(const WinTable& tab, const WinTable* dtab, const BinLayout& L, const long long* key_off,
                            long long n, long long ch_s, int ch_ib, int* bin_start, int* s0, int* b0, int* s1, int* b1,
                            cudaStream_t s);
cudaError_t launch_group_bounds(const ListScanParam& lp, int ngroups, int* bounds, cudaStream_t s);
cudaError_t launch_emit_items(const WinTable& tab, const WinTable* dtab, const BinLayout& L, const long long* key_cnt,
                              const long long* key_off, long long n, long long ch_s, int ch_i, int ch_ib,
                              const int* const off[6], WorkItem* const out[6], cudaStream_t s);
cudaError_t scan_excl_ll(const long long* in, long long* out, long long len, void** temp, size_t* temp_bytes,
                         cudaStream_t s);
cudaError_t scan_excl_int(const int* in, int* out, long long len, void** temp, size_t* temp_bytes, cudaStream_t s);
struct WinGroupMap {
  int group[kMaxWin];  // window -> its group's position in the launch order
};
cudaError_t sort_points(long long n, const WinTable& tab, const WinTable* dtab, const BinLayout& L, long long nkeys,
                        const WinGroupMap& order, const double* u_tmp, long long n_split, unsigned* keys,
                        unsigned* keys_alt, int* vals, int* vals_alt, void** temp, size_t* temp_bytes,
                        double* u_sorted, int* perm, cudaStream_t s);
cudaError_t sort_items_larger_first(const WorkItem* in, long long cnt, int maxc, const WinGroupMap& gm, int ngroups,
                                    unsigned* keys, unsigned* keys_alt, int* idx, int* idx_alt, void** temp,
                                    size_t* temp_bytes, WorkItem* out, cudaStream_t s);

cudaError_t launch_kernel_samples(int family, int d, int N, double ell_eff, int deriv, double* out, cudaStream_t s);
cudaError_t launch_cos_dft_axis(int d, int N, int axis, const double* in, double* out, cudaStream_t s);
cudaError_t launch_deconv_table(int N, int n_g, int m, double sigma_over, double* i0sq, cudaStream_t s);
cudaError_t launch_multiplier(const WinTable& tab, const WinTable* dtab, int win, const double* bK, const double* bL,
                              int ops_mask, double inv_c, const double* i0sq, double* D, cudaStream_t s);
cudaError_t launch_twiddles(const WinTable& tab, const WinTable* dtab, double2* tw, cudaStream_t s);
cudaError_t launch_window_poly(int m, double beta, double* coef, cudaStream_t s);

// regularize.cu
cudaError_t launch_reg_coef(int family, double ell_eff, double eps_I, double eps_B, int p, double* coef, cudaStream_t s);
cudaError_t launch_kernel_samples_reg(int family, int d, int N, double ell_eff, int deriv, double eps_I, double eps_B,
                                      int p, const double* coef, double* out, cudaStream_t s);
cudaError_t launch_near_field(const WinTable* dtab, const WorkItem* items, int n_items, const int2* cell_tab,
                              const long long* cell_off, const double* u_sorted, const int* perm, const double* V,
                              long long ldv, double* Vs, long long n, int P, int r, int ops, int slotK, int slotL,
                              int family, double ell, double eps_I, int p, const double* coef, double* part,
                              cudaStream_t s);
int near_field_launches(int r);

// aafn.cu
size_t fps_scratch_bytes();
cudaError_t launch_fps(const double* Xc, long long n, int nf, const int* cols, int d, int k, int* picks, double* dmin,
                       void* scratch, cudaStream_t s);
cudaError_t launch_lmpos(long long n, int k, const int* lm, int* lmpos, cudaStream_t s);
cudaError_t launch_aafn_factor(const double* Xc, long long n, int nf, const WinTable& tab, int family, double sf,
                               double ell, double se, const int* lm, const int* lmpos, int k, double* L, double* Linv,
                               double* LinvT, double* Phi, double* K21, double* Sdiag, double* g, double* scal,
                               double* part, int* flag, double jitter, cudaStream_t s);
size_t aafn_part_doubles(long long n, int k, int R);
cudaError_t launch_resid_norms(long long n, const double* y, const double* Kx, double* part, double* out, cudaStream_t s);
cudaError_t launch_aafn_uinv(long long n, int k, int R, const int* lm, const int* lmpos, const double* Linv,
                             const double* Phi, const double* g, const double* T, double* y1, double* tmp,
                             double* part, double* out, cudaStream_t s);
cudaError_t launch_aafn_uinvT(long long n, int k, int R, const int* lm, const int* lmpos, const double* LinvT,
                              const double* Phi, const double* g, const double* Y, double* part, double* tmp,
                              double* w1, double* w2buf, double* out, cudaStream_t s);

// spread_mma.cu
bool spread_mma_choose(int M, int Nn, int Fmax, int rc, int& MB, int& NB, int& WM, int& WN);
size_t spread_mma_smem(int PB, int M, int Nn, int Fmax, int rc);
cudaError_t launch_spread_mma(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                              const double* u_sorted,
                              const int* perm, const double* V, long long ldv, long long n, int r0, int rc,
                              int r_total, double* grid, int MB, int NB, int WM, int WN, int PB, size_t smem,
                              cudaStream_t s, const DetAcc& da = DetAcc{});

// spread_v5.cu (one warp per SM sub-partition, fragments formed on the fly)
bool spread_v5_choose(int M, int Nn, int& MB, int& NB, int& WN);
size_t spread_v5_smem(int Fmax, int rc, int MB, int NB, int WN);
cudaError_t launch_spread_v5(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                             const double* u_sorted, const int* perm, const double* V, long long ldv, long long n,
                             int r0, int rc, int r_total, double* grid, int MB, int NB, int WN, size_t smem,
                             cudaStream_t s, const DetAcc& da = DetAcc{});

// spread_strip.cu (2-D windows: per bin, one DMMA GEMM per strip of 1 x B cells, M = the 2m axis-1 taps)
int spread_strip_nb(int d, int taps, int F, int rc);
cudaError_t launch_spread_strip(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                                const double* u_sorted, const int* perm, const double* V, long long ldv, long long n,
                                int r0, int rc, int r_total, double* grid, int taps, int F, int nb, cudaStream_t s,
                                const DetAcc& da);

// interp_pt.cu (small launches: one warp per point, taps over the lanes, H straight from L2)
bool interp_pt_choose(int d, int taps, int ops, int rc, int n_items_bin);
cudaError_t launch_interp_pt(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                             const double* u_sorted, const int* perm, const double* H, int d, int taps, int ops,
                             int r, int r0, int rc, double* part, long long n, cudaStream_t s);

// interp_strip.cu (2-D windows: per bin, one DMMA GEMM per strip of 1 x B cells, K = axis-2 nodes)
bool interp_strip_supported(int d, int taps, int F, int ops, int rc);
cudaError_t launch_interp_strip(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                                const double* u_sorted, const int* perm, const double* H, int taps, int F, int ops,
                                int r, int r0, int rc, double* part, long long n, cudaStream_t s);

// interp_t.cu (3-D windows, many values per node: GEMM over (o0, o1) with N = (o2, v))
bool interp_t_supported(int d, int taps, int fp, int ops, int rc);
cudaError_t launch_interp_t(const WinTable* dtab, const PolyParam& pp, const WorkItem* items, int n_items,
                            const double* u_sorted, const int* perm, const double* H, int taps, int fp, int ops, int r,
                            int r0, int rc, double* part, long long n, cudaStream_t s, int bscale);

// fft.cu
cudaError_t launch_fft_forward(const WinTable& tab, const WinTable* dtab, const double* grid, double2* A1,
                               double2* A2, const double2* tw, int r, cudaStream_t s);
cudaError_t launch_fft_multiply_inverse(const WinTable& tab, const WinTable* dtab, const double2* A2, double2* A3,
                                        double2* C, double2* C2, const double2* tw, const double* D, int ops, int dslot0, int r,
                                        double* H, cudaStream_t s);
cudaError_t launch_zero(double* p, long long count, cudaStream_t s);

cudaError_t launch_det_prepare(const double* V, long long ldv, long long n, int r, const DetWin& dw,
                               unsigned long long* colmax, int* S, unsigned long long* limbs, long long stride,
                               cudaStream_t s);
cudaError_t launch_det_finish(const unsigned long long* limbs, const int* S, long long stride, int r,
                              const DetWin& dw, double* grid, cudaStream_t s);
int fft_launch_count(const WinTable& tab, int r);

// krylov.cu (config-5 objective driver)
size_t kr_state_bytes();
// block PCG for the gradient (krylov.cu)
size_t bcg_state_bytes();
cudaError_t launch_bcg_init(void* st, const double* part, int R, double c, cudaStream_t s);
cudaError_t launch_bcg_start(long long n, int R, const void* st, const double* B, double* Rr, double* P, double* X,
                             cudaStream_t s);
cudaError_t launch_bcg_after_dots(void* st, const double* part, int R, cudaStream_t s);
cudaError_t launch_bcg_update(long long n, int R, const void* st, const double* P, const double* KP, double* Rr,
                              double* X, cudaStream_t s);
cudaError_t launch_bcg_after_norms(void* st, const double* part, int R, int t, cudaStream_t s);
cudaError_t launch_bcg_dir(long long n, int R, const void* st, const double* Rr, double* P, cudaStream_t s);
cudaError_t launch_bcg_grad_rhs(long long n, int R, const double* X, const double* B, double* B2, cudaStream_t s);
cudaError_t launch_bcg_store(void* st, const double* part, int R, int slot, cudaStream_t s);
void bcg_offsets(size_t* off_hist, size_t* off_out, size_t* off_bnorm);
int kr_blocks();
cudaError_t launch_kr_col2(long long n, int R, const double* A, const double* B, double* part, cudaStream_t s);
cudaError_t launch_kr_load(long long n, int R, const double* y, const double* Z, long long ldz, double* B,
                           double* ybuf, cudaStream_t s);
cudaError_t launch_kr_init(void* st, const double* part, int R, double c, cudaStream_t s);
cudaError_t launch_kr_start(long long n, int R, const void* st, double* B, double* W, double* Q0, double* x,
                            cudaStream_t s);
cudaError_t launch_kr_after_dots(void* st, const double* part, int R, int cg_iters, int lanczos_steps, cudaStream_t s);
cudaError_t launch_kr_update(long long n, int R, const void* st, const double* B, const double* KB, double* W,
                             const double* Qt, const double* Qtm1, double* x, cudaStream_t s);
cudaError_t launch_kr_reorth(long long n, int R, int nq, const void* st, const double* Q, long long slab, double* W,
                             double* part, double* h, cudaStream_t s);
cudaError_t launch_kr_after_norms(void* st, const double* part, int R, cudaStream_t s);
cudaError_t launch_kr_finalize(long long n, int R, void* st, double* B, const double* W, double* Qn, cudaStream_t s);
cudaError_t launch_kr_advance(void* st, int R, cudaStream_t s);
cudaError_t launch_kr_slq_quad(void* st, int R, const double* part_yx, int* err, cudaStream_t s);
void kr_summary_offsets(size_t* off_quad, size_t* off_samples, size_t* off_steps, size_t* off_hist, size_t* off_znorm);

// interp.cu (tma: host TmaMaps of the H grids for the TMA-staged k_interp_mma, or nullptr)
size_t interp_tma_maps_bytes();
bool interp_tma_build(const WinTable& tab, const double* H, int ops, int r, void* maps);
int interp_rc_for(int r_remaining);
cudaError_t launch_interp(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                          int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm, const double* H,
                          int d, int taps, int ops, int r, int r0, int rc, double* part, long long n, const void* tma,
                          cudaStream_t s);
cudaError_t launch_epilogue_cross(long long n, long long n_src, int P, int r, int ops, int slotK, const double* part,
                                  double sigma_f, double* Yt, long long ldy, cudaStream_t s);
cudaError_t launch_epilogue(long long n, int P, int r, int ops, const double* part, const double* V, long long ldv,
                            double sigma_f, double sigma_eps, double* Y, double* dYl, double* dYsf, long long ldy,
                            int slotK, int slotL, cudaStream_t s);
cudaError_t launch_scaled_copy(long long n, int r, double alpha, const double* V, long long ldv, double* Y,
                               long long ldy, cudaStream_t s);
}  // namespace akm
