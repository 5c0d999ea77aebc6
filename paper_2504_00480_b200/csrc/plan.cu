// plan.cu -- the C ABI of include/akm.h: plan state, validation, workspace, orchestration.
//
// Host code here only validates arguments, sizes buffers, chooses bin sizes / tiles from
// device-computed histograms, and enqueues the kernels of setup_kernels.cu, spread.cu, fft.cu and
// interp.cu on the caller's stream.  All per-point, per-grid-node and per-frequency arithmetic
// of the method runs in those kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/akm.h"
#include "akm_internal.cuh"

using namespace akm;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  // grow-only; contents are not preserved
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    release();
    if (need == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc(&p, need);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      return e;
    }
    bytes = need;
    return cudaSuccess;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};


struct ItemSlice {  // a group's slice of the concatenated work items of one item set
  int spread_begin = 0, spread_count = 0;
  int interp_begin = 0, interp_count = 0;
  int interp_bin_begin = 0, interp_bin_count = 0;
  bool sparse = false;  // few points per occupied cell: interpolate per bin (scalar) rather than per cell
};

struct Group {  // windows sharing (d, F) -> one spread / interp launch
  int d = 0, F = 0;
  std::vector<int> wins;
  ItemSlice sl[2];  // item set 0: square product; 1: cross product (sources -> targets)
};

}  // namespace


struct akm_plan {
  int device = 0;
  std::string err;
  bool have_points = false, have_theta = false;

  // problem
  long long n = 0;
  int p = 0, P = 0, family = 0, N = 0, m = 0, n_g = 0;
  double sigma_over = 2.0, eps_B = 0.0, beta = 0.0;
  std::vector<int> win_len, win_feat;       // as given
  std::vector<int> feat_used;               // distinct features, compact column order
  double sigma_f = 1.0, ell = 1.0, sigma_eps = 0.0;
  std::vector<double> scale_override;       // empty = automatic rule (reading R2)

  // per-window host data
  std::vector<double> lo, hi;               // [w*3 + a] bounding box (padded axes)
  std::vector<double> radius;               // R_w (global after akm_set_radius)
  std::vector<double> radius_local;         // R_w of this plan's own points about the current centers
  std::vector<int> bin_override;            // empty = cost-model choice of B per window (rebuild_bins)
  // AAFN preconditioner (aafn.cu; akm_set_preconditioner).  Landmarks depend on the points only, the
  // factors on theta (rebuilt lazily when theta_version moved).
  struct Aafn {
    int kpw = 0;                  // landmarks per window; 0 = diagonal preconditioner
    bool lm_ready = false;
    long long theta_built = -1;
    int k = 0;
    double logdet = 0.0;          // log det M
    DevBuf lm, lmpos, L, Linv, LinvT, Phi, K21, Sdiag, g, y1, part, tmp, scal, flag, fps_scratch, dmin, picks, Bt, KBt,
        yh, Bh, w2;
  } aafn;
  long long theta_version = 0;
  struct BkKey {
    bool valid = false;
    int family = 0, d = 0, N = 0, reg_p = 0;
    double ell_eff = 0.0, eps_I = 0.0, eps_B = 0.0;
    bool operator==(const BkKey& o) const {
      return valid && o.valid && family == o.family && d == o.d && N == o.N && reg_p == o.reg_p &&
             ell_eff == o.ell_eff && eps_I == o.eps_I && eps_B == o.eps_B;
    }
  };
  std::vector<BkKey> bk_keys;  // per window: what its b_k tables were built for
  long long bk_stride = 0;
  DevBuf bk;
  int reg_p = 0;                            // kappa_R regularisation (akm_set_regularization; 0 = off)
  double reg_eps_I = 0.0;
  bool near_field() const { return reg_p > 0 && reg_eps_I > 0.0; }
  std::vector<double> c_w, c_w_binned;      // current scale, scale the bins were built for
  WinTable tab{};                           // host copy
  PolyParam poly_param{};                   // window polynomials, passed to kernels by value
  size_t n_items_spread[2] = {0, 0}, n_items_interp[2] = {0, 0}, n_items_interp_bin[2] = {0, 0};  // [item set]
  std::vector<Group> groups;
  std::vector<long long> occupied, maxbin;
  long long total_taps = 0, szA1 = 0, szA2 = 0, szA3 = 0, szC = 0, szC2 = 0, szTW = 0, szD = 0;

  // device buffers
  DevBuf dtab, Xc, u_tmp, u_sorted, perm, hist, hist_off, err_flag, minmax, r2;
  DevBuf items_s[2], items_i[2], items_ib[2];  // [item set]
  long long n_split = 0;  // rows >= n_split are class 1 (cross-product targets); n = no targets
  DevBuf grid, H, A1, A2, A3, C, C2, tw, D, part, bs0, bs1, bs2, bs3;
  DevBuf reg_coef, bin_start;  // regularisation polynomials [w][op][kRegStride]; per-window bin start tables
  DevBuf cell_tab, nfV;        // near field: (start, count) per (cell, class) slot; bin-sorted copy of V
  bool cell_tab_ok = false;      // cell_tab matches the last bin sort (built on demand: near field only)
  DevBuf deconv;                 // [3][N + 1] per-axis deconvolution factors (setup_kernels.cu k_deconv_table)
  bool det = false;              // deterministic spreading (akm_set_deterministic)
  DevBuf det_limbs, det_colmax, det_S;
  DetWin det_win{};
  bool deconv_ok = false;
  // S0 on the device (binsort.cu): candidate statistics, key space (bin-major slot order) counts and
  // offsets, per-list item counts / offsets, unsorted items, sort scratch, group bounds
  DevBuf bs_bc, bs_stats, key_cnt, key_off, lcnt[kItemLists], loff[kItemLists], items_u[kItemLists];
  DevBuf sort_keys, sort_idx, bounds, pt_keys, pt_vals;
  void* cub_temp = nullptr;
  size_t cub_temp_bytes = 0;
  BinLayout bl{};
  std::vector<unsigned char> tma_maps = std::vector<unsigned char>(interp_tma_maps_bytes());  // TmaMaps (host)
  DevBuf stageV, stageY, stageL, stageS;
  DevBuf crossV, crossY;  // akm_kernel_cross_mvm: zero-padded V and the union's product
  DevBuf gX, gP, gB2, gD1, gD2, gState;  // akm_gradient_diag: block PCG and derivative products
  DevBuf krB, krKB, krW, krX, krY, krQ, krPart, krH, krState, krErr, krStage, krRes;
  long long r_cap = 0;

  // CUDA graph of the last MVM launch sequence (replayed when called again with the same buffers)
  struct GraphKey {
    const void *V, *Y, *dYl, *dYsf;
    long long ldv, ldy;
    int r;
    long long epoch;
    int set;
    bool operator==(const GraphKey& o) const {
      return V == o.V && Y == o.Y && dYl == o.dYl && dYsf == o.dYsf && ldv == o.ldv && ldy == o.ldy && r == o.r &&
             epoch == o.epoch && set == o.set;
    }
  };
  long long epoch = 0;                 // bumped whenever buffers, items or theta change
  // small LRU of captured launch sequences: the Krylov drivers alternate between a few (V, Y, r)
  // combinations; entries of an older epoch are never matched and age out
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    GraphKey key{};
    long long launches = 0, spread = 0, interp = 0, last_use = 0;
  };
  static constexpr int kGraphSlots = 4;
  GraphEntry graphs[kGraphSlots];
  long long graph_clock = 0;
  cudaStream_t own_stream = nullptr;   // used to capture / replay when the caller passes the legacy stream
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  bool use_graphs = true;

  // akm_kernel_mvm_pipelined: two device slots (V in, outputs out) and the copy streams; slot j's
  // events order the copy-in after the product that last read V[j], the product after the copy-out
  // that last read O[j], and the copy-out after its product
  struct Pipe {
    cudaStream_t cin = nullptr, cout = nullptr;
    DevBuf V[2], O[2][3];
    cudaEvent_t in_done[2] = {}, comp_done[2] = {}, out_done[2] = {};
    bool live[2] = {false, false};
    int next = 0, last = -1;
  } pipe;

  // profiling (akm_set_profiling / akm_get_stage_times): a ring of event sets, drained lazily
  // e[0] spread start, e[1] spread end, e[5] finish start (== e[1] unless the grids were exchanged
  // between akm_spread_grid and akm_mvm_from_grid), e[2] DFT end, e[3] interpolation end, e[4] end
  static constexpr int kRing = 512;
  struct EvSet { cudaEvent_t e[6]; bool pending = false; };
  bool profiling = false;
  std::vector<EvSet> ring;
  int ring_pos = 0;
  EvSet* split_ev = nullptr;  // set by akm_spread_grid, consumed by akm_mvm_from_grid
  double stage_ms[5] = {0, 0, 0, 0, 0};  // spread, fft, interp, epilogue, exchange
  long long prof_calls = 0, launches = 0, spread_launches = 0, interp_launches = 0;

  void drain(EvSet& es) {
    if (!es.pending) return;
    cudaEventSynchronize(es.e[4]);
    const int from[5] = {0, 5, 2, 3, 1}, to[5] = {1, 2, 3, 4, 5};
    for (int k = 0; k < 5; ++k) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, es.e[from[k]], es.e[to[k]]) == cudaSuccess) stage_ms[k] += ms;
      else cudaGetLastError();
    }
    es.pending = false;
  }
  EvSet* next_set() {
    if (ring.empty()) {
      ring.resize(kRing);
      for (auto& es : ring)
        for (auto& e : es.e) cudaEventCreate(&e);
    }
    EvSet& es = ring[ring_pos];
    ring_pos = (ring_pos + 1) % kRing;
    drain(es);
    es.pending = true;
    ++prof_calls;
    return &es;
  }
  ~akm_plan() {
    if (cub_temp) cudaFree(cub_temp);
    for (auto& es : ring)
      for (auto& e : es.e) cudaEventDestroy(e);
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (pipe.cin) cudaStreamDestroy(pipe.cin);
    if (pipe.cout) cudaStreamDestroy(pipe.cout);
    for (int j = 0; j < 2; ++j)
      for (cudaEvent_t e : {pipe.in_done[j], pipe.comp_done[j], pipe.out_done[j]})
        if (e) cudaEventDestroy(e);
  }

  akm_status fail(akm_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return st;
  }
};

// NVTX ranges per stage: visible in Nsight Systems / ncu --nvtx; header-only NVTX3
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

#define AKM_CK(call)                                                                              \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) {                                                                      \
      akm_status st_ = (e_ == cudaErrorMemoryAllocation) ? AKM_ERR_OOM : AKM_ERR_CUDA;            \
      return plan->fail(st_, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    }                                                                                             \
  } while (0)

namespace {

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

bool is_pinned_host(const void* ptr) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// Row-block copies: one linear copy when both sides are contiguous (a 2-D copy of a million
// 88-byte rows runs row by row on the copy engine), else the strided 2-D copy.
cudaError_t copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                      cudaMemcpyKind kind, cudaStream_t s) {
  if (rows == 0 || width == 0) return cudaSuccess;
  if (dpitch == width && spitch == width) return cudaMemcpyAsync(dst, src, width * rows, kind, s);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, s);
}

}  // namespace


// ================================================================== geometry / binning
// (start, count) of every (cell, class) slot in the window-relative sorted order of the last bin
// sort, for the near-field correction; built on demand (only kappa_R's inner part reads it) from the
// device key counts and offsets of that sort (binsort.cu)
static akm_status ensure_cell_tab(akm_plan* plan, cudaStream_t s) {
  if (plan->cell_tab_ok) return AKM_OK;
  long long ncells = 0;
  for (int w = 0; w < plan->P; ++w) ncells += 2LL * plan->tab.w[w].ncell[0] * plan->tab.w[w].ncell[1] * plan->tab.w[w].ncell[2];
  AKM_CK(plan->cell_tab.ensure(sizeof(int2) * std::max<long long>(ncells, 1)));
  AKM_CK(launch_slot_cursor(plan->tab, plan->dtab.as<WinTable>(), plan->hist_off.as<long long>(), plan->bl,
                            plan->key_cnt.as<long long>(), plan->key_off.as<long long>(), nullptr,
                            plan->cell_tab.as<int2>(), s));
  plan->cell_tab_ok = true;
  return AKM_OK;
}


// AKM_SETUP_TIMES=1: the stages of set_theta / rebuild_bins on stderr (stream synchronised at each mark)
struct SetupTimer {
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit SetupTimer(cudaStream_t st) : s(st), on(std::getenv("AKM_SETUP_TIMES") != nullptr) {
    if (on) t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[akm setup] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

static akm_status rebuild_bins(akm_plan* plan, cudaStream_t s) {
  NvtxRange nvtx("akm S0 bin sort");
  SetupTimer tm(s);
  ++plan->epoch;
  const int P = plan->P, m = plan->m, n_g = plan->n_g;
  const long long n = plan->n;
  WinTable& tab = plan->tab;
  tab.P = P;
  tab.N = plan->N;
  tab.n_g = n_g;
  tab.m = m;
  // pass 0: boxes and cells (independent of B)
  std::vector<long long> hoff(P + 1, 0);
  for (int w = 0; w < P; ++w) {
    WinGeom& g = tab.w[w];
    const double c = plan->c_w[w];
    g.scale = (double)n_g / c;
    for (int a = 0; a < 3; ++a) {
      if (a < 3 - g.d) {
        g.box_lo[a] = 0; g.L[a] = 1; g.ncell[a] = 1; g.K[a] = 1;
        continue;
      }
      // u of the extreme points, computed with the same two IEEE operations as k_scale_and_key
      // (a subtraction and a multiplication cannot be contracted into an FMA), so floor() agrees
      // bit for bit; one cell of slack is kept on each side only when the box still fits n_g.
      const double umin = (plan->lo[w * 3 + a] - g.center[a]) * g.scale;
      const double umax = (plan->hi[w * 3 + a] - g.center[a]) * g.scale;
      int fmin = (int)std::floor(umin), fmax = (int)std::floor(umax);
      if ((fmax - fmin + 2) + 2 * m - 1 <= n_g) {
        fmin -= 1;
        fmax += 1;
      }
      g.box_lo[a] = fmin - m + 1;
      g.ncell[a] = fmax - fmin + 1;
      g.L[a] = g.ncell[a] + 2 * m - 1;
      g.K[a] = (a == 2) ? plan->N / 2 + 1 : plan->N + 1;
    }
    hoff[w + 1] = hoff[w] + 2LL * g.ncell[0] * g.ncell[1] * g.ncell[2];  // (cell, class) slots
  }
  const long long ncells = hoff[P];
  AKM_CK(plan->hist.ensure(sizeof(int) * std::max<long long>(ncells, 1)));
  AKM_CK(plan->hist_off.ensure(sizeof(long long) * (P + 1)));
  AKM_CK(plan->err_flag.ensure(sizeof(int)));
  AKM_CK(plan->u_tmp.ensure(sizeof(double) * 3 * P * std::max<long long>(n, 1)));
  AKM_CK(plan->u_sorted.ensure(sizeof(double) * 3 * P * std::max<long long>(n, 1)));
  AKM_CK(plan->perm.ensure(sizeof(int) * P * std::max<long long>(n, 1)));
  AKM_CK(plan->dtab.ensure(sizeof(WinTable)));
  AKM_CK(cudaMemcpyAsync(plan->dtab.p, &tab, sizeof(WinTable), cudaMemcpyHostToDevice, s));
  AKM_CK(cudaMemcpyAsync(plan->hist_off.p, hoff.data(), sizeof(long long) * (P + 1), cudaMemcpyHostToDevice, s));
  AKM_CK(cudaMemsetAsync(plan->hist.p, 0, sizeof(int) * std::max<long long>(ncells, 1), s));
  AKM_CK(cudaMemsetAsync(plan->err_flag.p, 0, sizeof(int), s));
  const int nf = (int)plan->feat_used.size();
  AKM_CK(launch_scale_and_key(plan->Xc.as<double>(), n, nf, tab, plan->dtab.as<WinTable>(), plan->u_tmp.as<double>(),
                              nullptr, plan->hist.as<int>(), plan->hist_off.as<long long>(), plan->err_flag.as<int>(),
                              plan->n_split, s));
  // S0 on the device (binsort.cu): statistics of every candidate bin edge -> B per window (host, the
  // cost model below) -> bin-major layout, bin starts, work items and the point sort on the device
  const long long total_pts = n * P;
  // spreading items of at most ch_s points: about AKM_CHS_WAVES (default 2) items per SM when the
  // points spread evenly (A/B switch; the clamp below decides at c4 / c5)
  static const int chs_waves = getenv("AKM_CHS_WAVES") ? std::max(1, atoi(getenv("AKM_CHS_WAVES"))) : 2;
  long long ch_s = total_pts / (148LL * chs_waves);
  static const long long chs_max = getenv("AKM_CHS_MAX") ? std::max(32LL, atoll(getenv("AKM_CHS_MAX"))) : 8192LL;
  // 8192: every item costs ~15-25 us of prologue and flush per launch (measured: c4 spreading 7.14 /
  // 7.01 / 6.91 / 6.85 / 6.83 ms at caps 1024 / 2048 / 4096 / 8192 / 16384, x4 7.13 / 6.99 / 6.89 / 6.80 /
  // 6.82), and the larger-first order keeps the tail short
  ch_s = std::max(32LL, std::min(chs_max, ch_s));
  const int ch_i = 128;   // per-cell interpolation items (64 thr x 2 pts, or 8 warps x 16 pts on DMMA)
  const int ch_ib = 128;  // per-bin interpolation items: up to 128 points of one bin
  // item set 0: the square product over all points; set 1: the cross product (spread the class-0
  // sources, interpolate at the class-1 targets; akm_kernel_cross_mvm) -- built only with a split
  const bool split = plan->n_split < n;
  const bool forced = !plan->bin_override.empty();
  static const int kB[kBinCands] = {1, 2, 3, 4, 6, 8};
  BinCandParam cp{};
  long long bc_total = 0;
  for (int k = 0; k < kBinCands; ++k) cp.B[k] = kB[k];
  for (int w = 0; w < P; ++w) {
    const WinGeom& g = tab.w[w];
    const int d = g.d;
    cp.mask[w] = 0;
    for (int k = 0; k < kBinCands; ++k) {
      const int B = kB[k];
      if (forced && B != plan->bin_override[w]) continue;
      const int F = B + 2 * m - 1;
      double Fd = 1;
      for (int t = 0; t < d; ++t) Fd *= F;
      if (Fd > 20000) continue;
      bool fits = true;
      for (int a = 3 - d; a < 3; ++a) fits = fits && ((g.ncell[a] + B - 1) / B) * B + 2 * m - 1 <= n_g;
      {  // both spreading kernels must have a tile for this footprint (enqueue_mvm picks by d)
        int MB_, NB_, WM_, WN_, Mr = 1;
        for (int t = 0; t < d - 1; ++t) Mr *= F;
        fits = fits && spread_mma_choose(Mr, F, F, 1, MB_, NB_, WM_, WN_);
        if (d >= 2) fits = fits && spread_v5_choose(Mr, F, MB_, NB_, WN_);
      }
      if (!fits) continue;
      cp.mask[w] |= 1 << k;
      long long nb = 1;
      for (int a = 3 - d; a < 3; ++a) nb *= (g.ncell[a] + B - 1) / B;
      cp.off[w][k] = bc_total;
      bc_total += nb;
    }
    if (forced && !cp.mask[w])
      return plan->fail(AKM_ERR_UNSUPPORTED, "window %d: forced bin edge %d does not fit the grid box", w,
                        plan->bin_override[w]);
  }
  AKM_CK(plan->bs_bc.ensure(sizeof(int) * std::max<long long>(bc_total, 1)));
  AKM_CK(plan->bs_stats.ensure(sizeof(int) * P * kBinCands * 3));
  AKM_CK(launch_bin_costs(tab, plan->dtab.as<WinTable>(), plan->hist.as<int>(), plan->hist_off.as<long long>(), cp,
                          bc_total, plan->bs_bc.as<int>(), ch_s, plan->bs_stats.as<int>(), s));
  std::vector<int> stats(P * kBinCands * 3);
  int errf = 0;
  AKM_CK(cudaMemcpyAsync(stats.data(), plan->bs_stats.p, sizeof(int) * stats.size(), cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaMemcpyAsync(&errf, plan->err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaStreamSynchronize(s));
  if (errf) return plan->fail(AKM_ERR_CUDA, "internal error: a scaled point fell outside its grid box");
  tm.mark("scale, histogram, B statistics");

  // B per window: cost model in FMA-equivalents per RHS.  Spreading: F^d FMAs per
  // point and RHS, plus one footprint flush of F^d RED.ADD.F64 (~34 FMA-equivalents each,
  // profiles/r01_fp64_peaks.txt) per work item.  2-D windows: the per-item prologue and flush weigh
  // more against the few points of a bin (~140 at c3) -- 60 per footprint tap matches the measured
  // optimum (c3: B = 4 0.724 ms, B = 3 0.771, B = 6 0.833)
  plan->occupied.assign(P, 0);
  plan->maxbin.assign(P, 0);
  long long nbins_total = 0;
  for (int w = 0; w < P; ++w) {
    WinGeom& g = tab.w[w];
    const int d = g.d;
    int bestB = 1, bestK = -1;
    double bestCost = 1e300;
    for (int k = 0; k < kBinCands; ++k) {
      if (!(cp.mask[w] & (1 << k))) continue;
      const int F = kB[k] + 2 * m - 1;
      double Fd = 1;
      for (int t = 0; t < d; ++t) Fd *= F;
      const double chunks_s = (double)stats[(w * kBinCands + k) * 3 + 0];
      const double per_item = (d == 2) ? 60.0 : 34.0;
      const double cost = Fd * ((double)n + per_item * chunks_s);
      if (cost < bestCost * 0.999) {
        bestCost = cost;
        bestB = kB[k];
        bestK = k;
      }
    }
    if (bestK < 0) return plan->fail(AKM_ERR_UNSUPPORTED, "window %d: no bin edge fits the grid box", w);
    plan->occupied[w] = stats[(w * kBinCands + bestK) * 3 + 1];
    plan->maxbin[w] = stats[(w * kBinCands + bestK) * 3 + 2];
    const int B = bestB;
    g.B = B;
    for (int a = 0; a < 3; ++a) {
      if (a < 3 - d) {
        g.nbin[a] = 1; g.F[a] = 1;
        continue;
      }
      g.nbin[a] = (g.ncell[a] + B - 1) / B;
      g.F[a] = B + 2 * m - 1;
      g.L[a] = g.nbin[a] * B + 2 * m - 1;  // covers the last bin's footprint
      if (g.L[a] > n_g)
        return plan->fail(AKM_ERR_UNSUPPORTED,
                          "window %d: grid box of %d nodes exceeds the oversampled grid (n_g = %d); "
                          "increase N or sigma_over, or decrease m", w, g.L[a], n_g);
    }
    g.bt_off = (int)(nbins_total + w);  // per window: start of every bin, then n
    nbins_total += (long long)g.nbin[0] * g.nbin[1] * g.nbin[2];
  }
  // groups of windows with equal (d, F); work items concatenated group by group, larger chunks first
  // inside a group (better tail behaviour); the key and bin spaces are laid out in group order
  plan->groups.clear();
  for (int w = 0; w < P; ++w) {
    const WinGeom& g = tab.w[w];
    const int F = g.F[2];
    Group* grp = nullptr;
    for (auto& gg : plan->groups)
      if (gg.d == g.d && gg.F == F) grp = &gg;
    if (!grp) {
      plan->groups.push_back(Group{});
      grp = &plan->groups.back();
      grp->d = g.d;
      grp->F = F;
    }
    grp->wins.push_back(w);
  }
  const int ngroups = (int)plan->groups.size();
  BinLayout& L = plan->bl;
  long long nkeys = 0, nbins = 0;
  std::vector<long long> gkey(ngroups + 1), gbin(ngroups + 1);
  for (int gi = 0; gi < ngroups; ++gi) {
    gkey[gi] = nkeys;
    gbin[gi] = nbins;
    for (int w : plan->groups[gi].wins) {
      const WinGeom& g = tab.w[w];
      long long bb = 1;
      for (int a = 3 - g.d; a < 3; ++a) bb *= g.B;
      const long long nb = (long long)g.nbin[0] * g.nbin[1] * g.nbin[2];
      L.keybase[w] = nkeys;
      L.binbase[w] = nbins;
      nkeys += nb * 2 * bb;
      nbins += nb;
    }
  }
  gkey[ngroups] = nkeys;
  if (nkeys >= (1LL << 31) - 1)  // (CUB scans take int sizes; keys are 32-bit)
    return plan->fail(AKM_ERR_UNSUPPORTED, "bin layout of %lld slots exceeds 2^31 - 1", nkeys);
  gbin[ngroups] = nbins;
  AKM_CK(cudaMemcpyAsync(plan->dtab.p, &tab, sizeof(WinTable), cudaMemcpyHostToDevice, s));
  // keys: counts, offsets, cursors
  AKM_CK(plan->key_cnt.ensure(sizeof(long long) * std::max<long long>(nkeys, 1)));
  AKM_CK(plan->key_off.ensure(sizeof(long long) * std::max<long long>(nkeys, 1)));
  const long long llen[kItemLists] = {nkeys, split ? nkeys : 0, nbins, nbins, split ? nbins : 0, split ? nbins : 0};
  for (int l = 0; l < kItemLists; ++l) {
    AKM_CK(plan->lcnt[l].ensure(sizeof(int) * std::max<long long>(llen[l], 1)));
    AKM_CK(plan->loff[l].ensure(sizeof(int) * std::max<long long>(llen[l], 1)));
  }
  AKM_CK(cudaMemsetAsync(plan->key_cnt.p, 0, sizeof(long long) * std::max<long long>(nkeys, 1), s));
  AKM_CK(cudaMemsetAsync(plan->lcnt[0].p, 0, sizeof(int) * std::max<long long>(nkeys, 1), s));
  if (split) AKM_CK(cudaMemsetAsync(plan->lcnt[1].p, 0, sizeof(int) * std::max<long long>(nkeys, 1), s));
  AKM_CK(launch_slot_keys(tab, plan->dtab.as<WinTable>(), plan->hist.as<int>(), plan->hist_off.as<long long>(), L,
                          plan->key_cnt.as<long long>(), plan->lcnt[0].as<int>(), split ? plan->lcnt[1].as<int>() : nullptr,
                          ch_i, s));
  AKM_CK(scan_excl_ll(plan->key_cnt.as<long long>(), plan->key_off.as<long long>(), nkeys, &plan->cub_temp,
                      &plan->cub_temp_bytes, s));
  int2* ctab = nullptr;
  if (plan->near_field()) {
    AKM_CK(plan->cell_tab.ensure(sizeof(int2) * std::max<long long>(ncells, 1)));
    ctab = plan->cell_tab.as<int2>();
  }
  if (ctab)
    AKM_CK(launch_slot_cursor(tab, plan->dtab.as<WinTable>(), plan->hist_off.as<long long>(), L,
                              plan->key_cnt.as<long long>(), plan->key_off.as<long long>(), nullptr, ctab, s));
  plan->cell_tab_ok = ctab != nullptr;
  AKM_CK(plan->bin_start.ensure(sizeof(int) * (nbins_total + P)));
  AKM_CK(launch_bin_pass(tab, plan->dtab.as<WinTable>(), L, plan->key_off.as<long long>(), n, ch_s, ch_ib,
                         plan->bin_start.as<int>(), plan->lcnt[2].as<int>(), plan->lcnt[3].as<int>(),
                         split ? plan->lcnt[4].as<int>() : nullptr, split ? plan->lcnt[5].as<int>() : nullptr, s));
  // item offsets per list, then each group's [begin, end)
  ListScanParam lp{};
  lp.nlists = kItemLists;
  for (int l = 0; l < kItemLists; ++l) {
    AKM_CK(scan_excl_int(plan->lcnt[l].as<int>(), plan->loff[l].as<int>(), llen[l], &plan->cub_temp,
                         &plan->cub_temp_bytes, s));
    lp.cnt[l] = plan->lcnt[l].as<int>();
    lp.off[l] = plan->loff[l].as<int>();
    lp.len[l] = llen[l];
    const std::vector<long long>& gb = (l < 2) ? gkey : gbin;
    for (int gi = 0; gi <= ngroups; ++gi) lp.gbeg[l][gi] = llen[l] ? gb[gi] : 0;
  }
  AKM_CK(plan->bounds.ensure(sizeof(int) * kItemLists * 2 * ngroups));
  AKM_CK(launch_group_bounds(lp, ngroups, plan->bounds.as<int>(), s));
  std::vector<int> bounds(kItemLists * 2 * ngroups);
  AKM_CK(cudaMemcpyAsync(bounds.data(), plan->bounds.p, sizeof(int) * bounds.size(), cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaStreamSynchronize(s));
  tm.mark("device layout + item scans");
  // list l of the final item sets: 0 -> items_i[0], 1 -> items_i[1], 2 -> items_s[0], 3 -> items_ib[0],
  // 4 -> items_s[1], 5 -> items_ib[1]
  DevBuf* finals[kItemLists] = {&plan->items_i[0], &plan->items_i[1], &plan->items_s[0],
                                &plan->items_ib[0], &plan->items_s[1], &plan->items_ib[1]};
  const int maxc[kItemLists] = {ch_i, ch_i, (int)ch_s, ch_ib, (int)ch_s, ch_ib};
  long long ltot[kItemLists];
  const int* offs[kItemLists];
  WorkItem* outs[kItemLists];
  for (int l = 0; l < kItemLists; ++l) {
    ltot[l] = ngroups ? bounds[(l * 2 + 1) * ngroups + ngroups - 1] : 0;
    AKM_CK(plan->items_u[l].ensure(sizeof(WorkItem) * std::max<long long>(ltot[l], 1)));
    AKM_CK(finals[l]->ensure(sizeof(WorkItem) * std::max<long long>(ltot[l], 1)));
    offs[l] = plan->loff[l].as<int>();
    outs[l] = llen[l] ? plan->items_u[l].as<WorkItem>() : nullptr;
  }
  AKM_CK(launch_emit_items(tab, plan->dtab.as<WinTable>(), L, plan->key_cnt.as<long long>(),
                           plan->key_off.as<long long>(), n, ch_s, ch_i, ch_ib, offs, outs, s));
  long long lmax = 1;
  for (int l = 0; l < kItemLists; ++l) lmax = std::max(lmax, ltot[l]);
  AKM_CK(plan->sort_keys.ensure(sizeof(unsigned) * 2 * lmax));
  AKM_CK(plan->sort_idx.ensure(sizeof(int) * 2 * lmax));
  WinGroupMap gm{};
  for (int gi = 0; gi < ngroups; ++gi)
    for (int w : plan->groups[gi].wins) gm.group[w] = gi;
  for (int l = 0; l < kItemLists; ++l) {
    if (!ltot[l]) continue;
    AKM_CK(sort_items_larger_first(plan->items_u[l].as<WorkItem>(), ltot[l], maxc[l], gm, ngroups,
                                   plan->sort_keys.as<unsigned>(), plan->sort_keys.as<unsigned>() + lmax,
                                   plan->sort_idx.as<int>(), plan->sort_idx.as<int>() + lmax, &plan->cub_temp,
                                   &plan->cub_temp_bytes, finals[l]->as<WorkItem>(), s));
  }
  for (int set = 0; set < 2; ++set) {
    plan->n_items_spread[set] = (size_t)ltot[set == 0 ? 2 : 4];
    plan->n_items_interp[set] = (size_t)ltot[set == 0 ? 0 : 1];
    plan->n_items_interp_bin[set] = (size_t)ltot[set == 0 ? 3 : 5];
  }
  for (int gi = 0; gi < ngroups; ++gi) {
    Group& grp = plan->groups[gi];
    for (int set = 0; set < 2; ++set) {
      const int ls = set == 0 ? 2 : 4, li = set == 0 ? 0 : 1, lb = set == 0 ? 3 : 5;
      auto beg = [&](int l) { return bounds[(l * 2 + 0) * ngroups + gi]; };
      auto end = [&](int l) { return bounds[(l * 2 + 1) * ngroups + gi]; };
      ItemSlice& sl = grp.sl[set];
      sl.spread_begin = beg(ls);
      sl.spread_count = end(ls) - beg(ls);
      sl.interp_begin = beg(li);
      sl.interp_count = end(li) - beg(li);
      sl.interp_bin_begin = beg(lb);
      sl.interp_bin_count = end(lb) - beg(lb);
      // per-cell DMMA items pay a whole cell footprint per item: with few points per occupied cell
      // the per-bin scalar kernel wins (c3: ~16 points per cell; c4/c5: hundreds)
      const double pts = (double)(set == 0 ? n : n - plan->n_split) * (double)grp.wins.size();
      sl.sparse = sl.interp_count > 0 && pts / (double)sl.interp_count < 48.0;
    }
  }

  // workspace layout (per RHS) for grids, spectra, twiddles and multipliers
  long long tap = 0, a1 = 0, a2 = 0, a3 = 0, cc = 0, c2 = 0, twc = 0, dd = 0;
  for (int w = 0; w < P; ++w) {
    WinGeom& g = tab.w[w];
    g.ntap = (long long)g.L[0] * g.L[1] * g.L[2];
    g.tap_off = tap;
    tap += g.ntap;
    g.pt_off = (long long)w * n;
    const long long s1 = (long long)g.L[0] * g.L[1] * g.K[2];
    const long long s2 = (long long)g.L[0] * g.K[1] * g.K[2];
    const long long s3 = (long long)g.K[0] * g.K[1] * g.K[2];
    g.a1_off = a1; a1 += s1;
    g.a2_off = a2; a2 += s2;
    g.a3_off = a3; a3 += s3;
    g.c_off = cc; cc += 2 * s2;
    g.c2_off = c2; c2 += 2 * s1;
    for (int a = 0; a < 3; ++a) {
      g.tw_off[a] = twc;
      twc += (long long)g.K[a] * g.L[a];
    }
    g.d_off = dd;
    dd += 2 * s3;
  }
  plan->total_taps = tap;
  plan->szA1 = a1; plan->szA2 = a2; plan->szA3 = a3; plan->szC = cc; plan->szC2 = c2; plan->szTW = twc; plan->szD = dd;
  plan->r_cap = 0;  // grid workspace must be re-sized

  // points into bin-major order: stable radix sort by slot key (binsort.cu sort_points)
  AKM_CK(cudaMemcpyAsync(plan->dtab.p, &tab, sizeof(WinTable), cudaMemcpyHostToDevice, s));
  {
    WinGroupMap order{};  // window of each n-point block of the sorted sequence (group order)
    int q = 0;
    for (const Group& grp : plan->groups)
      for (int w : grp.wins) order.group[q++] = w;
    AKM_CK(plan->pt_keys.ensure(sizeof(unsigned) * 2 * std::max<long long>(n * P, 1)));
    AKM_CK(plan->pt_vals.ensure(sizeof(int) * 2 * std::max<long long>(n * P, 1)));
    AKM_CK(sort_points(n, tab, plan->dtab.as<WinTable>(), L, nkeys, order, plan->u_tmp.as<double>(), plan->n_split,
                       plan->pt_keys.as<unsigned>(), plan->pt_keys.as<unsigned>() + n * P, plan->pt_vals.as<int>(),
                       plan->pt_vals.as<int>() + n * P, &plan->cub_temp, &plan->cub_temp_bytes,
                       plan->u_sorted.as<double>(), plan->perm.as<int>(), s));
  }
  // twiddles
  AKM_CK(plan->tw.ensure(sizeof(double2) * std::max<long long>(twc, 1)));
  AKM_CK(launch_twiddles(tab, plan->dtab.as<WinTable>(), plan->tw.as<double2>(), s));
  AKM_CK(plan->D.ensure(sizeof(double) * std::max<long long>(dd, 1)));
  tm.mark("items, point sort, twiddles");
  plan->c_w_binned = plan->c_w;
  return AKM_OK;
}

// b_k of eq. (3.2) for kappa and kappa^der at ell_eff, then the multiplier tables.
static akm_status rebuild_tables(akm_plan* plan, cudaStream_t s) {
  NvtxRange nvtx("akm S1 b_k + multipliers");
  const int N = plan->N;
  long long maxNd = 1;
  for (int w = 0; w < plan->P; ++w) {
    long long v = 1;
    for (int t = 0; t < plan->tab.w[w].d; ++t) v *= N;
    maxNd = std::max(maxNd, v);
  }
  AKM_CK(plan->bs0.ensure(sizeof(double) * maxNd));
  AKM_CK(plan->bs1.ensure(sizeof(double) * maxNd));
  // per-window b_k tables of kappa and kappa^der, kept across set_theta calls: they depend only on
  // (family, d, N, ell_eff, regularisation), and for Gaussian windows the scale rule keeps ell_eff
  // fixed while ell moves (reading R2), so only the multipliers (1/c_w) are rebuilt then
  if (plan->bk_stride != maxNd || plan->bk_keys.size() != (size_t)plan->P) {
    AKM_CK(plan->bk.ensure(sizeof(double) * 2 * maxNd * plan->P));
    plan->bk_stride = maxNd;
    plan->bk_keys.assign(plan->P, akm_plan::BkKey{});
  }
  if (plan->reg_p > 0) AKM_CK(plan->reg_coef.ensure(sizeof(double) * plan->P * 2 * kRegStride));
  if (!plan->deconv_ok) {  // per-axis deconvolution factors: fixed by (N, n_g, m, sigma) at set_points
    AKM_CK(plan->deconv.ensure(sizeof(double) * 3 * (N + 1)));
    AKM_CK(launch_deconv_table(N, plan->n_g, plan->m, plan->sigma_over, plan->deconv.as<double>(), s));
    plan->deconv_ok = true;
  }
  for (int w = 0; w < plan->P; ++w) {
    const int d = plan->tab.w[w].d;
    const double ell_eff = plan->ell / plan->c_w[w];
    double* bK = plan->bk.as<double>() + (long long)w * 2 * maxNd;
    double* bL = bK + maxNd;
    const akm_plan::BkKey key{true, plan->family, d, N, plan->reg_p, ell_eff, plan->reg_eps_I, plan->eps_B};
    if (!(plan->bk_keys[w] == key)) {
      double* bufs[2] = {bK, bL};
      double* coef = plan->reg_p > 0 ? plan->reg_coef.as<double>() + (long long)w * 2 * kRegStride : nullptr;
      if (coef) {
        AKM_CK(cudaMemsetAsync(coef, 0, sizeof(double) * 2 * kRegStride, s));
        AKM_CK(launch_reg_coef(plan->family, ell_eff, plan->reg_eps_I, plan->eps_B, plan->reg_p, coef, s));
      }
      for (int deriv = 0; deriv < 2; ++deriv) {
        double* a = plan->bs0.as<double>();
        double* b = plan->bs1.as<double>();
        if (coef)
          AKM_CK(launch_kernel_samples_reg(plan->family, d, N, ell_eff, deriv, plan->reg_eps_I, plan->eps_B,
                                           plan->reg_p, coef, a, s));
        else
          AKM_CK(launch_kernel_samples(plan->family, d, N, ell_eff, deriv, a, s));
        for (int t = 0; t < d; ++t) {
          double* out = (t == d - 1) ? bufs[deriv] : b;
          AKM_CK(launch_cos_dft_axis(d, N, t, a, out, s));
          std::swap(a, b);  // after the swap, `a` holds the latest result
        }
      }
      plan->bk_keys[w] = key;
    }
    AKM_CK(launch_multiplier(plan->tab, plan->dtab.as<WinTable>(), w, bK, bL, 3, 1.0 / plan->c_w[w],
                             plan->deconv.as<double>(), plan->D.as<double>(), s));
  }
  return AKM_OK;
}

static akm_status ensure_rhs_workspace(akm_plan* plan, int r) {
  if (r <= plan->r_cap) return AKM_OK;
  ++plan->epoch;
  const long long R = r;
  AKM_CK(plan->grid.ensure(sizeof(double) * std::max<long long>(plan->total_taps * R, 1)));
  AKM_CK(plan->H.ensure(sizeof(double) * std::max<long long>(plan->total_taps * 2 * R, 1)));
  AKM_CK(plan->A1.ensure(sizeof(double2) * std::max<long long>(plan->szA1 * R, 1)));
  AKM_CK(plan->A2.ensure(sizeof(double2) * std::max<long long>(plan->szA2 * R, 1)));
  AKM_CK(plan->A3.ensure(sizeof(double2) * std::max<long long>(plan->szA3 * R, 1)));
  AKM_CK(plan->C.ensure(sizeof(double2) * std::max<long long>(plan->szC * R, 1)));
  AKM_CK(plan->C2.ensure(sizeof(double2) * std::max<long long>(plan->szC2 * R, 1)));
  AKM_CK(plan->part.ensure(sizeof(double) * std::max<long long>(plan->P * plan->n * 2 * R, 1)));
  if (plan->near_field()) AKM_CK(plan->nfV.ensure(sizeof(double) * std::max<long long>(plan->P * plan->n * R, 1)));
  if (plan->det) {  // deterministic spreading: integer limbs of the grids, per-column scales (spread_det.cu)
    AKM_CK(plan->det_limbs.ensure(sizeof(unsigned long long) * 3 * std::max<long long>(plan->total_taps * R, 1)));
    AKM_CK(plan->det_colmax.ensure(sizeof(unsigned long long) * R));
    AKM_CK(plan->det_S.ensure(sizeof(int) * plan->P * R));
  }
  plan->r_cap = r;
  return AKM_OK;
}

// choose the spread register tile for a (M = F^{d-1}) x (Nn = F*rc) footprint matrix
static bool choose_spread_tile(int M, int Nn, int& MT, int& NT, int& threads) {
  static const int cand[][2] = {{2, 8}, {2, 16}, {4, 4}, {4, 6}, {4, 8}, {4, 11}, {4, 12}, {4, 16},
                                {8, 4}, {8, 6}, {8, 8}, {8, 11}, {8, 12}};
  double best = 1e300;
  bool found = false;
  for (auto& c : cand) {
    const int mt = c[0], nt = c[1];
    const int TM = (M + mt - 1) / mt, TN = (Nn + nt - 1) / nt;
    const int thr = TM * TN;
    if (thr > 256) continue;  // k_spread is compiled with __launch_bounds__(256)
    const double waste = (double)TM * mt * TN * nt / ((double)M * Nn);
    const double ldratio = (double)(mt + nt) / (mt * nt);
    double score = waste * (1.0 + 1.5 * ldratio);
    if (thr < 64) score *= 1.25;
    if (score < best) {
      best = score;
      MT = mt;
      NT = nt;
      threads = ((thr + 31) / 32) * 32;
      found = true;
    }
  }
  return found;
}

// ================================================================== the MVM
// set 0: the square products over all n points (Y: n x r).  set 1: the cross product (Y: the
// (n - n_split) x r target rows; V holds the n_split source rows; only Y = K_{*X} V).
// The product is split at the grids: enqueue_spread (S2: zero + adjoint NFFT of the plan's points
// into `grid`, total_taps x r doubles) and enqueue_finish (S3-S7 from a complete grid).  The
// single-GPU product runs both on the plan's own grid; the point-sharded product (akm_spread_grid /
// akm_mvm_from_grid) sums the ranks' grids in between.
static akm_status enqueue_spread(akm_plan* plan, const double* V, long long ldv, int r, double* grid, cudaStream_t s,
                                 int set) {
  NvtxRange nvtx("akm S2 spread");
  const long long n = plan->n;
  const WinTable* dtab = plan->dtab.as<WinTable>();
  if (n == 0 || !plan->det) AKM_CK(launch_zero(grid, plan->total_taps * r, s));
  if (n == 0) return AKM_OK;
  DetAcc da{};
  if (plan->det) {  // integer-limb accumulation, converted into `grid` after the launches
    const long long rows = (set == 1) ? plan->n_split : n;  // the cross product's V holds the sources only
    da.limbs = plan->det_limbs.as<unsigned long long>();
    da.S = plan->det_S.as<int>();
    da.stride = plan->total_taps * r;
    // W^d_w bound of a contribution's window product: W = max over taps of sum_k |c_k| >= max |tap|
    double W = 1.0;
    for (int q = 0; q < 2 * plan->m; ++q) {
      double sum = 0.0;
      for (int k = 0; k < kPolyLen; ++k) sum += std::fabs(plan->poly_param.c[q * kPolyLen + k]);
      W = std::max(W, sum);
    }
    DetWin& dw = plan->det_win;
    dw.P = plan->P;
    for (int w = 0; w < plan->P; ++w) {
      dw.wbits[w] = (int)std::ceil(plan->tab.w[w].d * std::log2(W)) + 1;
      dw.tap_off[w] = plan->tab.w[w].tap_off;
    }
    dw.tap_off[plan->P] = plan->total_taps;
    da.r_total = r;
    AKM_CK(launch_det_prepare(V, ldv, rows, r, dw, plan->det_colmax.as<unsigned long long>(),
                              plan->det_S.as<int>(), da.limbs, da.stride, s));
  }
  for (const Group& grp : plan->groups) {
    const int F = grp.F, d = grp.d;
    int M = 1;
    for (int t = 0; t < d - 1; ++t) M *= F;
    int r0 = 0;
    // 2-D groups: strips (spread_strip.cu); 3-D: spread_v5.cu; k_spread_mma for 1-D
    // windows; AKM_SPREAD_V5=0/1 forces either kernel (A/B measurement)
    static const int v5_env = getenv("AKM_SPREAD_V5") ? atoi(getenv("AKM_SPREAD_V5")) : -1;
    const bool v5 = v5_env >= 0 ? v5_env != 0 : d >= 2;
    while (v5 && r0 < r) {
      // 2-D windows: strips of 1 x B cells as their own GEMMs (spread_strip.cu), when a tile exists
      if (d == 2 && spread_strip_nb(d, 2 * plan->m, F, 1) > 0) {
        static const int ss_rcmax = getenv("AKM_SS_RCMAX") ? std::max(1, atoi(getenv("AKM_SS_RCMAX"))) : 12;
        int rc = std::min(ss_rcmax, r - r0);
        while (rc > 1 && spread_strip_nb(d, 2 * plan->m, F, rc) == 0) --rc;
        if (rc < r - r0 && rc > (r - r0 + 1) / 2) rc = (r - r0 + 1) / 2;
        const int nb = spread_strip_nb(d, 2 * plan->m, F, rc);
        AKM_CK(launch_spread_strip(dtab, plan->poly_param,
                                   plan->items_s[set].as<WorkItem>() + grp.sl[set].spread_begin,
                                   grp.sl[set].spread_count, plan->u_sorted.as<double>(), plan->perm.as<int>(), V, ldv,
                                   n, r0, rc, r, grid, 2 * plan->m, F, nb, s, da));
        if (grp.sl[set].spread_count > 0) {
          ++plan->launches;
          ++plan->spread_launches;
        }
        r0 += rc;
        continue;
      }
      int rc = std::min(12, r - r0), MB = 0, NB = 0, WN = 0;
      while (rc > 1 && !(spread_v5_choose(M, F * rc, MB, NB, WN) && spread_v5_smem(F, rc, MB, NB, WN) <= 220 * 1024)) --rc;
      if (rc < r - r0 && rc > (r - r0 + 1) / 2) rc = (r - r0 + 1) / 2;
      if (!spread_v5_choose(M, F * rc, MB, NB, WN))
        return plan->fail(AKM_ERR_UNSUPPORTED, "no spread tile for footprint %d x %d", M, F * rc);
      AKM_CK(launch_spread_v5(dtab, plan->poly_param, plan->items_s[set].as<WorkItem>() + grp.sl[set].spread_begin,
                              grp.sl[set].spread_count, plan->u_sorted.as<double>(), plan->perm.as<int>(), V, ldv, n, r0, rc,
                              r, grid, MB, NB, WN, spread_v5_smem(F, rc, MB, NB, WN), s, da));
      if (grp.sl[set].spread_count > 0) {
        ++plan->launches;
        ++plan->spread_launches;
      }
      r0 += rc;
    }
    while (r0 < r) {
      // largest RHS chunk (<= 12) whose footprint accumulator fits the 8 warps' DMMA tiles and whose
      // panels fit shared memory; split the rest evenly
      int rc = std::min(12, r - r0), MB = 0, NB = 0, WM = 0, WN = 0;
      while (rc > 1 && !spread_mma_choose(M, F * rc, F, rc, MB, NB, WM, WN)) --rc;
      if (rc < r - r0 && rc > (r - r0 + 1) / 2) rc = (r - r0 + 1) / 2;  // balanced chunks (e.g. 6 + 5)
      if (!spread_mma_choose(M, F * rc, F, rc, MB, NB, WM, WN))
        return plan->fail(AKM_ERR_UNSUPPORTED, "no spread tile for footprint %d x %d", M, F * rc);
      const int PB = 0;  // fixed inside the kernel (kSpreadPB)
      const size_t smem = spread_mma_smem(PB, M, F * rc, F, rc);
      AKM_CK(launch_spread_mma(dtab, plan->poly_param, plan->items_s[set].as<WorkItem>() + grp.sl[set].spread_begin, grp.sl[set].spread_count,
                               plan->u_sorted.as<double>(), plan->perm.as<int>(), V, ldv, n, r0, rc, r,
                               grid, MB, NB, WM, WN, PB, smem, s, da));
      if (grp.sl[set].spread_count > 0) {
        ++plan->launches;
        ++plan->spread_launches;
      }
      r0 += rc;
    }
  }
  if (da.limbs) AKM_CK(launch_det_finish(da.limbs, da.S, da.stride, r, plan->det_win, grid, s));
  return AKM_OK;
}

static akm_status enqueue_finish(akm_plan* plan, const double* grid, const double* V, long long ldv, int r, double* Y,
                                 double* dYl, double* dYsf, long long ldy, cudaStream_t s, int set,
                                 akm_plan::EvSet* ev) {
  NvtxRange nvtx("akm S3-S7 DFT, multiply, interpolate, epilogue");
  const bool needK = (Y != nullptr) || (dYsf != nullptr);
  const bool needL = dYl != nullptr;
  const int ops = (needK ? 1 : 0) + (needL ? 1 : 0);
  const int slotK = needK ? 0 : -1;
  const int slotL = needL ? (needK ? 1 : 0) : -1;
  const int dslot0 = needK ? 0 : 1;
  const long long n = plan->n;
  const WinTable* dtab = plan->dtab.as<WinTable>();
  if (ev) AKM_CK(cudaEventRecord(ev->e[5], s));
  // S3-S5: DFT, multiply, inverse DFT
  AKM_CK(launch_fft_forward(plan->tab, dtab, grid, plan->A1.as<double2>(), plan->A2.as<double2>(),
                            plan->tw.as<double2>(), r, s));
  AKM_CK(launch_fft_multiply_inverse(plan->tab, dtab, plan->A2.as<double2>(), plan->A3.as<double2>(),
                                     plan->C.as<double2>(), plan->C2.as<double2>(), plan->tw.as<double2>(),
                                     plan->D.as<double>(), ops, dslot0, r, plan->H.as<double>(), s));
  plan->launches += fft_launch_count(plan->tab, r);
  if (ev) AKM_CK(cudaEventRecord(ev->e[2], s));
  if (n == 0) {
    if (ev) AKM_CK(cudaEventRecord(ev->e[3], s));
    if (ev) AKM_CK(cudaEventRecord(ev->e[4], s));
    return AKM_OK;
  }
  // S6: interpolation
  int r0 = 0;
  while (r0 < r) {
    const int rc = interp_rc_for(r - r0);
    for (const Group& grp : plan->groups) {
      // small launches (fewer than 2 x 148 per-bin items, c1): one warp per point (interp_pt.cu)
      if (interp_pt_choose(grp.d, 2 * plan->m, ops, rc, grp.sl[set].interp_bin_count)) {
        AKM_CK(launch_interp_pt(dtab, plan->poly_param,
                                plan->items_ib[set].as<WorkItem>() + grp.sl[set].interp_bin_begin,
                                grp.sl[set].interp_bin_count, plan->u_sorted.as<double>(), plan->perm.as<int>(),
                                plan->H.as<double>(), grp.d, 2 * plan->m, ops, r, r0, rc, plan->part.as<double>(), n,
                                s));
        ++plan->launches;
        ++plan->interp_launches;
        continue;
      }
      // 2-D windows: per-bin strips of 1 x B cells as DMMA GEMMs (interp_strip.cu)
      if (interp_strip_supported(grp.d, 2 * plan->m, grp.F, ops, rc)) {
        AKM_CK(launch_interp_strip(dtab, plan->poly_param,
                                   plan->items_ib[set].as<WorkItem>() + grp.sl[set].interp_bin_begin,
                                   grp.sl[set].interp_bin_count, plan->u_sorted.as<double>(), plan->perm.as<int>(),
                                   plan->H.as<double>(), 2 * plan->m, grp.F, ops, r, r0, rc, plan->part.as<double>(),
                                   n, s));
        if (grp.sl[set].interp_bin_count > 0) {
          ++plan->launches;
          ++plan->interp_launches;
        }
        continue;
      }
      // 3-D windows: per-bin GEMM over the footprint rows (o0, o1), N = (o2, v) (interp_t.cu);
      // AKM_INTERP_T=0 selects the per-plane kernel (A/B measurement)
      static const bool it_off = getenv("AKM_INTERP_T") && atoi(getenv("AKM_INTERP_T")) == 0;
      // with bins of B = 2 cells the per-cell items (points of one cell are consecutive inside the
      // bin) give an exact 2m footprint: no padded taps and more, shorter CTAs (c2: 57 -> 48 us)
      const int taps = 2 * plan->m;
      if (!it_off && grp.F == taps + 1 && interp_t_supported(grp.d, taps, taps, ops, rc)) {
        AKM_CK(launch_interp_t(dtab, plan->poly_param, plan->items_i[set].as<WorkItem>() + grp.sl[set].interp_begin,
                               grp.sl[set].interp_count, plan->u_sorted.as<double>(), plan->perm.as<int>(),
                               plan->H.as<double>(), taps, taps, ops, r, r0, rc, plan->part.as<double>(), n, s, 1));
        if (grp.sl[set].interp_count > 0) {
          ++plan->launches;
          ++plan->interp_launches;
        }
        continue;
      }
      if (!it_off && interp_t_supported(grp.d, 2 * plan->m, grp.F, ops, rc)) {
        AKM_CK(launch_interp_t(dtab, plan->poly_param, plan->items_ib[set].as<WorkItem>() + grp.sl[set].interp_bin_begin,
                               grp.sl[set].interp_bin_count, plan->u_sorted.as<double>(), plan->perm.as<int>(),
                               plan->H.as<double>(), 2 * plan->m, grp.F, ops, r, r0, rc, plan->part.as<double>(), n,
                               s, grp.F - 2 * plan->m + 1));
        if (grp.sl[set].interp_bin_count > 0) {
          ++plan->launches;
          ++plan->interp_launches;
        }
        continue;
      }
      const bool tma = rc == r && r0 == 0 &&
                       interp_tma_build(plan->tab, plan->H.as<double>(), ops, r, plan->tma_maps.data());
      AKM_CK(launch_interp(dtab, plan->items_i[set].as<WorkItem>() + grp.sl[set].interp_begin, grp.sl[set].interp_count,
                           plan->items_ib[set].as<WorkItem>() + grp.sl[set].interp_bin_begin, grp.sl[set].interp_bin_count,
                           grp.d >= 2 ? grp.F : 1, grp.F, grp.sl[set].sparse, plan->u_sorted.as<double>(), plan->perm.as<int>(),
                           plan->H.as<double>(), grp.d,
                           2 * plan->m, ops, r, r0, rc, plan->part.as<double>(), n,
                           tma ? plan->tma_maps.data() : nullptr, s));
      if (grp.sl[set].interp_count > 0) {
        ++plan->launches;
        ++plan->interp_launches;
      }
    }
    r0 += rc;
  }
  if (plan->near_field()) {  // kappa_R's inner part: add sum_j (kappa - T_I)(r_ij) v_j (regularize.cu)
    if (set != 0) return plan->fail(AKM_ERR_UNSUPPORTED, "the near-field correction is built for the square products only");
    if (!plan->cell_tab_ok) return plan->fail(AKM_ERR_STATE, "internal error: near-field cell table not built");
    const int nitems = (int)plan->n_items_interp_bin[0];
    AKM_CK(launch_near_field(dtab, plan->items_ib[0].as<WorkItem>(), nitems, plan->cell_tab.as<int2>(),
                             plan->hist_off.as<long long>(), plan->u_sorted.as<double>(), plan->perm.as<int>(), V, ldv,
                             plan->nfV.as<double>(), n, plan->P, r, ops, slotK, slotL, plan->family, plan->ell,
                             plan->reg_eps_I, plan->reg_p, plan->reg_coef.as<double>(), plan->part.as<double>(), s));
    if (nitems > 0) plan->launches += near_field_launches(r);
  }
  if (ev) AKM_CK(cudaEventRecord(ev->e[3], s));
  // S7: epilogue
  if (set == 0) {
    AKM_CK(launch_epilogue(n, plan->P, r, ops, plan->part.as<double>(), V, ldv, plan->sigma_f, plan->sigma_eps, Y, dYl,
                           dYsf, ldy, slotK, slotL, s));
  } else {
    AKM_CK(launch_epilogue_cross(n, plan->n_split, plan->P, r, ops, slotK, plan->part.as<double>(), plan->sigma_f, Y,
                                 ldy, s));
  }
  ++plan->launches;
  if (ev) AKM_CK(cudaEventRecord(ev->e[4], s));
  return AKM_OK;
}

static akm_status enqueue_mvm(akm_plan* plan, const double* V, long long ldv, int r, double* Y, double* dYl,
                              double* dYsf, long long ldy, cudaStream_t s, int set = 0) {
  if (plan->n == 0) return AKM_OK;
  akm_status st = ensure_rhs_workspace(plan, r);
  if (st != AKM_OK) return st;
  akm_plan::EvSet* ev = plan->profiling ? plan->next_set() : nullptr;
  if (ev) AKM_CK(cudaEventRecord(ev->e[0], s));
  st = enqueue_spread(plan, V, ldv, r, plan->grid.as<double>(), s, set);
  if (st != AKM_OK) return st;
  if (ev) AKM_CK(cudaEventRecord(ev->e[1], s));
  return enqueue_finish(plan, plan->grid.as<double>(), V, ldv, r, Y, dYl, dYsf, ldy, s, set, ev);
}

// The MVM launch sequence (a memset and ~9 kernels) is captured once into a CUDA graph and
// replayed while the buffers, items and theta stay the same: the small configurations are
// launch-latency bound.  The legacy default stream cannot be captured; calls on it run the graph
// on a plan-owned stream ordered by two events.  Profiling (stage events) uses direct launches.
static akm_status run_mvm(akm_plan* plan, const double* V, long long ldv, int r, double* Y, double* dYl,
                          double* dYsf, long long ldy, cudaStream_t s, int set = 0) {
  if (plan->n == 0) return AKM_OK;
  if (plan->profiling || !plan->use_graphs) return enqueue_mvm(plan, V, ldv, r, Y, dYl, dYsf, ldy, s, set);
  akm_status st = ensure_rhs_workspace(plan, r);
  if (st != AKM_OK) return st;
  const akm_plan::GraphKey key{V, Y, dYl, dYsf, ldv, ldy, r, plan->epoch, set};
  cudaStream_t cs = s;
  if (s == nullptr || s == cudaStreamLegacy) {
    if (!plan->own_stream) {
      AKM_CK(cudaStreamCreateWithFlags(&plan->own_stream, cudaStreamNonBlocking));
      AKM_CK(cudaEventCreateWithFlags(&plan->ev_in, cudaEventDisableTiming));
      AKM_CK(cudaEventCreateWithFlags(&plan->ev_out, cudaEventDisableTiming));
    }
    cs = plan->own_stream;
    AKM_CK(cudaEventRecord(plan->ev_in, s));
    AKM_CK(cudaStreamWaitEvent(cs, plan->ev_in, 0));
  }
  akm_plan::GraphEntry* ge = nullptr;
  for (auto& g : plan->graphs)
    if (g.exec && g.key == key) ge = &g;
  if (!ge) {
    ge = &plan->graphs[0];  // least recently used slot (empty slots have last_use 0)
    for (auto& g : plan->graphs)
      if (!g.exec || g.last_use < ge->last_use) {
        ge = &g;
        if (!g.exec) break;
      }
    if (ge->exec) {
      cudaGraphExecDestroy(ge->exec);
      ge->exec = nullptr;
    }
    const long long l0 = plan->launches, s0 = plan->spread_launches, i0 = plan->interp_launches;
    cudaGraph_t graph = nullptr;
    AKM_CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    st = enqueue_mvm(plan, V, ldv, r, Y, dYl, dYsf, ldy, cs, set);
    cudaError_t ec = cudaStreamEndCapture(cs, &graph);
    if (st != AKM_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    AKM_CK(ec);
    cudaError_t ei = cudaGraphInstantiate(&ge->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) ge->exec = nullptr;
    AKM_CK(ei);
    ge->key = key;
    ge->launches = plan->launches - l0;
    ge->spread = plan->spread_launches - s0;
    ge->interp = plan->interp_launches - i0;
    plan->launches = l0;  // counted again below, once per replay
    plan->spread_launches = s0;
    plan->interp_launches = i0;
  }
  ge->last_use = ++plan->graph_clock;
  AKM_CK(cudaGraphLaunch(ge->exec, cs));
  plan->launches += ge->launches;
  plan->spread_launches += ge->spread;
  plan->interp_launches += ge->interp;
  if (cs != s) {
    AKM_CK(cudaEventRecord(plan->ev_out, cs));
    AKM_CK(cudaStreamWaitEvent(s, plan->ev_out, 0));
  }
  return AKM_OK;
}

// host/device staging around run_mvm
static akm_status mvm_entry(akm_plan* plan, const double* V, long long ldv, int r, double* Y, double* dYl,
                            double* dYsf, double* dYse, long long ldy, cudaStream_t s) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points || !plan->have_theta)
    return plan->fail(AKM_ERR_STATE, "kernel_mvm called before set_points and set_theta");
  if (r < 1 || ldv < r || ldy < r) return plan->fail(AKM_ERR_INVALID_ARG, "bad r/ldv/ldy (r=%d ldv=%lld ldy=%lld)", r, ldv, ldy);
  if (!Y && !dYl && !dYsf && !dYse) return plan->fail(AKM_ERR_INVALID_ARG, "no output requested");
  const long long n = plan->n;
  if (n > 0 && !V) return plan->fail(AKM_ERR_INVALID_ARG, "V is NULL");
  AKM_CK(cudaSetDevice(plan->device));
  if (n == 0) return AKM_OK;
  const bool v_dev = is_device_ptr(V);
  double* outs[4] = {Y, dYl, dYsf, dYse};
  bool out_dev[4];
  bool any_host = !v_dev;
  for (int k = 0; k < 4; ++k) {
    out_dev[k] = outs[k] ? is_device_ptr(outs[k]) : true;
    any_host = any_host || !out_dev[k];
  }
  const double* Vd = V;
  long long ldvd = ldv;
  if (!v_dev) {
    AKM_CK(plan->stageV.ensure(sizeof(double) * n * r));
    AKM_CK(copy_rows(plan->stageV.p, sizeof(double) * r, V, sizeof(double) * ldv, sizeof(double) * r, n,
                             cudaMemcpyHostToDevice, s));
    Vd = plan->stageV.as<double>();
    ldvd = r;
  }
  DevBuf* stages[4] = {&plan->stageY, &plan->stageL, &plan->stageS, nullptr};
  double* od[4];
  long long ldyd = ldy;
  bool staged = false;
  for (int k = 0; k < 4; ++k) {
    od[k] = outs[k];
    if (outs[k] && !out_dev[k]) staged = true;
  }
  if (staged) {
    // stage every output (one leading dimension for all)
    ldyd = r;
    for (int k = 0; k < 4; ++k) {
      if (!outs[k]) continue;
      DevBuf* b = stages[k] ? stages[k] : &plan->bs0;
      if (k == 3) {
        AKM_CK(plan->bs0.ensure(sizeof(double) * n * r));  // reuse (tables are already built)
        b = &plan->bs0;
      }
      AKM_CK(b->ensure(sizeof(double) * n * r));
      od[k] = b->as<double>();
    }
  }
  if (od[0] || od[1] || od[2]) {
    akm_status st = run_mvm(plan, Vd, ldvd, r, od[0], od[1], od[2], ldyd, s);
    if (st != AKM_OK) return st;
  }
  if (od[3]) {
    AKM_CK(launch_scaled_copy(n, r, 2.0 * plan->sigma_eps, Vd, ldvd, od[3], ldyd, s));
    ++plan->launches;
  }
  if (staged) {
    for (int k = 0; k < 4; ++k) {
      if (!outs[k]) continue;
      AKM_CK(copy_rows(outs[k], sizeof(double) * ldy, od[k], sizeof(double) * r, sizeof(double) * r, n,
                               out_dev[k] ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    }
  }
  if (any_host) AKM_CK(cudaStreamSynchronize(s));
  return AKM_OK;
}

// Streaming host batches (include/akm.h akm_kernel_mvm_pipelined): copy-in | product | copy-out on
// three streams over two device slots, so batch k's outputs go back while batch k+1 is computed.
akm_status akm_kernel_mvm_pipelined(akm_plan* plan, const double* V, int64_t ldv, int32_t r, double* Y,
                                    double* dY_ell, double* dY_sf, int64_t ldy, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points || !plan->have_theta)
    return plan->fail(AKM_ERR_STATE, "kernel_mvm_pipelined called before set_points and set_theta");
  if (r < 1 || ldv < r || ldy < r) return plan->fail(AKM_ERR_INVALID_ARG, "bad r/ldv/ldy (r=%d ldv=%lld ldy=%lld)", r, (long long)ldv, (long long)ldy);
  double* outs[3] = {Y, dY_ell, dY_sf};
  if (!Y && !dY_ell && !dY_sf) return plan->fail(AKM_ERR_INVALID_ARG, "no output requested");
  const long long n = plan->n;
  AKM_CK(cudaSetDevice(plan->device));
  if (n == 0) return AKM_OK;
  if (!V || !is_pinned_host(V)) return plan->fail(AKM_ERR_INVALID_ARG, "kernel_mvm_pipelined: V must be pinned host memory");
  for (int k = 0; k < 3; ++k)
    if (outs[k] && !is_pinned_host(outs[k]))
      return plan->fail(AKM_ERR_INVALID_ARG, "kernel_mvm_pipelined: outputs must be pinned host memory");
  auto& P = plan->pipe;
  const cudaStream_t s = S(stream);
  if (!P.cin) {
    AKM_CK(cudaStreamCreateWithFlags(&P.cin, cudaStreamNonBlocking));
    AKM_CK(cudaStreamCreateWithFlags(&P.cout, cudaStreamNonBlocking));
    for (int j = 0; j < 2; ++j) {
      AKM_CK(cudaEventCreateWithFlags(&P.in_done[j], cudaEventDisableTiming));
      AKM_CK(cudaEventCreateWithFlags(&P.comp_done[j], cudaEventDisableTiming));
      AKM_CK(cudaEventCreateWithFlags(&P.out_done[j], cudaEventDisableTiming));
    }
  }
  const int j = P.next;
  const size_t blk = sizeof(double) * (size_t)n * r;
  bool grow = P.V[j].bytes < blk;
  for (int k = 0; k < 3; ++k) grow = grow || (outs[k] && P.O[j][k].bytes < blk);
  if (grow) {  // a slot in flight is never freed under its copies or product
    AKM_CK(cudaStreamSynchronize(P.cin));
    AKM_CK(cudaStreamSynchronize(P.cout));
    AKM_CK(cudaStreamSynchronize(s));
    AKM_CK(P.V[j].ensure(blk));
    for (int k = 0; k < 3; ++k)
      if (outs[k]) AKM_CK(P.O[j][k].ensure(blk));
  }
  double* Vd = P.V[j].as<double>();
  double* od[3];
  for (int k = 0; k < 3; ++k) od[k] = outs[k] ? P.O[j][k].as<double>() : nullptr;
  // small batches (< 4 MiB of V: copies of a few microseconds) keep the copies on the caller's
  // stream: the cross-stream event handshakes cost more than the overlap hides (c1 / c2 measured
  // 10% / 1% slower through the copy streams); the host still does not block
  const char* split_env = std::getenv("AKM_PIPE_SPLIT_MIN_BYTES");  // tests force either mode
  const bool split = blk >= (split_env ? (size_t)std::atoll(split_env) : (size_t)4 << 20);
  const cudaStream_t cin = split ? P.cin : s, cout = split ? P.cout : s;
  // copy-in: slot j is free once the product two calls back has read it
  if (split && P.live[j]) AKM_CK(cudaStreamWaitEvent(cin, P.comp_done[j], 0));
  AKM_CK(copy_rows(Vd, sizeof(double) * r, V, sizeof(double) * ldv, sizeof(double) * r, n, cudaMemcpyHostToDevice, cin));
  // product on the caller's stream (after its earlier work: the plan's workspaces stay ordered)
  if (split) {
    AKM_CK(cudaEventRecord(P.in_done[j], cin));
    AKM_CK(cudaStreamWaitEvent(s, P.in_done[j], 0));
  }
  // O[j] is free once the copy-out two calls back has read it (a no-op when that ran on s)
  if (P.live[j]) AKM_CK(cudaStreamWaitEvent(s, P.out_done[j], 0));
  akm_status st = run_mvm(plan, Vd, r, r, od[0], od[1], od[2], r, s);
  if (st != AKM_OK) return st;
  AKM_CK(cudaEventRecord(P.comp_done[j], s));
  // copy-out
  if (split) AKM_CK(cudaStreamWaitEvent(cout, P.comp_done[j], 0));
  for (int k = 0; k < 3; ++k)
    if (outs[k])
      AKM_CK(copy_rows(outs[k], sizeof(double) * ldy, od[k], sizeof(double) * r, sizeof(double) * r, n,
                       cudaMemcpyDeviceToHost, cout));
  AKM_CK(cudaEventRecord(P.out_done[j], cout));
  P.live[j] = true;
  P.last = j;
  P.next = j ^ 1;
  return AKM_OK;
}

akm_status akm_pipeline_wait(akm_plan* plan, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (plan->pipe.last < 0) return AKM_OK;
  AKM_CK(cudaSetDevice(plan->device));
  // each slot's last copy-out follows every earlier use of that slot (the product of a call waits for
  // the copy-out two calls back), and each copy-out follows its product and copy-in
  for (int j = 0; j < 2; ++j)
    if (plan->pipe.live[j]) AKM_CK(cudaStreamWaitEvent(S(stream), plan->pipe.out_done[j], 0));
  return AKM_OK;
}

// ================================================================== AAFN (aafn.cu)
// Landmarks: FPS per window (k = min(kpw, n) picks each), merged in window order without duplicates.
static akm_status aafn_landmarks(akm_plan* plan, cudaStream_t s) {
  auto& A = plan->aafn;
  const long long n = plan->n;
  const int P = plan->P, nf = (int)plan->feat_used.size();
  const int kw = (int)std::min<long long>(A.kpw, n);
  AKM_CK(A.picks.ensure(sizeof(int) * P * kw));
  AKM_CK(A.dmin.ensure(sizeof(double) * n));
  AKM_CK(A.fps_scratch.ensure(fps_scratch_bytes()));
  for (int w = 0; w < P; ++w) {
    const WinGeom& g = plan->tab.w[w];
    int cols[3] = {0, 0, 0};
    for (int t = 0; t < g.d; ++t) cols[t] = g.feat[3 - g.d + t];
    AKM_CK(launch_fps(plan->Xc.as<double>(), n, nf, cols, g.d, kw, A.picks.as<int>() + (long long)w * kw,
                      A.dmin.as<double>(), A.fps_scratch.p, s));
  }
  std::vector<int> picks((size_t)P * kw);
  AKM_CK(cudaMemcpyAsync(picks.data(), A.picks.p, sizeof(int) * picks.size(), cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaStreamSynchronize(s));
  std::vector<int> lm;
  std::set<int> seen;
  for (int v : picks)
    if (seen.insert(v).second) lm.push_back(v);
  A.k = (int)lm.size();
  AKM_CK(A.lm.ensure(sizeof(int) * A.k));
  AKM_CK(A.lmpos.ensure(sizeof(int) * n));
  AKM_CK(cudaMemcpyAsync(A.lm.p, lm.data(), sizeof(int) * A.k, cudaMemcpyHostToDevice, s));
  AKM_CK(launch_lmpos(n, A.k, A.lm.as<int>(), A.lmpos.as<int>(), s));
  AKM_CK(cudaStreamSynchronize(s));
  A.lm_ready = true;
  return AKM_OK;
}

// Factors for the current theta: L11 (Cholesky of the landmark block, one jitter retry as in SPEC's
// DESIGN DECISIONS), L11^{-1}, Phi = K21 L11^{-T}, G = diag(S_aa^{-1/2}), log det M.
static akm_status aafn_build(akm_plan* plan, int R, cudaStream_t s) {
  NvtxRange nvtx("akm AAFN build");
  auto& A = plan->aafn;
  if (!A.lm_ready) {
    akm_status st = aafn_landmarks(plan, s);
    if (st != AKM_OK) return st;
  }
  const long long n = plan->n;
  const int k = A.k;
  AKM_CK(A.y1.ensure(sizeof(double) * k * std::max(R, 1)));
  AKM_CK(A.tmp.ensure(sizeof(double) * k * std::max(R, 1)));
  AKM_CK(A.part.ensure(sizeof(double) * aafn_part_doubles(n, k, std::max(R, 1))));
  AKM_CK(A.w2.ensure(sizeof(double) * std::max<long long>(n, 1) * std::max(R, 1)));
  if (A.theta_built == plan->theta_version) return AKM_OK;
  if (k > 4096) return plan->fail(AKM_ERR_UNSUPPORTED, "AAFN with %d landmarks (at most 4096 built)", k);
  AKM_CK(A.L.ensure(sizeof(double) * k * k));
  AKM_CK(A.Linv.ensure(sizeof(double) * k * k));
  AKM_CK(A.LinvT.ensure(sizeof(double) * k * k));
  AKM_CK(A.Phi.ensure(sizeof(double) * n * k));
  AKM_CK(A.K21.ensure(sizeof(double) * n * k));
  AKM_CK(A.Sdiag.ensure(sizeof(double) * n));
  AKM_CK(A.g.ensure(sizeof(double) * n));
  AKM_CK(A.scal.ensure(sizeof(double) * 2));
  AKM_CK(A.flag.ensure(sizeof(int)));
  double jitter = 0.0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    int flag = 0;
    AKM_CK(cudaMemsetAsync(A.flag.p, 0, sizeof(int), s));
    AKM_CK(launch_aafn_factor(plan->Xc.as<double>(), n, (int)plan->feat_used.size(), plan->tab, plan->family,
                              plan->sigma_f, plan->ell, plan->sigma_eps, A.lm.as<int>(), A.lmpos.as<int>(), k,
                              A.L.as<double>(), A.Linv.as<double>(), A.LinvT.as<double>(), A.Phi.as<double>(),
                              A.K21.as<double>(),
                              A.Sdiag.as<double>(),
                              A.g.as<double>(), A.scal.as<double>(), A.part.as<double>(), A.flag.as<int>(), jitter, s));
    double sc[2];
    AKM_CK(cudaMemcpyAsync(sc, A.scal.p, sizeof(sc), cudaMemcpyDeviceToHost, s));
    AKM_CK(cudaMemcpyAsync(&flag, A.flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    AKM_CK(cudaStreamSynchronize(s));
    if (flag == 0) {
      A.logdet = sc[0] + sc[1];
      A.theta_built = plan->theta_version;
      return AKM_OK;
    }
    // K11 is SPD in exact arithmetic: one retry with 1e-10 trace(K11)/k on the diagonal
    jitter = 1e-10 * (plan->sigma_f * plan->sigma_f * plan->P + plan->sigma_eps * plan->sigma_eps);
  }
  return plan->fail(AKM_ERR_NONFINITE, "AAFN: the landmark block is not positive definite (Cholesky breakdown)");
}

// out = U^{-1} T  /  U^{-T} T  (n x R row-major, device)
static akm_status aafn_uinv(akm_plan* plan, int R, const double* T, double* out, cudaStream_t s) {
  auto& A = plan->aafn;
  AKM_CK(launch_aafn_uinv(plan->n, A.k, R, A.lm.as<int>(), A.lmpos.as<int>(), A.Linv.as<double>(), A.Phi.as<double>(),
                          A.g.as<double>(), T, A.y1.as<double>(), A.tmp.as<double>(), A.part.as<double>(), out, s));
  plan->launches += 4;
  return AKM_OK;
}
static akm_status aafn_uinvT(akm_plan* plan, int R, const double* T, double* out, cudaStream_t s) {
  auto& A = plan->aafn;
  AKM_CK(launch_aafn_uinvT(plan->n, A.k, R, A.lm.as<int>(), A.lmpos.as<int>(), A.LinvT.as<double>(),
                           A.Phi.as<double>(), A.g.as<double>(), T, A.part.as<double>(), A.tmp.as<double>(),
                           A.y1.as<double>(), A.w2.as<double>(), out, s));
  plan->launches += 5;
  return AKM_OK;
}

// ================================================================== C ABI
extern "C" {

const char* akm_version(void) { return "akm 0.1 (sm_100a, float64 NFFT fast summation)"; }

akm_status akm_create(akm_plan** out, int device) {
  if (!out) return AKM_ERR_INVALID_ARG;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
    cudaGetLastError();
    return AKM_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return AKM_ERR_CUDA;
  akm_plan* p = new (std::nothrow) akm_plan();
  if (!p) return AKM_ERR_OOM;
  p->device = device;
  *out = p;
  return AKM_OK;
}

void akm_destroy(akm_plan* plan) {
  if (!plan) return;
  cudaSetDevice(plan->device);
  cudaDeviceSynchronize();
  delete plan;
}

const char* akm_last_error(const akm_plan* plan) { return plan ? plan->err.c_str() : "null plan"; }

akm_status akm_set_points(akm_plan* plan, const double* X, int64_t n, int32_t p, int64_t ldx, const int32_t* win_feat,
                          const int32_t* win_len, int32_t P, int32_t family, int32_t N, double sigma_over, int32_t m,
                          double eps_B, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  plan->have_points = false;
  plan->have_theta = false;
  cudaStream_t s = S(stream);
  if (n < 0 || n > 2000000000LL) return plan->fail(AKM_ERR_INVALID_ARG, "n out of range (%lld)", (long long)n);
  if (p < 1 || ldx < p) return plan->fail(AKM_ERR_INVALID_ARG, "bad p/ldx (p=%d ldx=%lld)", p, (long long)ldx);
  if (P < 1 || P > AKM_MAX_WINDOWS) return plan->fail(AKM_ERR_INVALID_ARG, "P must be in [1, %d]", AKM_MAX_WINDOWS);
  if (!win_feat || !win_len) return plan->fail(AKM_ERR_INVALID_ARG, "null window arrays");
  if (family != AKM_GAUSSIAN && family != AKM_MATERN12) return plan->fail(AKM_ERR_INVALID_ARG, "unknown family %d", family);
  if (N < 4 || (N % 2) != 0) return plan->fail(AKM_ERR_INVALID_ARG, "N must be even and >= 4 (got %d)", N);
  if (!(sigma_over > 1.0) || !std::isfinite(sigma_over)) return plan->fail(AKM_ERR_INVALID_ARG, "sigma_over must be > 1");
  const double ngd = sigma_over * N;
  const int n_g = (int)std::lround(ngd);
  if (std::fabs(ngd - n_g) > 1e-9 || (n_g % 2) != 0)
    return plan->fail(AKM_ERR_INVALID_ARG, "sigma_over * N must be an even integer (got %g)", ngd);
  if (m < 1 || 2 * m >= n_g) return plan->fail(AKM_ERR_INVALID_ARG, "need 1 <= m and 2m < sigma_over*N");
  if (m != 4 && m != 6 && m != 8) return plan->fail(AKM_ERR_UNSUPPORTED, "window support m = %d not built (4, 6, 8)", m);
  if (!(eps_B >= 0.0 && eps_B < 0.5)) return plan->fail(AKM_ERR_INVALID_ARG, "eps_B must be in [0, 1/2)");
  if (n > 0 && !X) return plan->fail(AKM_ERR_INVALID_ARG, "X is NULL");
  // windows: sizes 1..3, ids in range, pairwise disjoint
  std::vector<int> lens(win_len, win_len + P);
  int tot = 0;
  for (int w = 0; w < P; ++w) {
    if (lens[w] < 1 || lens[w] > 3) return plan->fail(AKM_ERR_INVALID_ARG, "window %d has size %d (must be 1..3)", w, lens[w]);
    tot += lens[w];
  }
  std::vector<int> feats(win_feat, win_feat + tot);
  std::set<int> seen;
  for (int f : feats) {
    if (f < 0 || f >= p) return plan->fail(AKM_ERR_INVALID_ARG, "feature id %d out of range [0, %d)", f, p);
    if (!seen.insert(f).second) return plan->fail(AKM_ERR_INVALID_ARG, "windows overlap in feature %d", f);
  }
  AKM_CK(cudaSetDevice(plan->device));
  plan->n = n;
  plan->n_split = n;  // no cross-product targets until akm_kernel_cross_mvm asks for a split
  plan->p = p;
  plan->P = P;
  plan->family = family;
  plan->N = N;
  plan->m = m;
  plan->deconv_ok = false;  // (N, m, sigma) may change: rebuild the deconvolution table
  plan->n_g = n_g;
  plan->sigma_over = sigma_over;
  plan->eps_B = eps_B;
  plan->beta = kPi * (2.0 - 1.0 / sigma_over);
  plan->win_len = lens;
  plan->win_feat = feats;
  plan->feat_used.assign(feats.begin(), feats.end());
  const int nf = (int)feats.size();
  // compact copy of the used features: Xc[i][j] = X[i][feats[j]]
  AKM_CK(plan->Xc.ensure(sizeof(double) * std::max<long long>(n * nf, 1)));
  if (n > 0) {
    const double* Xd = X;
    DevBuf xstage, fdev;
    if (!is_device_ptr(X)) {
      AKM_CK(xstage.ensure(sizeof(double) * (size_t)((n - 1) * ldx + p)));
      AKM_CK(cudaMemcpyAsync(xstage.p, X, sizeof(double) * (size_t)((n - 1) * ldx + p), cudaMemcpyHostToDevice, s));
      Xd = xstage.as<double>();
    }
    AKM_CK(fdev.ensure(sizeof(int) * nf));
    AKM_CK(cudaMemcpyAsync(fdev.p, feats.data(), sizeof(int) * nf, cudaMemcpyHostToDevice, s));
    AKM_CK(launch_gather_columns(Xd, n, ldx, fdev.as<int>(), nf, plan->Xc.as<double>(), s));
    AKM_CK(cudaStreamSynchronize(s));  // the staging buffers are freed on scope exit
  }
  // per-window table skeleton (feature -> compact column)
  WinTable& tab = plan->tab;
  std::memset(&tab, 0, sizeof(tab));
  tab.P = P;
  tab.N = N;
  tab.n_g = n_g;
  tab.m = m;
  int col = 0;
  for (int w = 0; w < P; ++w) {
    WinGeom& g = tab.w[w];
    g.d = lens[w];
    for (int a = 0; a < 3; ++a) g.feat[a] = 0;
    for (int t = 0; t < g.d; ++t) g.feat[3 - g.d + t] = col++;
  }
  {  // window polynomials (depend on m and sigma only)
    DevBuf pc;
    AKM_CK(pc.ensure(sizeof(double) * kMaxTaps * kPolyLen));
    AKM_CK(cudaMemsetAsync(pc.p, 0, sizeof(double) * kMaxTaps * kPolyLen, s));
    AKM_CK(launch_window_poly(m, plan->beta, pc.as<double>(), s));
    AKM_CK(cudaMemcpyAsync(tab.poly, pc.p, sizeof(double) * kMaxTaps * kPolyLen, cudaMemcpyDeviceToHost, s));
    AKM_CK(cudaStreamSynchronize(s));
    std::memcpy(plan->poly_param.c, tab.poly, sizeof(plan->poly_param.c));
  }
  plan->lo.assign(3 * P, 0.0);
  plan->hi.assign(3 * P, 0.0);
  plan->radius.assign(P, 0.0);
  if (n > 0) {
    std::vector<int> idx(nf);
    for (int j = 0; j < nf; ++j) idx[j] = j;
    DevBuf fd;
    AKM_CK(fd.ensure(sizeof(int) * nf));
    AKM_CK(cudaMemcpyAsync(fd.p, idx.data(), sizeof(int) * nf, cudaMemcpyHostToDevice, s));
    AKM_CK(plan->minmax.ensure(sizeof(double) * 3 * nf));
    AKM_CK(launch_window_minmax(plan->Xc.as<double>(), n, nf, fd.as<int>(), nf, plan->minmax.as<double>(), s));
    std::vector<double> mm(3 * nf);
    AKM_CK(cudaMemcpyAsync(mm.data(), plan->minmax.p, sizeof(double) * 3 * nf, cudaMemcpyDeviceToHost, s));
    AKM_CK(cudaStreamSynchronize(s));
    for (int j = 0; j < nf; ++j)
      if (mm[3 * j + 2] != 0.0) return plan->fail(AKM_ERR_NONFINITE, "X has non-finite values in feature %d", feats[j]);
    for (int w = 0; w < P; ++w) {
      WinGeom& g = tab.w[w];
      for (int a = 3 - g.d; a < 3; ++a) {
        const int j = g.feat[a];
        plan->lo[w * 3 + a] = mm[3 * j];
        plan->hi[w * 3 + a] = mm[3 * j + 1];
        g.center[a] = 0.5 * (mm[3 * j] + mm[3 * j + 1]);  // bounding-box midpoint (reading R2)
      }
    }
    AKM_CK(plan->dtab.ensure(sizeof(WinTable)));
    AKM_CK(cudaMemcpyAsync(plan->dtab.p, &tab, sizeof(WinTable), cudaMemcpyHostToDevice, s));
    AKM_CK(plan->r2.ensure(sizeof(double) * P));
    AKM_CK(launch_window_radius(plan->Xc.as<double>(), n, nf, tab, plan->dtab.as<WinTable>(), plan->r2.as<double>(), s));
    std::vector<double> r2(P);
    AKM_CK(cudaMemcpyAsync(r2.data(), plan->r2.p, sizeof(double) * P, cudaMemcpyDeviceToHost, s));
    AKM_CK(cudaStreamSynchronize(s));
    for (int w = 0; w < P; ++w) plan->radius[w] = std::sqrt(r2[w]);
  }
  plan->radius_local = plan->radius;
  plan->bin_override.clear();
  plan->reg_p = 0;
  plan->reg_eps_I = 0.0;
  plan->aafn.lm_ready = false;
  plan->aafn.theta_built = -1;
  plan->bk_keys.clear();
  plan->c_w.assign(P, 0.0);
  plan->c_w_binned.assign(P, -1.0);
  plan->r_cap = 0;
  plan->have_points = true;
  return AKM_OK;
}

akm_status akm_set_scale_override(akm_plan* plan, const double* c_w) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points) return plan->fail(AKM_ERR_STATE, "set_scale_override before set_points");
  if (!c_w) {
    plan->scale_override.clear();
    return AKM_OK;
  }
  const double rho = 0.25 - plan->eps_B / 2.0;
  for (int w = 0; w < plan->P; ++w) {
    if (!(c_w[w] > 0.0) || !std::isfinite(c_w[w])) return plan->fail(AKM_ERR_INVALID_ARG, "c_w[%d] must be > 0", w);
    if (plan->radius[w] / c_w[w] > rho * (1.0 + 1e-12))
      return plan->fail(AKM_ERR_INVALID_ARG, "c_w[%d] = %g puts points outside the radius-%g ball", w, c_w[w], rho);
  }
  plan->scale_override.assign(c_w, c_w + plan->P);
  plan->have_theta = false;
  return AKM_OK;
}

akm_status akm_set_theta(akm_plan* plan, double sigma_f, double ell, double sigma_eps, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points) return plan->fail(AKM_ERR_STATE, "set_theta before set_points");
  if (!std::isfinite(sigma_f) || !std::isfinite(ell) || !std::isfinite(sigma_eps))
    return plan->fail(AKM_ERR_NONFINITE, "theta has non-finite entries");
  if (!(sigma_f > 0.0) || !(ell > 0.0) || !(sigma_eps >= 0.0))
    return plan->fail(AKM_ERR_INVALID_ARG, "need sigma_f > 0, ell > 0, sigma_eps >= 0");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  plan->have_theta = false;
  ++plan->epoch;  // theta is baked into captured launch sequences
  ++plan->theta_version;
  plan->sigma_f = sigma_f;
  plan->ell = ell;
  plan->sigma_eps = sigma_eps;
  // scale factors (reading R2): Matern fills the ball; Gaussian additionally keeps ell_eff <= 1/sqrt(2 pi N)
  const double rho = 0.25 - plan->eps_B / 2.0;
  bool changed = false;
  for (int w = 0; w < plan->P; ++w) {
    double c;
    if (!plan->scale_override.empty()) {
      c = plan->scale_override[w];
    } else {
      c = plan->radius[w] > 0.0 ? plan->radius[w] / rho : 1.0;
      if (plan->family == AKM_GAUSSIAN) c = std::max(c, ell * std::sqrt(2.0 * kPi * plan->N));
    }
    plan->c_w[w] = c;
    if (c != plan->c_w_binned[w]) changed = true;
  }
  if (plan->n == 0) {
    plan->have_theta = true;
    return AKM_OK;
  }
  if (changed) {
    akm_status st = rebuild_bins(plan, s);
    if (st != AKM_OK) return st;
  }
  if (plan->near_field()) {
    akm_status st = ensure_cell_tab(plan, s);
    if (st != AKM_OK) return st;
  }
  SetupTimer tm(s);
  akm_status st = rebuild_tables(plan, s);
  if (st != AKM_OK) return st;
  tm.mark("b_k + multipliers");
  AKM_CK(cudaGetLastError());
  plan->have_theta = true;
  return AKM_OK;
}

akm_status akm_kernel_mvm(akm_plan* plan, const double* V, int64_t ldv, int32_t r, double* Y, int64_t ldy, void* stream) {
  if (!Y) {
    if (plan) plan->fail(AKM_ERR_INVALID_ARG, "Y is NULL");
    return AKM_ERR_INVALID_ARG;
  }
  return mvm_entry(plan, V, ldv, r, Y, nullptr, nullptr, nullptr, ldy, S(stream));
}

akm_status akm_kernel_deriv_mvm(akm_plan* plan, int32_t which, const double* V, int64_t ldv, int32_t r, double* dY,
                                int64_t ldy, void* stream) {
  if (!dY) {
    if (plan) plan->fail(AKM_ERR_INVALID_ARG, "dY is NULL");
    return AKM_ERR_INVALID_ARG;
  }
  switch (which) {
    case AKM_D_ELL: return mvm_entry(plan, V, ldv, r, nullptr, dY, nullptr, nullptr, ldy, S(stream));
    case AKM_D_SIGMA_F: return mvm_entry(plan, V, ldv, r, nullptr, nullptr, dY, nullptr, ldy, S(stream));
    case AKM_D_SIGMA_EPS: return mvm_entry(plan, V, ldv, r, nullptr, nullptr, nullptr, dY, ldy, S(stream));
    default:
      if (plan) plan->fail(AKM_ERR_INVALID_ARG, "unknown derivative parameter %d", which);
      return AKM_ERR_INVALID_ARG;
  }
}

akm_status akm_kernel_mvm_multi(akm_plan* plan, const double* V, int64_t ldv, int32_t r, double* Y, double* dY_ell,
                                double* dY_sf, int64_t ldy, void* stream) {
  return mvm_entry(plan, V, ldv, r, Y, dY_ell, dY_sf, nullptr, ldy, S(stream));
}

akm_status akm_kernel_cross_mvm(akm_plan* plan, int64_t n_src, const double* V, int64_t ldv, int32_t r, double* Yt,
                                int64_t ldy, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points || !plan->have_theta)
    return plan->fail(AKM_ERR_STATE, "kernel_cross_mvm called before set_points and set_theta");
  const long long n = plan->n;
  if (n_src < 0 || n_src > n) return plan->fail(AKM_ERR_INVALID_ARG, "n_src = %lld outside [0, n = %lld]", (long long)n_src, n);
  if (plan->near_field())
    return plan->fail(AKM_ERR_UNSUPPORTED, "cross product with the inner regularisation (near-field) is not built");
  if (r < 1 || ldv < r || ldy < r) return plan->fail(AKM_ERR_INVALID_ARG, "bad r/ldv/ldy (r=%d ldv=%lld ldy=%lld)", r, (long long)ldv, (long long)ldy);
  const long long n_t = n - n_src;
  if (n_t == 0) return AKM_OK;
  if (!Yt) return plan->fail(AKM_ERR_INVALID_ARG, "Yt is NULL");
  if (n_src > 0 && !V) return plan->fail(AKM_ERR_INVALID_ARG, "V is NULL");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  if (plan->n_split != n_src) {
    // re-sort so that every bin holds its sources first and its targets after them; the spreading
    // then reads only sources and the interpolation visits only targets (item set 1)
    plan->n_split = n_src;
    akm_status st = rebuild_bins(plan, s);
    if (st != AKM_OK) return st;
  }
  const double* Vd = V;
  long long ldvd = ldv;
  if (n_src > 0 && !is_device_ptr(V)) {
    AKM_CK(plan->crossV.ensure(sizeof(double) * n_src * r));
    AKM_CK(copy_rows(plan->crossV.p, sizeof(double) * r, V, sizeof(double) * ldv, sizeof(double) * r, n_src,
                             cudaMemcpyHostToDevice, s));
    Vd = plan->crossV.as<double>();
    ldvd = r;
  }
  if (n_src == 0) {  // nothing to spread: the product is zero
    if (is_device_ptr(Yt)) {
      AKM_CK(cudaMemset2DAsync(Yt, sizeof(double) * ldy, 0, sizeof(double) * r, n_t, s));
    } else {
      for (long long i = 0; i < n_t; ++i) std::memset(Yt + i * ldy, 0, sizeof(double) * r);
    }
    return AKM_OK;
  }
  const bool y_dev = is_device_ptr(Yt);
  double* Yd = Yt;
  long long ldyd = ldy;
  if (!y_dev) {
    AKM_CK(plan->crossY.ensure(sizeof(double) * n_t * r));
    Yd = plan->crossY.as<double>();
    ldyd = r;
  }
  akm_status st = run_mvm(plan, Vd, ldvd, r, Yd, nullptr, nullptr, ldyd, s, /*set=*/1);
  if (st != AKM_OK) return st;
  if (!y_dev) {
    AKM_CK(copy_rows(Yt, sizeof(double) * ldy, Yd, sizeof(double) * r, sizeof(double) * r, n_t,
                             cudaMemcpyDeviceToHost, s));
    AKM_CK(cudaStreamSynchronize(s));
  }
  return AKM_OK;
}

static akm_status objective_impl(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                                 int32_t cg_iters, int32_t lanczos_steps, akm_objective_out* out, double* cg_relres,
                                 void* stream, bool use_aafn);

akm_status akm_objective_diag(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                              int32_t cg_iters, int32_t lanczos_steps, akm_objective_out* out, double* cg_relres,
                              void* stream) {
  return objective_impl(plan, y, Z, ldz, n_z, cg_iters, lanczos_steps, out, cg_relres, stream, false);
}

akm_status akm_objective(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z, int32_t cg_iters,
                         int32_t lanczos_steps, akm_objective_out* out, double* cg_relres, void* stream) {
  return objective_impl(plan, y, Z, ldz, n_z, cg_iters, lanczos_steps, out, cg_relres, stream,
                        plan && plan->aafn.kpw > 0);
}

static akm_status objective_impl(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                                 int32_t cg_iters, int32_t lanczos_steps, akm_objective_out* out, double* cg_relres,
                                 void* stream, bool use_aafn) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  NvtxRange nvtx("akm S8 objective");
  plan->err.clear();
  if (!plan->have_points || !plan->have_theta)
    return plan->fail(AKM_ERR_STATE, "objective_diag called before set_points and set_theta");
  if (!out) return plan->fail(AKM_ERR_INVALID_ARG, "out is NULL");
  if (n_z < 1 || n_z > AKM_MAX_PROBES) return plan->fail(AKM_ERR_INVALID_ARG, "n_z must be in [1, %d]", AKM_MAX_PROBES);
  if (ldz < n_z) return plan->fail(AKM_ERR_INVALID_ARG, "ldz < n_z");
  if (cg_iters < 0 || cg_iters > kKrMaxIters) return plan->fail(AKM_ERR_INVALID_ARG, "cg_iters must be in [0, %d]", kKrMaxIters);
  if (lanczos_steps < 0 || lanczos_steps > kKrMaxSteps)
    return plan->fail(AKM_ERR_INVALID_ARG, "lanczos_steps must be in [0, %d]", kKrMaxSteps);
  const long long n = plan->n;
  if (n < 1) return plan->fail(AKM_ERR_INVALID_ARG, "objective needs n >= 1");
  if (!y || !Z) return plan->fail(AKM_ERR_INVALID_ARG, "y or Z is NULL");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  const int R = 1 + n_z;
  const int L = std::max(lanczos_steps, 1);
  const long long slab = n * R;
  // stage host inputs
  const double* yd = y;
  const double* Zd = Z;
  long long ldzd = ldz;
  const bool y_dev = is_device_ptr(y), z_dev = is_device_ptr(Z);
  if (!y_dev || !z_dev) {
    AKM_CK(plan->krStage.ensure(sizeof(double) * (size_t)(n + n * n_z)));
    double* st = plan->krStage.as<double>();
    if (!y_dev) {
      AKM_CK(cudaMemcpyAsync(st, y, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      yd = st;
    }
    if (!z_dev) {
      AKM_CK(copy_rows(st + n, sizeof(double) * n_z, Z, sizeof(double) * ldz, sizeof(double) * n_z, n,
                               cudaMemcpyHostToDevice, s));
      Zd = st + n;
      ldzd = n_z;
    }
  }
  const int nblk = kr_blocks();
  AKM_CK(plan->krB.ensure(sizeof(double) * slab));
  AKM_CK(plan->krKB.ensure(sizeof(double) * slab));
  AKM_CK(plan->krW.ensure(sizeof(double) * slab));
  AKM_CK(plan->krX.ensure(sizeof(double) * n));
  AKM_CK(plan->krY.ensure(sizeof(double) * n));
  AKM_CK(plan->krQ.ensure(sizeof(double) * slab * L));
  AKM_CK(plan->krPart.ensure(sizeof(double) * (size_t)nblk * std::max(2, L) * R));
  AKM_CK(plan->krH.ensure(sizeof(double) * (size_t)L * R));
  AKM_CK(plan->krState.ensure(kr_state_bytes()));
  AKM_CK(plan->krErr.ensure(sizeof(int)));
  AKM_CK(cudaMemsetAsync(plan->krErr.p, 0, sizeof(int), s));
  double* B = plan->krB.as<double>();
  double* KB = plan->krKB.as<double>();
  double* W = plan->krW.as<double>();
  double* Q = plan->krQ.as<double>();
  double* part = plan->krPart.as<double>();
  void* st = plan->krState.p;
  // M = diag(Khat): kappa(0) = 1 for every sub-kernel (reading R11).  AAFN (reading R15): the drivers
  // run on S_op = U^{-1} Khat U^{-T} with M = I there, column 0 = U^{-1} y (CG on S_op x^ = U^{-1} y is
  // PCG on Khat x = y with x = U^{-T} x^, and y^T x = (U^{-1} y)^T x^)
  double c = plan->sigma_f * plan->sigma_f * plan->P + plan->sigma_eps * plan->sigma_eps;
  auto& A = plan->aafn;
  const double* y_user = yd;
  if (use_aafn) {
    akm_status sb = aafn_build(plan, R, s);
    if (sb != AKM_OK) return sb;
    AKM_CK(A.Bt.ensure(sizeof(double) * slab));
    AKM_CK(A.KBt.ensure(sizeof(double) * slab));
    AKM_CK(A.yh.ensure(sizeof(double) * n));
    sb = aafn_uinv(plan, 1, yd, A.yh.as<double>(), s);
    if (sb != AKM_OK) return sb;
    yd = A.yh.as<double>();
    c = 1.0;
  }
  AKM_CK(launch_kr_load(n, R, yd, Zd, ldzd, B, plan->krY.as<double>(), s));
  AKM_CK(launch_kr_col2(n, R, B, B, part, s));
  AKM_CK(launch_kr_init(st, part, R, c, s));
  AKM_CK(launch_kr_start(n, R, st, B, W, Q, plan->krX.as<double>(), s));
  const int T = std::max(cg_iters, lanczos_steps);
  int products = 0;
  long long live_units = 0;  // sum over products of the columns multiplied
  for (int t = 0; t < T; ++t) {
    akm_status stt;
    // once every Lanczos recurrence has finished (t >= lanczos_steps) only the CG column is live: the
    // product runs at r = 1 on column 0 (the dead columns of KB keep stale values nobody reads)
    const int rr = (t >= lanczos_steps) ? 1 : R;
    if (use_aafn) {
      stt = aafn_uinvT(plan, R, B, A.Bt.as<double>(), s);
      if (stt == AKM_OK) stt = run_mvm(plan, A.Bt.as<double>(), R, rr, A.KBt.as<double>(), nullptr, nullptr, R, s);
      if (stt == AKM_OK) stt = aafn_uinv(plan, R, A.KBt.as<double>(), KB, s);
    } else {
      stt = run_mvm(plan, B, R, rr, KB, nullptr, nullptr, R, s);
    }
    live_units += rr;
    if (stt != AKM_OK) return stt;
    ++products;
    AKM_CK(launch_kr_col2(n, R, B, KB, part, s));
    AKM_CK(launch_kr_after_dots(st, part, R, cg_iters, lanczos_steps, s));
    const double* Qt = Q + (long long)std::min(t, L - 1) * slab;
    const double* Qtm1 = (t > 0 && t < L) ? Q + (long long)(t - 1) * slab : nullptr;
    AKM_CK(launch_kr_update(n, R, st, B, KB, W, Qt, Qtm1, plan->krX.as<double>(), s));
    if (t + 1 < lanczos_steps) {
      for (int pass = 0; pass < 2; ++pass)  // classical Gram-Schmidt, twice (reading R11)
        AKM_CK(launch_kr_reorth(n, R, t + 1, st, Q, slab, W, part, plan->krH.as<double>(), s));
    }
    AKM_CK(launch_kr_col2(n, R, W, W, part, s));
    AKM_CK(launch_kr_after_norms(st, part, R, s));
    AKM_CK(launch_kr_finalize(n, R, st, B, W, (t + 1 < L) ? Q + (long long)(t + 1) * slab : nullptr, s));
    AKM_CK(launch_kr_advance(st, R, s));
    plan->launches += 7 + ((t + 1 < lanczos_steps) ? 6 : 0);
  }
  AKM_CK(launch_kr_col2(n, 1, plan->krY.as<double>(), plan->krX.as<double>(), part, s));
  AKM_CK(launch_kr_slq_quad(st, R, part, plan->krErr.as<int>(), s));
  // true relative residual ||y - Khat x|| / ||y|| of the CG solution (one extra product with r = 1)
  double rn[2] = {0.0, 0.0};
  if (cg_iters > 0) {
    AKM_CK(plan->krRes.ensure(sizeof(double) * (2 * n + 8)));
    double* xu = plan->krRes.as<double>();      // x in the user's space
    double* kx = xu + n;                       // Khat x
    double* nrm = kx + n;                      // the two norms
    const double* x = plan->krX.as<double>();
    if (use_aafn) {
      akm_status sx = aafn_uinvT(plan, 1, x, xu, s);
      if (sx != AKM_OK) return sx;
      x = xu;
    }
    akm_status sx = run_mvm(plan, x, 1, 1, kx, nullptr, nullptr, 1, s);
    if (sx != AKM_OK) return sx;
    AKM_CK(launch_resid_norms(n, y_user, kx, part, nrm, s));
    AKM_CK(cudaMemcpyAsync(rn, nrm, sizeof(rn), cudaMemcpyDeviceToHost, s));
  }
  size_t o_quad, o_samp, o_steps, o_hist, o_zn;
  kr_summary_offsets(&o_quad, &o_samp, &o_steps, &o_hist, &o_zn);
  double quad = 0.0;
  std::vector<double> samples(R), hist(std::max(cg_iters, 1));
  std::vector<int> steps(R);
  int errf = 0;
  const char* base = static_cast<const char*>(st);
  AKM_CK(cudaMemcpyAsync(&quad, base + o_quad, sizeof(double), cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaMemcpyAsync(samples.data(), base + o_samp, sizeof(double) * R, cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaMemcpyAsync(steps.data(), base + o_steps, sizeof(int) * R, cudaMemcpyDeviceToHost, s));
  if (cg_iters > 0)
    AKM_CK(cudaMemcpyAsync(hist.data(), base + o_hist, sizeof(double) * cg_iters, cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaMemcpyAsync(&errf, plan->krErr.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaStreamSynchronize(s));
  std::memset(out, 0, sizeof(*out));
  out->quad = quad;
  out->logdet_M = use_aafn ? A.logdet : (double)n * std::log(c);
  out->cg_relres_true = (cg_iters > 0 && rn[1] > 0.0) ? std::sqrt(rn[0] / rn[1]) : 0.0;
  out->landmarks = use_aafn ? A.k : 0;
  out->n_log_2pi = (double)n * std::log(2.0 * kPi);
  double acc = 0.0;
  for (int i = 0; i < n_z; ++i) {
    out->samples[i] = samples[i + 1];
    out->steps[i] = steps[i + 1];
    acc += samples[i + 1];
  }
  out->slq = acc / n_z;
  out->Z = 0.5 * (out->quad + out->logdet_M + out->slq + out->n_log_2pi);
  out->n_z = n_z;
  out->cg_iters = cg_iters;
  out->lanczos_steps = lanczos_steps;
  out->products = products;
  out->product_columns = live_units;
  // iterations after an exactly-zero residual are not run (history -1): report the last one run
  out->cg_relres = 1.0;
  for (int t = 0; t < cg_iters; ++t)
    if (hist[t] >= 0.0) out->cg_relres = hist[t];
  if (cg_relres)
    for (int t = 0; t < cg_iters; ++t) cg_relres[t] = hist[t];
  if (errf) return plan->fail(AKM_ERR_NONFINITE, "SLQ: tridiagonal eigensolve failed or non-positive Ritz value (flags %d)", errf);
  return AKM_OK;
}

static akm_status gradient_impl(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                                int32_t cg_iters, double* grad, double* cg_relres, void* stream, bool use_aafn,
                                double* dots = nullptr, double* sqnorms = nullptr);

akm_status akm_gradient_diag(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                             int32_t cg_iters, double* grad, double* cg_relres, void* stream) {
  return gradient_impl(plan, y, Z, ldz, n_z, cg_iters, grad, cg_relres, stream, false);
}

akm_status akm_gradient(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z, int32_t cg_iters,
                        double* grad, double* cg_relres, void* stream) {
  return gradient_impl(plan, y, Z, ldz, n_z, cg_iters, grad, cg_relres, stream, plan && plan->aafn.kpw > 0);
}

akm_status akm_gradient_columns(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                                int32_t cg_iters, int32_t preconditioned, double* dots, double* sqnorms,
                                double* cg_relres, void* stream) {
  if (plan && (!dots || !sqnorms)) return plan->fail(AKM_ERR_INVALID_ARG, "dots / sqnorms are NULL");
  double grad[3];
  return gradient_impl(plan, y, Z, ldz, n_z, cg_iters, grad, cg_relres, stream,
                       plan && preconditioned && plan->aafn.kpw > 0, dots, sqnorms);
}

static akm_status gradient_impl(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                                int32_t cg_iters, double* grad, double* cg_relres, void* stream, bool use_aafn,
                                double* dots, double* sqnorms) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  NvtxRange nvtx("akm f1 gradient");
  plan->err.clear();
  if (!plan->have_points || !plan->have_theta)
    return plan->fail(AKM_ERR_STATE, "gradient_diag called before set_points and set_theta");
  if (!grad) return plan->fail(AKM_ERR_INVALID_ARG, "grad is NULL");
  if (n_z < 1 || n_z > AKM_MAX_PROBES) return plan->fail(AKM_ERR_INVALID_ARG, "n_z must be in [1, %d]", AKM_MAX_PROBES);
  if (ldz < n_z) return plan->fail(AKM_ERR_INVALID_ARG, "ldz < n_z");
  if (cg_iters < 0 || cg_iters > kKrMaxIters) return plan->fail(AKM_ERR_INVALID_ARG, "cg_iters must be in [0, %d]", kKrMaxIters);
  const long long n = plan->n;
  if (n < 1) return plan->fail(AKM_ERR_INVALID_ARG, "gradient needs n >= 1");
  if (!y || !Z) return plan->fail(AKM_ERR_INVALID_ARG, "y or Z is NULL");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  const int R = 1 + n_z;
  const long long blk = n * R;
  const double* yd = y;
  const double* Zd = Z;
  long long ldzd = ldz;
  const bool y_dev = is_device_ptr(y), z_dev = is_device_ptr(Z);
  if (!y_dev || !z_dev) {
    AKM_CK(plan->krStage.ensure(sizeof(double) * (size_t)(n + n * n_z)));
    double* st = plan->krStage.as<double>();
    if (!y_dev) {
      AKM_CK(cudaMemcpyAsync(st, y, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      yd = st;
    }
    if (!z_dev) {
      AKM_CK(copy_rows(st + n, sizeof(double) * n_z, Z, sizeof(double) * ldz, sizeof(double) * n_z, n,
                               cudaMemcpyHostToDevice, s));
      Zd = st + n;
      ldzd = n_z;
    }
  }
  const int nblk = kr_blocks();
  AKM_CK(plan->krB.ensure(sizeof(double) * blk));
  AKM_CK(plan->krKB.ensure(sizeof(double) * blk));
  AKM_CK(plan->krW.ensure(sizeof(double) * blk));
  AKM_CK(plan->krY.ensure(sizeof(double) * n));
  AKM_CK(plan->gX.ensure(sizeof(double) * blk));
  AKM_CK(plan->gP.ensure(sizeof(double) * blk));
  AKM_CK(plan->gB2.ensure(sizeof(double) * blk));
  AKM_CK(plan->gD1.ensure(sizeof(double) * blk));
  AKM_CK(plan->gD2.ensure(sizeof(double) * blk));
  AKM_CK(plan->krPart.ensure(sizeof(double) * (size_t)nblk * 2 * R));
  AKM_CK(plan->gState.ensure(bcg_state_bytes()));
  double* B = plan->krB.as<double>();
  double* KP = plan->krKB.as<double>();
  double* Rr = plan->krW.as<double>();
  double* X = plan->gX.as<double>();
  double* P = plan->gP.as<double>();
  double* part = plan->krPart.as<double>();
  void* st = plan->gState.p;
  // M = diag(Khat) = c I (reading R11); dc/dsigma_f = 2 sigma_f P, dc/dsigma_eps = 2 sigma_eps.
  // AAFN (reading R15): block CG on S_op = U^{-1} Khat U^{-T} from U^{-1} [y | Z] (M = I there), the
  // solutions mapped back by U^{-T}; the plain Hutchinson form (no dM/dtheta terms: dc = 0 below)
  const double c = use_aafn ? 1.0 : plan->sigma_f * plan->sigma_f * plan->P + plan->sigma_eps * plan->sigma_eps;
  auto& A = plan->aafn;
  AKM_CK(launch_kr_load(n, R, yd, Zd, ldzd, B, plan->krY.as<double>(), s));
  const double* Bcg = B;  // right-hand sides of the CG
  if (use_aafn) {
    akm_status sb = aafn_build(plan, R, s);
    if (sb != AKM_OK) return sb;
    AKM_CK(A.Bt.ensure(sizeof(double) * blk));
    AKM_CK(A.KBt.ensure(sizeof(double) * blk));
    AKM_CK(A.Bh.ensure(sizeof(double) * blk));
    sb = aafn_uinv(plan, R, B, A.Bh.as<double>(), s);
    if (sb != AKM_OK) return sb;
    Bcg = A.Bh.as<double>();
  }
  AKM_CK(launch_kr_col2(n, R, Bcg, Bcg, part, s));
  AKM_CK(launch_bcg_init(st, part, R, c, s));
  AKM_CK(launch_bcg_start(n, R, st, Bcg, Rr, P, X, s));
  plan->launches += 5;
  for (int t = 0; t < cg_iters; ++t) {
    akm_status stt;
    if (use_aafn) {
      stt = aafn_uinvT(plan, R, P, A.Bt.as<double>(), s);
      if (stt == AKM_OK) stt = run_mvm(plan, A.Bt.as<double>(), R, R, A.KBt.as<double>(), nullptr, nullptr, R, s);
      if (stt == AKM_OK) stt = aafn_uinv(plan, R, A.KBt.as<double>(), KP, s);
    } else {
      stt = run_mvm(plan, P, R, R, KP, nullptr, nullptr, R, s);
    }
    if (stt != AKM_OK) return stt;
    AKM_CK(launch_kr_col2(n, R, P, KP, part, s));
    AKM_CK(launch_bcg_after_dots(st, part, R, s));
    AKM_CK(launch_bcg_update(n, R, st, P, KP, Rr, X, s));
    AKM_CK(launch_kr_col2(n, R, Rr, Rr, part, s));
    AKM_CK(launch_bcg_after_norms(st, part, R, t, s));
    AKM_CK(launch_bcg_dir(n, R, st, Rr, P, s));
    plan->launches += 6;
  }
  if (use_aafn) {  // X = U^{-T} X^ (the solutions of Khat X = [y | Z])
    akm_status sx = aafn_uinvT(plan, R, X, A.Bt.as<double>(), s);
    if (sx != AKM_OK) return sx;
    AKM_CK(cudaMemcpyAsync(X, A.Bt.p, sizeof(double) * blk, cudaMemcpyDeviceToDevice, s));
  }
  // one fused derivative product on [alpha | Z]
  double* B2 = plan->gB2.as<double>();
  double* D1 = plan->gD1.as<double>();
  double* D2 = plan->gD2.as<double>();
  AKM_CK(launch_bcg_grad_rhs(n, R, X, B, B2, s));
  akm_status stt = run_mvm(plan, B2, R, R, nullptr, D1, D2, R, s);
  if (stt != AKM_OK) return stt;
  const double* Ds[3] = {D1, D2, B2};  // ell, sigma_f, sigma_eps (dKhat/dsigma_eps = 2 sigma_eps I)
  for (int j = 0; j < 3; ++j) {
    AKM_CK(launch_kr_col2(n, R, X, Ds[j], part, s));
    AKM_CK(launch_bcg_store(st, part, R, j, s));
  }
  plan->launches += 7;
  size_t o_hist, o_out, o_bn;
  bcg_offsets(&o_hist, &o_out, &o_bn);
  std::vector<double> outv(3 * 2 * kKrMaxR), bn(R), hist(std::max(cg_iters, 1));
  const char* base = static_cast<const char*>(st);
  AKM_CK(cudaMemcpyAsync(outv.data(), base + o_out, sizeof(double) * outv.size(), cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaMemcpyAsync(bn.data(), base + o_bn, sizeof(double) * R, cudaMemcpyDeviceToHost, s));
  if (cg_iters > 0)
    AKM_CK(cudaMemcpyAsync(hist.data(), base + o_hist, sizeof(double) * cg_iters, cudaMemcpyDeviceToHost, s));
  AKM_CK(cudaStreamSynchronize(s));
  // eq. (div): 1/2 (-alpha^T dK alpha + n dc/c + (1/n_z) sum_i [(Khat^{-1} z_i)^T dK z_i - dc/c ||z_i||^2])
  const double sf = plan->sigma_f, se = plan->sigma_eps;
  const double scale[3] = {1.0, 1.0, 2.0 * se};          // dK applied: D1, D2 as computed; 2 se * B2
  const double dc[3] = {0.0, use_aafn ? 0.0 : 2.0 * sf * plan->P, use_aafn ? 0.0 : 2.0 * se};
  const int slot_of_param[3] = {1, 0, 2};                  // grad order (sigma_f, ell, sigma_eps)
  if (dots) {  // raw per-column terms for the probe-sharded gradient (dist.sharded_gradient)
    for (int k = 0; k < 3; ++k) {
      const int j = slot_of_param[k];
      for (int i = 0; i < R; ++i) dots[k * R + i] = scale[j] * outv[j * 2 * kKrMaxR + 2 * i];
    }
    for (int i = 0; i < R; ++i) sqnorms[i] = bn[i] * bn[i];
  }
  for (int k = 0; k < 3; ++k) {
    const int j = slot_of_param[k];
    const double* o = outv.data() + j * 2 * kKrMaxR;
    double probes = 0.0;
    for (int i = 1; i < R; ++i) probes += scale[j] * o[2 * i] - dc[j] / c * bn[i] * bn[i];
    grad[k] = 0.5 * (-scale[j] * o[0] + (double)n * dc[j] / c + probes / n_z);
  }
  if (cg_relres)
    for (int t = 0; t < cg_iters; ++t) cg_relres[t] = hist[t];
  return AKM_OK;
}

// ---------------------------------------------------------------- point sharding
akm_status akm_get_bounds(const akm_plan* plan, double* lo, double* hi) {
  if (!plan || !lo || !hi) return AKM_ERR_INVALID_ARG;
  if (!plan->have_points) return AKM_ERR_STATE;
  for (int w = 0; w < plan->P; ++w)
    for (int a = 0; a < 3; ++a) {
      const bool real = a >= 3 - plan->tab.w[w].d;
      lo[w * 3 + a] = !real ? 0.0 : plan->n > 0 ? plan->lo[w * 3 + a] : HUGE_VAL;
      hi[w * 3 + a] = !real ? 0.0 : plan->n > 0 ? plan->hi[w * 3 + a] : -HUGE_VAL;
    }
  return AKM_OK;
}

akm_status akm_set_bounds(akm_plan* plan, const double* lo, const double* hi, double* radius_local, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points) return plan->fail(AKM_ERR_STATE, "set_bounds before set_points");
  if (!lo || !hi || !radius_local) return plan->fail(AKM_ERR_INVALID_ARG, "null bounds / radius array");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  WinTable& tab = plan->tab;
  for (int w = 0; w < plan->P; ++w)
    for (int a = 3 - tab.w[w].d; a < 3; ++a) {
      const int k = w * 3 + a;
      if (!std::isfinite(lo[k]) || !std::isfinite(hi[k]) || lo[k] > hi[k])
        return plan->fail(AKM_ERR_INVALID_ARG, "window %d axis %d: bounds [%g, %g] are not a finite interval", w, a,
                          lo[k], hi[k]);
      if (plan->n > 0 && (lo[k] > plan->lo[k] || hi[k] < plan->hi[k]))
        return plan->fail(AKM_ERR_INVALID_ARG, "window %d axis %d: bounds [%g, %g] do not contain this plan's points",
                          w, a, lo[k], hi[k]);
    }
  for (int w = 0; w < plan->P; ++w)
    for (int a = 3 - tab.w[w].d; a < 3; ++a) {
      const int k = w * 3 + a;
      plan->lo[k] = lo[k];
      plan->hi[k] = hi[k];
      tab.w[w].center[a] = 0.5 * (lo[k] + hi[k]);  // bounding-box midpoint of the union (reading R2)
    }
  std::vector<double> r2(plan->P, 0.0);
  if (plan->n > 0) {
    AKM_CK(cudaMemcpyAsync(plan->dtab.p, &tab, sizeof(WinTable), cudaMemcpyHostToDevice, s));
    AKM_CK(launch_window_radius(plan->Xc.as<double>(), plan->n, (long long)plan->feat_used.size(), tab,
                                plan->dtab.as<WinTable>(), plan->r2.as<double>(), s));
    AKM_CK(cudaMemcpyAsync(r2.data(), plan->r2.p, sizeof(double) * plan->P, cudaMemcpyDeviceToHost, s));
    AKM_CK(cudaStreamSynchronize(s));
  }
  for (int w = 0; w < plan->P; ++w) radius_local[w] = plan->radius[w] = plan->radius_local[w] = std::sqrt(r2[w]);
  plan->c_w_binned.assign(plan->P, -1.0);
  plan->have_theta = false;
  return AKM_OK;
}

akm_status akm_set_radius(akm_plan* plan, const double* radius) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points) return plan->fail(AKM_ERR_STATE, "set_radius before set_points");
  if (!radius) return plan->fail(AKM_ERR_INVALID_ARG, "radius is NULL");
  for (int w = 0; w < plan->P; ++w)
    if (!std::isfinite(radius[w]) || radius[w] < plan->radius_local[w])
      return plan->fail(AKM_ERR_INVALID_ARG, "radius[%d] = %g is below this plan's own radius %g", w, radius[w],
                        plan->radius_local[w]);
  plan->radius.assign(radius, radius + plan->P);
  plan->c_w_binned.assign(plan->P, -1.0);
  plan->have_theta = false;
  return AKM_OK;
}

akm_status akm_set_bin_override(akm_plan* plan, const int32_t* bins) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points) return plan->fail(AKM_ERR_STATE, "set_bin_override before set_points");
  if (!bins) {
    plan->bin_override.clear();
  } else {
    for (int w = 0; w < plan->P; ++w)
      if (bins[w] != 1 && bins[w] != 2 && bins[w] != 3 && bins[w] != 4 && bins[w] != 6 && bins[w] != 8)
        return plan->fail(AKM_ERR_INVALID_ARG, "bin edge %d of window %d not in {1,2,3,4,6,8}", bins[w], w);
    plan->bin_override.assign(bins, bins + plan->P);
  }
  plan->c_w_binned.assign(plan->P, -1.0);
  plan->have_theta = false;
  return AKM_OK;
}

akm_status akm_grid_size(const akm_plan* plan, int32_t r, int64_t* count) {
  if (!plan || !count || r < 1) return AKM_ERR_INVALID_ARG;
  if (!plan->have_points || !plan->have_theta) return AKM_ERR_STATE;
  *count = (int64_t)plan->total_taps * r;
  return AKM_OK;
}

akm_status akm_spread_grid(akm_plan* plan, const double* V, int64_t ldv, int32_t r, double* grid, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points || !plan->have_theta) return plan->fail(AKM_ERR_STATE, "spread_grid before set_points / set_theta");
  if (r < 1 || ldv < r) return plan->fail(AKM_ERR_INVALID_ARG, "bad r/ldv (r=%d ldv=%lld)", r, (long long)ldv);
  if (plan->n == 0) return plan->fail(AKM_ERR_INVALID_ARG, "spread_grid needs n >= 1 on this plan");
  if (!is_device_ptr(V) || !is_device_ptr(grid)) return plan->fail(AKM_ERR_INVALID_ARG, "V and grid must be device memory");
  if (plan->n_split != plan->n) return plan->fail(AKM_ERR_STATE, "spread_grid on a plan sorted for a cross product");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  akm_status st = ensure_rhs_workspace(plan, r);
  if (st != AKM_OK) return st;
  akm_plan::EvSet* ev = plan->profiling ? plan->next_set() : nullptr;
  if (ev) AKM_CK(cudaEventRecord(ev->e[0], s));
  st = enqueue_spread(plan, V, ldv, r, grid, s, 0);
  if (st != AKM_OK) return st;
  if (ev) AKM_CK(cudaEventRecord(ev->e[1], s));
  plan->split_ev = ev;
  return AKM_OK;
}

akm_status akm_mvm_from_grid(akm_plan* plan, const double* grid, const double* V, int64_t ldv, int32_t r, double* Y,
                             double* dY_ell, double* dY_sf, int64_t ldy, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points || !plan->have_theta) return plan->fail(AKM_ERR_STATE, "mvm_from_grid before set_points / set_theta");
  if (r < 1 || ldv < r || ldy < r) return plan->fail(AKM_ERR_INVALID_ARG, "bad r/ldv/ldy (r=%d ldv=%lld ldy=%lld)", r,
                                                   (long long)ldv, (long long)ldy);
  if (!Y && !dY_ell && !dY_sf) return plan->fail(AKM_ERR_INVALID_ARG, "no output requested");
  if (plan->n == 0) return plan->fail(AKM_ERR_INVALID_ARG, "mvm_from_grid needs n >= 1 on this plan");
  const double* outs[3] = {Y, dY_ell, dY_sf};
  for (const double* o : outs)
    if (o && !is_device_ptr(o)) return plan->fail(AKM_ERR_INVALID_ARG, "outputs must be device memory");
  if (!is_device_ptr(V) || !is_device_ptr(grid)) return plan->fail(AKM_ERR_INVALID_ARG, "V and grid must be device memory");
  if (plan->n_split != plan->n) return plan->fail(AKM_ERR_STATE, "mvm_from_grid on a plan sorted for a cross product");
  if (plan->near_field())
    return plan->fail(AKM_ERR_UNSUPPORTED, "point sharding with the inner regularisation (near-field) is not built");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  akm_status st = ensure_rhs_workspace(plan, r);
  if (st != AKM_OK) return st;
  akm_plan::EvSet* ev = plan->profiling ? plan->split_ev : nullptr;
  plan->split_ev = nullptr;
  return enqueue_finish(plan, grid, V, ldv, r, Y, dY_ell, dY_sf, ldy, s, 0, ev);
}

akm_status akm_set_preconditioner(akm_plan* plan, int32_t k_per_window) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points) return plan->fail(AKM_ERR_STATE, "set_preconditioner before set_points");
  if (k_per_window < 0 || k_per_window > 4096) return plan->fail(AKM_ERR_INVALID_ARG, "k_per_window must be in [0, 4096]");
  if (k_per_window != plan->aafn.kpw) {
    plan->aafn.kpw = k_per_window;
    plan->aafn.lm_ready = false;
    plan->aafn.theta_built = -1;
  }
  return AKM_OK;
}

akm_status akm_precond_apply(akm_plan* plan, int32_t transpose, const double* T, int32_t r, double* out, double* logdet,
                             int32_t* landmarks, void* stream) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points || !plan->have_theta) return plan->fail(AKM_ERR_STATE, "precond_apply before set_points / set_theta");
  if (plan->aafn.kpw <= 0) return plan->fail(AKM_ERR_STATE, "no AAFN preconditioner set (akm_set_preconditioner)");
  if (r < 1 || r > kKrMaxR) return plan->fail(AKM_ERR_INVALID_ARG, "r must be in [1, %d]", kKrMaxR);
  if (plan->n < 1) return plan->fail(AKM_ERR_INVALID_ARG, "precond_apply needs n >= 1");
  if (!is_device_ptr(T) || !is_device_ptr(out)) return plan->fail(AKM_ERR_INVALID_ARG, "T and out must be device memory");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  akm_status st = aafn_build(plan, r, s);
  if (st != AKM_OK) return st;
  st = transpose ? aafn_uinvT(plan, r, T, out, s) : aafn_uinv(plan, r, T, out, s);
  if (st != AKM_OK) return st;
  if (logdet) *logdet = plan->aafn.logdet;
  if (landmarks) {
    AKM_CK(cudaMemcpyAsync(landmarks, plan->aafn.lm.p, sizeof(int) * plan->aafn.k, cudaMemcpyDeviceToHost, s));
    AKM_CK(cudaStreamSynchronize(s));
  }
  return AKM_OK;
}

akm_status akm_precond_landmarks(akm_plan* plan, int32_t* count, void* stream) {
  if (!plan || !count) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points) return plan->fail(AKM_ERR_STATE, "precond_landmarks before set_points");
  if (plan->aafn.kpw <= 0) return plan->fail(AKM_ERR_STATE, "no AAFN preconditioner set (akm_set_preconditioner)");
  if (plan->n < 1) return plan->fail(AKM_ERR_INVALID_ARG, "needs n >= 1");
  cudaStream_t s = S(stream);
  AKM_CK(cudaSetDevice(plan->device));
  if (!plan->aafn.lm_ready) {
    akm_status st = aafn_landmarks(plan, s);
    if (st != AKM_OK) return st;
  }
  *count = plan->aafn.k;
  return AKM_OK;
}

akm_status akm_set_regularization(akm_plan* plan, double eps_I, int32_t p) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  if (!plan->have_points) return plan->fail(AKM_ERR_STATE, "set_regularization before set_points");
  if (p < 0 || p > kRegMaxP) return plan->fail(AKM_ERR_INVALID_ARG, "p must be in [0, %d]", kRegMaxP);
  if (!(eps_I >= 0.0 && eps_I < 0.25)) return plan->fail(AKM_ERR_INVALID_ARG, "eps_I must be in [0, 1/4)");
  if (p > 0 && eps_I > 0.0 && eps_I >= 0.5 - plan->eps_B)
    return plan->fail(AKM_ERR_INVALID_ARG, "eps_I must stay below 1/2 - eps_B");
  plan->reg_p = p;
  plan->reg_eps_I = p > 0 ? eps_I : 0.0;
  plan->have_theta = false;
  plan->r_cap = 0;  // the near-field workspace is sized in ensure_rhs_workspace (never inside a graph capture)
  return AKM_OK;
}

akm_status akm_set_deterministic(akm_plan* plan, int32_t on) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->err.clear();
  plan->det = on != 0;
  ++plan->epoch;     // captured launch sequences bake the flush mode in
  plan->r_cap = 0;   // the limb workspace is sized in ensure_rhs_workspace (never inside a graph capture)
  return AKM_OK;
}

akm_status akm_get_window_poly(const akm_plan* plan, double* coef, int32_t* taps, int32_t* degree) {
  if (!plan || !coef || !taps || !degree) return AKM_ERR_INVALID_ARG;
  if (!plan->have_points) return AKM_ERR_STATE;
  *taps = 2 * plan->m;
  *degree = kPolyDeg;
  std::memcpy(coef, plan->poly_param.c, sizeof(double) * 2 * plan->m * kPolyLen);
  return AKM_OK;
}

akm_status akm_set_profiling(akm_plan* plan, int32_t enable) {
  if (!plan) return AKM_ERR_INVALID_ARG;
  plan->profiling = enable != 0;
  return AKM_OK;
}

akm_status akm_get_stage_times(akm_plan* plan, akm_stage_times* out, int32_t reset) {
  if (!plan || !out) return AKM_ERR_INVALID_ARG;
  cudaSetDevice(plan->device);
  for (auto& es : plan->ring) plan->drain(es);
  out->spread_ms = plan->stage_ms[0];
  out->fft_ms = plan->stage_ms[1];
  out->interp_ms = plan->stage_ms[2];
  out->epilogue_ms = plan->stage_ms[3];
  out->exchange_ms = plan->stage_ms[4];
  out->calls = plan->prof_calls;
  out->kernel_launches = plan->launches;
  out->spread_launches = plan->spread_launches;
  out->interp_launches = plan->interp_launches;
  if (reset) {
    for (double& v : plan->stage_ms) v = 0.0;
    plan->prof_calls = plan->launches = plan->spread_launches = plan->interp_launches = 0;
  }
  return AKM_OK;
}

akm_status akm_get_info(const akm_plan* plan, akm_info* out) {
  if (!plan || !out) return AKM_ERR_INVALID_ARG;
  std::memset(out, 0, sizeof(*out));
  out->n = plan->n;
  out->p = plan->p;
  out->P = plan->P;
  out->N = plan->N;
  out->m = plan->m;
  out->n_g = plan->n_g;
  out->family = plan->family;
  out->sigma_f = plan->sigma_f;
  out->ell = plan->ell;
  out->sigma_eps = plan->sigma_eps;
  for (int w = 0; w < plan->P && w < AKM_MAX_WINDOWS; ++w) {
    const WinGeom& g = plan->tab.w[w];
    out->d[w] = g.d;
    out->c_w[w] = plan->c_w.empty() ? 0.0 : plan->c_w[w];
    out->ell_eff[w] = (plan->c_w.empty() || plan->c_w[w] == 0.0) ? 0.0 : plan->ell / plan->c_w[w];
    out->radius[w] = plan->radius.empty() ? 0.0 : plan->radius[w];
    for (int a = 0; a < 3; ++a) out->box[w][a] = g.L[a];
    out->bin[w] = g.B;
    out->occupied_bins[w] = plan->occupied.empty() ? 0 : plan->occupied[w];
    out->max_bin_points[w] = plan->maxbin.empty() ? 0 : plan->maxbin[w];
  }
  out->work_items_spread = (int64_t)plan->n_items_spread[0];
  out->work_items_interp = (int64_t)plan->n_items_interp[0];
  long long ws = 0;
  const DevBuf* bufs[] = {&plan->Xc, &plan->u_tmp, &plan->u_sorted, &plan->perm, &plan->hist, &plan->grid, &plan->H,
                          &plan->A1, &plan->A2, &plan->A3, &plan->C, &plan->C2, &plan->tw, &plan->D, &plan->part,
                          &plan->items_s[0], &plan->items_i[0], &plan->items_ib[0], &plan->items_s[1],
                          &plan->items_i[1], &plan->items_ib[1]};
  for (const DevBuf* b : bufs) ws += (long long)b->bytes;
  out->workspace_bytes = ws;
  return AKM_OK;
}

}  // extern "C"
