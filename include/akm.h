/*
 * akm.h -- C ABI of the B200-native additive-kernel MVM (NFFT fast summation).
 *
 * The library applies, to an n x r block V, the regularized additive kernel matrix
 *     Khat = sigma_f^2 (K_1 + ... + K_P) + sigma_eps^2 I
 * and its hyperparameter derivatives
 *     dKhat/dell     = sigma_f^2 sum_w K_w^der                             (eq. 2.3)
 *     dKhat/dsigma_f = 2 sigma_f sum_w K_w,  dKhat/dsigma_eps = 2 sigma_eps I ("straightforward")
 * where K_w is the Gaussian or Matern(1/2) sub-kernel (eqs. 1.1/2.2) over
 * feature window W_w of d_w <= 3 coordinates (eq. 2.1).  Each K_w v is evaluated by
 * NFFT fast summation (eq. 3.3): the window's points are scaled into the ball of
 * radius 1/4 - eps_B/2, the kernel is replaced by its truncated Fourier series with the
 * coefficients b_k of eq. (3.2) on N^d frequencies, and the two sums of eq. (3.3)
 * are done by an adjoint NFFT (spreading with a Kaiser-Bessel window onto the oversampled grid
 * of (sigma N)^d points, App. A), a d-dimensional DFT, multiplication by b_k and
 * the window deconvolution, an inverse DFT, and an NFFT (interpolation).  The ell-derivative
 * uses the derivative kernel's coefficients (eq. 3.5).
 *
 * Notation: N = the paper's bandwidth m (Fourier coefficients per axis); m = the paper's window
 * support parameter s (grid cells on each side); sigma_over = the paper's oversampling sigma.
 *
 * Conventions
 *   - All floating point is IEEE float64.  Row-major n x p (X) and n x r (V, Y) blocks.
 *   - Pointers: X, V, Y, dY may be DEVICE pointers (cudaMalloc / torch CUDA tensors) or HOST
 *     pointers (pinned or pageable); host buffers are staged through library-owned device
 *     memory with cudaMemcpyAsync on the given stream (for pageable memory the call returns
 *     after the copies complete).  win_feat / win_len / c_w are always host pointers.
 *   - All calls are stream-ordered on `stream` (a cudaStream_t; NULL = legacy default stream).
 *     set_points / set_theta synchronise `stream` once (they read back small histograms).
 *     The MVM calls are asynchronous for device buffers.
 *   - Ownership: the caller owns X, V, Y, dY and the stream.  The plan owns every workspace
 *     (scaled/sorted coordinates, permutation, grids, spectra, multiplier tables), grows it on
 *     demand, and frees it in akm_destroy.  set_points copies what it needs from X.
 *   - State machine: create -> set_points -> set_theta -> mvm*.  set_points invalidates theta.
 *     MVM calls before both setters return AKM_ERR_STATE.
 *   - Errors are returned synchronously; the message of the last error is akm_last_error().
 *     A device fault surfaces as AKM_ERR_CUDA on the call that observes it.
 *   - A plan is not thread-safe; distinct plans are independent.
 */
#ifndef AKM_H
#define AKM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct akm_plan akm_plan; /* opaque, library-owned */

typedef enum {
  AKM_OK = 0,
  AKM_ERR_INVALID_ARG = 1, /* bad size/stride/window/parameter                              */
  AKM_ERR_NONFINITE = 2,   /* NaN/Inf in X or theta                                          */
  AKM_ERR_STATE = 3,       /* call out of order (e.g. mvm before set_theta)                  */
  AKM_ERR_OOM = 4,         /* device allocation failed                                       */
  AKM_ERR_CUDA = 5,        /* CUDA runtime / kernel error                                    */
  AKM_ERR_UNSUPPORTED = 6  /* legal but not implemented (e.g. window support m not in {4,6,8}) */
} akm_status;

typedef enum { AKM_GAUSSIAN = 0, AKM_MATERN12 = 1 } akm_family;
typedef enum { AKM_D_ELL = 0, AKM_D_SIGMA_F = 1, AKM_D_SIGMA_EPS = 2 } akm_param;

#define AKM_MAX_WINDOWS 32

typedef struct {
  int64_t n;
  int32_t p, P, N, m, n_g;           /* n_g = sigma_over * N (oversampled grid per axis)     */
  int32_t family;
  double sigma_f, ell, sigma_eps;
  int32_t d[AKM_MAX_WINDOWS];        /* window dimensions                                    */
  double c_w[AKM_MAX_WINDOWS];       /* scale factors: x~ = (x - center_w) / c_w             */
  double ell_eff[AKM_MAX_WINDOWS];   /* ell / c_w                                            */
  double radius[AKM_MAX_WINDOWS];    /* R_w = max_i ||x_i^W - center_w||_2 (user units)      */
  int32_t box[AKM_MAX_WINDOWS][3];   /* grid box extent per axis (leading axes 1 if d < 3)   */
  int32_t bin[AKM_MAX_WINDOWS];      /* bin edge (grid cells) used by spreading/interpolation */
  int64_t occupied_bins[AKM_MAX_WINDOWS];
  int64_t max_bin_points[AKM_MAX_WINDOWS];
  int64_t work_items_spread, work_items_interp;
  int64_t workspace_bytes;
} akm_info;

/* Create an empty plan on CUDA device `device`.  *out receives the plan (NULL on error). */
akm_status akm_create(akm_plan** out, int device);

/* Set the points and feature windows (eq. 2.1) and the NFFT parameters.
 *   X        n x p row-major float64, leading dimension ldx >= p (device or host)
 *   win_feat concatenated 0-based feature ids of the P windows (host), win_len[P] in {1,2,3};
 *            windows must be pairwise disjoint and ids in [0, p)
 *   family   AKM_GAUSSIAN (kappa^G) or AKM_MATERN12 (kappa^M)   (eq. 2.2)
 *   N        even >= 4 (bandwidth, paper's m, index set I_N = {-N/2..N/2-1}^d)
 *   sigma_over > 1 with sigma_over*N an even integer n_g (oversampling, App. A)
 *   m        window half-support in grid cells (paper's s); supported: 4, 6, 8; need 4m <= n_g
 *   eps_B    in [0, 1/2): points are scaled into the ball of radius 1/4 - eps_B/2
 * Errors: INVALID_ARG (sizes, windows, parameters), NONFINITE (X), UNSUPPORTED (m), OOM, CUDA.
 * n == 0 is legal (every product is then empty). */
akm_status akm_set_points(akm_plan* plan, const double* X, int64_t n, int32_t p, int64_t ldx,
                          const int32_t* win_feat, const int32_t* win_len, int32_t P, int32_t family,
                          int32_t N, double sigma_over, int32_t m, double eps_B, void* stream);

/* Set theta = (sigma_f, ell, sigma_eps); all must be finite and > 0 (sigma_eps >= 0).
 * Recomputes the per-window scale factors (reading R2), re-bins the points when a
 * scale factor changed, and rebuilds the coefficient tables b_k (eq. 3.2) of kappa and
 * kappa^der at ell_eff = ell / c_w and the multiplier tables (window deconvolution). */
akm_status akm_set_theta(akm_plan* plan, double sigma_f, double ell, double sigma_eps, void* stream);

/* Y = Khat V.  V: n x r (ld ldv >= r), Y: n x r (ld ldy >= r).  r >= 1. */
akm_status akm_kernel_mvm(akm_plan* plan, const double* V, int64_t ldv, int32_t r, double* Y, int64_t ldy,
                          void* stream);

/* dY = (dKhat / d theta_which) V for which in {AKM_D_ELL, AKM_D_SIGMA_F, AKM_D_SIGMA_EPS}. */
akm_status akm_kernel_deriv_mvm(akm_plan* plan, int32_t which, const double* V, int64_t ldv, int32_t r,
                                double* dY, int64_t ldy, void* stream);

/* Fused form sharing spreading and the forward DFT: any of Y, dY_ell, dY_sf may be NULL
 * (at least one non-NULL).  All outputs use the same leading dimension ldy. */
akm_status akm_kernel_mvm_multi(akm_plan* plan, const double* V, int64_t ldv, int32_t r, double* Y,
                                double* dY_ell, double* dY_sf, int64_t ldy, void* stream);

/* Streaming form of akm_kernel_mvm_multi for a sequence of independent batches held in PINNED host
 * memory (the batched K^V throughput of BASELINE.json's metric, fed from the host).  Same operation,
 * arguments and outputs as akm_kernel_mvm_multi; V, Y, dY_ell, dY_sf must be page-locked host
 * buffers (cudaHostAlloc / cudaHostRegister / torch pin_memory), else INVALID_ARG.  The call only
 * enqueues: V goes to one of two library-owned device slots on a copy-in stream, the product runs on
 * `stream` (ordered after earlier work there, so it shares the plan's workspaces safely), and the
 * outputs come back on a copy-out stream.  Consecutive calls therefore overlap batch k's
 * device-to-host copy and batch k+1's host-to-device copy with the products.  Batches under 4 MiB
 * of V (env AKM_PIPE_SPLIT_MIN_BYTES) keep their copies on `stream` (the stream handshakes would
 * cost more than the overlap hides); the call still returns without blocking.  The copy-in is NOT
 * ordered after earlier work on `stream` (only after the product two calls back, which used the same
 * slot): the caller must not write V, nor read or write the outputs, until akm_pipeline_wait.
 * Errors as akm_kernel_mvm_multi. */
akm_status akm_kernel_mvm_pipelined(akm_plan* plan, const double* V, int64_t ldv, int32_t r, double* Y,
                                    double* dY_ell, double* dY_sf, int64_t ldy, void* stream);

/* Make `stream` wait (stream-ordered, no host block) until every akm_kernel_mvm_pipelined call
 * issued so far has finished its copies: after it, synchronising `stream` means the host outputs
 * are complete and the host inputs may be reused.  No-op without pipelined calls. */
akm_status akm_pipeline_wait(akm_plan* plan, void* stream);

/* Cross product for prediction (posterior mean / variance use K_{*X} V,
 * P:947):  Yt = sigma_f^2 sum_w K_w(X_t, X_s) V  (no noise term).
 * The points of the last akm_set_points are read as [sources X_s = rows 0 .. n_src-1; targets
 * X_t = rows n_src .. n-1]: both sets are centred, scaled and binned together (the scaled ball of
 * reading R2 holds the union), so every source-target difference stays inside the torus window.
 * V: n_src x r (ld ldv >= r); Yt: (n - n_src) x r (ld ldy >= r); row-major float64, device or host
 * memory (host buffers are staged).  0 <= n_src <= n, else INVALID_ARG; n_src == n is a no-op;
 * n_src == 0 gives Yt = 0.  The first call with a given n_src re-sorts the points so that every
 * bin holds its sources, then its targets; the product then spreads only the sources and
 * interpolates only at the targets (the square products keep working on the same plan). */
akm_status akm_kernel_cross_mvm(akm_plan* plan, int64_t n_src, const double* V, int64_t ldv, int32_t r,
                                double* Yt, int64_t ldy, void* stream);

/* Plan description (scale factors, grid boxes, bin sizes, workspace). */
akm_status akm_get_info(const akm_plan* plan, akm_info* out);

/* Test hook: freeze the per-window scale factors c_w (host array of P entries) or restore the
 * automatic rule (c_w == NULL).  Takes effect at the next akm_set_theta.  Every frozen c_w must
 * keep all scaled points inside the radius-(1/4 - eps_B/2) ball, else INVALID_ARG. */
akm_status akm_set_scale_override(akm_plan* plan, const double* c_w);

/* Message of the last error on this plan ("" if none).  Valid until the next call. */
const char* akm_last_error(const akm_plan* plan);

/* Free the plan and all its device memory (NULL is a no-op).  Synchronises the device. */
void akm_destroy(akm_plan* plan);

/* Profiling hooks (used by bench.py).  While enabled, every MVM call records CUDA events on the
 * caller's stream around its stages (spreading S2, DFT/multiply/inverse DFT S3-S5,
 * interpolation S6, epilogue S7); akm_get_stage_times synchronises on them and returns the
 * accumulated device milliseconds per stage.  kernel_launches counts the library's own kernel
 * launches issued by MVM calls (always counted).  reset != 0 clears the accumulators. */
typedef struct {
  double spread_ms, fft_ms, interp_ms, epilogue_ms;
  double exchange_ms; /* point-sharded products: akm_spread_grid end -> akm_mvm_from_grid start (the caller's grid all-reduce) */
  int64_t calls;
  int64_t kernel_launches;
  int64_t spread_launches, interp_launches;
} akm_stage_times;
akm_status akm_set_profiling(akm_plan* plan, int32_t enable);
akm_status akm_get_stage_times(akm_plan* plan, akm_stage_times* out, int32_t reset);

/* One evaluation of the preconditioned objective (eq. 1.4) with the diagonal
 * preconditioner M = diag(Khat) = (sigma_f^2 P + sigma_eps^2) I (reading R11):
 *     Z~ = 1/2 ( y^T x + log det M + (1/n_z) sum_i z_i^T logm(M^{-1} Khat) z_i + n log 2 pi ),
 * x = cg_iters steps of preconditioned CG on Khat x = y from x0 = 0, and each
 * quadratic form by stochastic Lanczos quadrature: lanczos_steps steps of Lanczos on
 * M^{-1/2} Khat M^{-1/2} from z_i/||z_i|| with full reorthogonalisation, stopped early on breakdown
 * beta_j <= 1e-12 ||S q_j|| (reading R14), Gauss quadrature ||z_i||^2 sum_j tau_j^2 log theta_j.
 * Every Krylov step is ONE product of Khat with the n x (1 + n_z) block [CG direction | Lanczos
 * vectors] through the NFFT path (reading R11); once the Lanczos steps are done the remaining CG
 * steps multiply the CG column alone (r = 1).
 *   y   n float64 (device or host);  Z  n x n_z row-major probes (ld ldz >= n_z; device or host)
 *   1 <= n_z <= AKM_MAX_PROBES, 0 <= cg_iters <= 1024, 0 <= lanczos_steps <= 64
 *   out (host) receives the terms; cg_relres (host, nullable) receives cg_iters relative residuals
 *   ||y - Khat x_t|| / ||y|| (recursively updated).
 * Synchronises `stream` before returning.  Workspace: about (lanczos_steps + 4) n (1 + n_z)
 * doubles on top of the product's.  Errors: STATE, INVALID_ARG, OOM, CUDA; a non-positive Ritz
 * value or a non-converged tridiagonal eigensolve returns AKM_ERR_NONFINITE. */
#define AKM_MAX_PROBES 31
typedef struct {
  double Z;                       /* Z~(theta), eq. 1.4                                      */
  double quad;                    /* y^T x                                                    */
  double logdet_M;                /* n log(sigma_f^2 P + sigma_eps^2)                        */
  double slq;                     /* (1/n_z) sum_i samples[i]                                 */
  double n_log_2pi;               /* n log 2 pi                                               */
  double samples[AKM_MAX_PROBES]; /* z_i^T logm(M^{-1} Khat) z_i estimates                    */
  int32_t steps[AKM_MAX_PROBES];  /* Lanczos steps used per probe (< lanczos_steps on breakdown) */
  int32_t n_z, cg_iters, lanczos_steps, products; /* products = Khat block products issued    */
  double cg_relres;               /* final recursive relative residual (of the preconditioned
                                     system S_op x^ = U^{-1} y under AAFN)                     */
  double cg_relres_true;          /* ||y - Khat x|| / ||y|| of the returned CG iterate (one extra
                                     r = 1 product)                                             */
  int32_t landmarks;              /* AAFN landmark count k (0: diagonal preconditioner)          */
  int64_t product_columns;        /* columns multiplied over all products (after the Lanczos
                                     steps only the CG column is multiplied: r = 1)             */
} akm_objective_out;
akm_status akm_objective_diag(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                              int32_t cg_iters, int32_t lanczos_steps, akm_objective_out* out, double* cg_relres,
                              void* stream);

/* ------------------------------------------------------------------ point sharding
 * The product is a sum over points (eq. 3.3: a_k = sum_j v_j e^{-2 pi i k.x_j}), so G
 * processes that each hold a disjoint row block of X and V can each spread their own points onto
 * the SAME oversampled grids, sum the grids (one all-reduce, done by the caller, e.g. NCCL), and
 * each run the DFT / multiply / inverse DFT on the summed grids and interpolate at their own points.
 * For the grids to coincide every shard must use the union's window frame:
 *   1. akm_set_points(local rows);  akm_get_bounds -> all-reduce MIN(lo), MAX(hi) over the shards;
 *   2. akm_set_bounds(global lo, hi) -> this shard's radius about the union's centers;
 *      all-reduce MAX(radius);  akm_set_radius(global radius);
 *   3. akm_set_theta on every shard; every shard must end with the same bin edges (akm_get_info .bin):
 *      otherwise pin them with akm_set_bin_override and call akm_set_theta again;
 *   4. per product: akm_spread_grid(local V, grid) -> all-reduce SUM(grid) -> akm_mvm_from_grid.
 * Each shard needs n >= 1.  These calls take DEVICE pointers only. */

/* Bounding box of this plan's points per window and padded axis: lo, hi host arrays of 3P doubles
 * ([w*3 + a]; the leading 3 - d_w axes are singletons and read 0).  n == 0 gives +inf / -inf.
 * Errors: INVALID_ARG, STATE (before set_points). */
akm_status akm_get_bounds(const akm_plan* plan, double* lo, double* hi);

/* Replace the bounding box by the union's (lo, hi as in akm_get_bounds; must contain this plan's
 * points), move the window centers to its midpoints (reading R2) and return in radius_local (host,
 * P doubles) the max distance of this plan's points from them.  Invalidates theta.  Synchronises. */
akm_status akm_set_bounds(akm_plan* plan, const double* lo, const double* hi, double* radius_local, void* stream);

/* Set the radius R_w used by the scale rule (reading R2) to the union's (host, P doubles, each >= this
 * plan's own radius, else INVALID_ARG).  Invalidates theta. */
akm_status akm_set_radius(akm_plan* plan, const double* radius);

/* Force the bin edge B of every window (host, P entries in {1,2,3,4,6,8}) instead of the cost model's
 * choice, or restore the choice (bins == NULL).  A forced B that does not fit the grid box makes the
 * next akm_set_theta fail with UNSUPPORTED.  Invalidates theta. */
akm_status akm_set_bin_override(akm_plan* plan, const int32_t* bins);

/* Number of doubles of the grids of one product with r right-hand sides (after set_theta). */
akm_status akm_grid_size(const akm_plan* plan, int32_t r, int64_t* count);

/* S2 only: zero `grid` (device, akm_grid_size doubles, caller-owned) and spread this plan's points
 * with weights V (device, n x r, ld ldv >= r) onto it (adjoint NFFT, App. A). */
akm_status akm_spread_grid(akm_plan* plan, const double* V, int64_t ldv, int32_t r, double* grid, void* stream);

/* S3-S7 from a complete (summed) grid: DFT, multiply by the multipliers, inverse DFT, interpolation at
 * this plan's points and the epilogue of akm_kernel_mvm_multi (V, the same local block, gives the
 * noise term).  Outputs as in akm_kernel_mvm_multi, device memory. */
akm_status akm_mvm_from_grid(akm_plan* plan, const double* grid, const double* V, int64_t ldv, int32_t r, double* Y,
                             double* dY_ell, double* dY_sf, int64_t ldy, void* stream);

/* Boundary-regularised kernel kappa_R (eq. 3.1 "a smooth or at least continuous
 * periodic function kappa_R"; "It is possible to smoothen the inner or outer boundaries",
 * P:155).  With p > 0 the b_k of eq. (3.2) are taken from the samples of
 *   kappa_R(r) = T_I(r) (r <= eps_I) | kappa(r) | T_B(r) (1/2 - eps_B < r <= 1/2) | kappa(1/2) (r > 1/2),
 * r = ||x~|| in every window's scaled coordinates, T_I / T_B the two-point Taylor interpolants of
 * degree 2p - 1 (kappa's derivatives 0..p-1 at +-eps_I; at 1/2 - eps_B and a flat kappa(1/2) at 1/2;
 * eps_B is set_points'), and the products add the near-field correction
 * sum_{||x~_i - x~_j|| < eps_I} (kappa - T_I)(||x~_i - x~_j||) v_j (and the same for kappa^der), so
 * they still approximate the plain kernel sums -- with the Matern cusp removed from the truncated
 * Fourier series.  p = 0 (default after set_points) is the paper's implementation (no smoothing).
 * eps_I in [0, 1/4), 0 <= p <= 8; eps_I = 0 keeps only the outer part.  Invalidates theta.  The
 * near-field correction is built for the square products (akm_kernel_mvm*, the Krylov drivers);
 * akm_kernel_cross_mvm and akm_mvm_from_grid return UNSUPPORTED while eps_I > 0. */
akm_status akm_set_regularization(akm_plan* plan, double eps_I, int32_t p);

/* Deterministic products (SURVEY.md §4 tier 3).  on != 0: every product (and so every Krylov driver
 * result) is bitwise reproducible from run to run on the same GPU model.  The only order-dependent
 * sums on the path are the spreading's footprint flushes (float64 atomics, reading R13);
 * in this mode they add v * 2^S_c as three signed 40-bit integer limbs with 64-bit integer atomics
 * (exact and associative; S_c = 112 - ceil(log2(rows * max_j |v_jc|)) per RHS column, resolution
 * ~1e-34 of the column's scale) and one pass converts the limb sums to float64.  The bin sort,
 * the DFTs, the interpolation, the epilogue and the Krylov reductions are order-fixed already.
 * Results differ from the default mode by rounding only.  on = 0 (default): float64 atomics. */
akm_status akm_set_deterministic(akm_plan* plan, int32_t on);

/* Test hook: the window polynomials the kernels evaluate.  For tap o in [0, 2m) of a
 * point with fractional grid position t = u - floor(u), the Kaiser-Bessel weight (App. A,
 * P:1240-1247) phi((t + m - 1 - o) / n_g) is replaced by sum_k coef[o*(degree+1) + k] x^k with
 * x = 2t - 1 (the degree-14 Chebyshev interpolant on t in [0, 1], built in akm_set_points).
 * coef: host array of at least 16 * 15 doubles (output); *taps = 2m, *degree = 14.
 * Errors: INVALID_ARG (NULL), STATE (before akm_set_points). */
akm_status akm_get_window_poly(const akm_plan* plan, double* coef, int32_t* taps, int32_t* degree);

/* ------------------------------------------------------------------ AAFN preconditioner
 * PAPER.md §2.3: landmarks by farthest point sampling per feature window, merged; the
 * landmark block Cholesky-factored and the Schur complement approximated by its inverse factor
 * (reading R15; the FSAI factor G is built with the diagonal pattern, G = diag(S_aa^{-1/2})):
 *     M = U U^T,  U = [L11, 0; K21 L11^{-T}, G^{-1}],  log det M = 2 sum log diag L11 - 2 sum log diag G.
 * k_per_window = 0 selects the diagonal preconditioner M = diag(Khat) (default); otherwise FPS picks
 * min(k_per_window, n) points per window (seed: farthest from the window centroid; then the point
 * farthest from the picks; ties to the lowest index), duplicates removed in pick order; at most 800
 * landmarks in total (UNSUPPORTED beyond).  Landmarks depend on the points only; the factors are
 * rebuilt lazily after every akm_set_theta. */
akm_status akm_set_preconditioner(akm_plan* plan, int32_t k_per_window);

/* out = U^{-1} T (transpose = 0) or U^{-T} T (transpose != 0) for the current theta, T and out n x r
 * row-major device blocks (1 <= r <= 32); logdet (host, nullable) receives log det M, landmarks (host,
 * nullable, akm_precond_landmarks entries) the landmark row indices in merge order.  M^{-1} = U^{-T} U^{-1}.
 * Errors: STATE (no AAFN set / before set_theta), INVALID_ARG, NONFINITE (Cholesky breakdown after one
 * jitter retry of 1e-10 trace(K11)/k), UNSUPPORTED, OOM, CUDA. */
akm_status akm_precond_apply(akm_plan* plan, int32_t transpose, const double* T, int32_t r, double* out, double* logdet,
                             int32_t* landmarks, void* stream);

/* Number of AAFN landmarks for the current points (runs FPS if needed). */
akm_status akm_precond_landmarks(akm_plan* plan, int32_t* count, void* stream);

/* akm_objective_diag with the plan's preconditioner (akm_set_preconditioner): with AAFN, CG and
 * Lanczos run on the split-preconditioned S_op = U^{-1} Khat U^{-T}: column 0 carries
 * U^{-1} y (PCG on Khat x = y), columns 1.. the probes z_i (tr logm(M^{-1} Khat) = tr logm(S_op)), and
 * log det M is AAFN's.  Same arguments and outputs as akm_objective_diag. */
akm_status akm_objective(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z, int32_t cg_iters,
                         int32_t lanczos_steps, akm_objective_out* out, double* cg_relres, void* stream);

/* Library version string. */
/* Gradient of the objective Z~ (eq. (div)) with M = diag(Khat) = c I,
 * c = sigma_f^2 P + sigma_eps^2 (reading R11):
 *   grad[k] = dZ~/dtheta_k ~= 1/2 ( -alpha^T dKhat_k alpha + tr(M^{-1} dM_k)
 *             + (1/n_z) sum_i z_i^T (M^{-1} Khat)^{-1} d(M^{-1} Khat)_k z_i ),  theta = (sigma_f, ell, sigma_eps),
 * where (M^{-1} Khat)^{-1} d(M^{-1} Khat)_k = Khat^{-1} dKhat_k - (dc_k / c) I and, Khat being
 * symmetric, z^T Khat^{-1} dKhat_k z = (Khat^{-1} z)^T (dKhat_k z).  alpha = Khat^{-1} y and
 * Khat^{-1} z_i come from cg_iters iterations of PCG (x0 = 0, M = c I) run on the n x (1 + n_z) block
 * [y | Z] through the NFFT product; then one fused derivative product (dKhat/dell, dKhat/dsigma_f)
 * on [alpha | Z] and column dot products on the device; the three sums are combined on the host.
 * y: n; Z: n x n_z row-major (ld ldz >= n_z); device or host.  grad: host double[3] (output).
 * cg_relres: optional host double[cg_iters] (column 0 relative residual per iteration, -1 if not
 * run).  1 <= n_z <= AKM_MAX_PROBES, 0 <= cg_iters <= 1024.  Products: cg_iters + 1. */
akm_status akm_gradient_diag(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                             int32_t cg_iters, double* grad, double* cg_relres, void* stream);

/* akm_gradient_diag with the plan's preconditioner (akm_set_preconditioner).  With AAFN the block CG
 * runs on S_op = U^{-1} Khat U^{-T} from U^{-1} [y | Z] and the solutions are mapped back by U^{-T};
 * eq. (div)'s control-variate term needs dM/dtheta, which AAFN does not define, so
 * the plain Hutchinson form is returned (reading R15):
 *   grad[k] = 1/2 ( -alpha^T dKhat_k alpha + (1/n_z) sum_i (Khat^{-1} z_i)^T dKhat_k z_i ).
 * cg_relres then holds the preconditioned system's residuals.  Same arguments as akm_gradient_diag. */
akm_status akm_gradient(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z, int32_t cg_iters,
                        double* grad, double* cg_relres, void* stream);

/* The raw per-column terms of the gradient (for probe sharding): with
 * R = 1 + n_z, X = Khat^{-1} [y | Z] from cg_iters CG iterations (preconditioned != 0: the plan's
 * preconditioner, else M = diag Khat), dots[k*R + i] = X_i^T (dKhat_k B_i) with B = [X_0 | Z] (i = 0:
 * alpha^T dKhat_k alpha; i >= 1: (Khat^{-1} z_i)^T dKhat_k z_i), k in (sigma_f, ell, sigma_eps), and
 * sqnorms[i] = ||b_i||^2 (host arrays of 3R and R doubles).  akm_gradient_diag combines them as
 *   grad[k] = 1/2 ( -dots[k*R] + n dc_k/c + (1/n_z) sum_{i>=1} (dots[k*R+i] - dc_k/c sqnorms[i]) ),
 * c = sigma_f^2 P + sigma_eps^2, dc = (2 sigma_f P, 0, 2 sigma_eps) (dc = 0 under AAFN). */
akm_status akm_gradient_columns(akm_plan* plan, const double* y, const double* Z, int64_t ldz, int32_t n_z,
                                int32_t cg_iters, int32_t preconditioned, double* dots, double* sqnorms,
                                double* cg_relres, void* stream);

const char* akm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AKM_H */
