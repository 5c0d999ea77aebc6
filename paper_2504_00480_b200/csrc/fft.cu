// fft.cu -- the d-dimensional DFT stage of the fast summation.
//
// For every window and RHS the spread grid g (box-local, real) is transformed to the
// frequencies the method keeps, multiplied by the Fourier multiplier D (b_k of eq. 3.2 times
// the window deconvolution and the Nyquist weights, see setup_kernels.cu) and transformed back
// onto the box (App. A; eq. 3.3):
//
//   h_l = sum_{k in S} D_k e^{2 pi i k.l/n_g} sum_{l'} g_{l'} e^{-2 pi i k.l'/n_g},
//   S = {-N/2..N/2}^d  (pruned: only these (N+1)^d of the n_g^d frequencies are nonzero),
//
// evaluated separably as six passes of small dense DFT matrices along one axis each:
//   FA  last axis, real -> half spectrum k2 in 0..N/2        A1[l0][l1][k2]
//   FB  middle axis                                           A2[l0][k1][k2]
//   FC1 first axis                                            A3[k0][k1][k2]
//   FC2 multiply by D_op and inverse first axis               C [op][l0][k1][k2]
//   FD  inverse middle axis                                   C2[op][l0][l1][k2]
//   FE  inverse last axis, Hermitian half-sum (k2 = 0 once, k2 > 0 twice, real part)
// Only the box (nodes any point can touch) is transformed in and out, so the zero padding of
// the oversampled grid and the frequencies outside S cost nothing.  Singleton (padded) axes
// have one node and k = 0 with twiddle 1.
//
// Every pass is the same batched operation Y[o][k][i] = sum_l M[k][l] X[o][l][i] (o = outer
// index, i = inner index incl. the RHS), run by one kernel body: a CTA stages the L inputs of 32
// consecutive columns (o, i) in shared memory with one read of each input, then each thread
// produces outputs (k, column) with broadcast twiddle reads.  (The first version computed every
// output straight from global memory and was latency-bound: profiles/r01_launches_c2_summary.txt.)
#include <algorithm>

#include <cstdlib>

#include "akm_internal.cuh"

namespace akm {


constexpr int kDftThreads = 256;

enum DftMode { kFA = 0, kFB, kFC1, kFC2, kFD, kFE };

struct DftShape {
  long long O, I;       // outer / inner extents (inner includes the RHS index)
  int L, K;             // input length along the axis, output length
  long long xo, xl;     // input strides (elements) of o and l; inner stride 1
  long long yo, yk;     // output strides of o and k; inner stride 1
};

__host__ __device__ inline DftShape dft_shape(const WinGeom& g, int mode, int r, int ops) {
  DftShape s;
  const long long R = r;
  switch (mode) {
    case kFA:   // G[(l0,l1)][l2][c] (real) -> A1[(l0,l1)][k2][c]
      s.O = (long long)g.L[0] * g.L[1]; s.I = R; s.L = g.L[2]; s.K = g.K[2];
      s.xo = (long long)g.L[2] * R; s.xl = R; s.yo = (long long)g.K[2] * R; s.yk = R;
      break;
    case kFB:   // A1[l0][l1][(k2,c)] -> A2[l0][k1][(k2,c)]
      s.O = g.L[0]; s.I = (long long)g.K[2] * R; s.L = g.L[1]; s.K = g.K[1];
      s.xo = (long long)g.L[1] * s.I; s.xl = s.I; s.yo = (long long)g.K[1] * s.I; s.yk = s.I;
      break;
    case kFC1:  // A2[l0][(k1,k2,c)] -> A3[k0][(k1,k2,c)]
      s.O = 1; s.I = (long long)g.K[1] * g.K[2] * R; s.L = g.L[0]; s.K = g.K[0];
      s.xo = 0; s.xl = s.I; s.yo = 0; s.yk = s.I;
      break;
    case kFC2:  // D_op A3[k0][(k1,k2,c)] -> C[op][l0][(k1,k2,c)]   (o = op)
      s.O = ops; s.I = (long long)g.K[1] * g.K[2] * R; s.L = g.K[0]; s.K = g.L[0];
      s.xo = 0; s.xl = s.I; s.yo = (long long)g.L[0] * s.I; s.yk = s.I;
      break;
    case kFD:   // C[(op,l0)][k1][(k2,c)] -> C2[(op,l0)][l1][(k2,c)]
      s.O = (long long)ops * g.L[0]; s.I = (long long)g.K[2] * R; s.L = g.K[1]; s.K = g.L[1];
      s.xo = (long long)g.K[1] * s.I; s.xl = s.I; s.yo = (long long)g.L[1] * s.I; s.yk = s.I;
      break;
    default:    // kFE: C2[(op,line)][k2][c] -> H[(line, l2)][op][c] (real)
      s.O = (long long)ops * g.L[0] * g.L[1]; s.I = R; s.L = g.K[2]; s.K = g.L[2];
      s.xo = (long long)g.K[2] * R; s.xl = R; s.yo = 0; s.yk = 0;  // output indexed explicitly
      break;
  }
  return s;
}

template <int MODE, int kDftCols>
__global__ void __launch_bounds__(kDftThreads) k_dft_axis(const WinTable* __restrict__ tabp, const void* __restrict__ Xv,
                                                          void* __restrict__ Yv, const double2* __restrict__ tw,
                                                          const double* __restrict__ D, int dslot0, int r, int ops) {
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[blockIdx.y];
  const DftShape sh = dft_shape(g, MODE, r, ops);
  const long long ncol = sh.O * sh.I;
  const long long col0 = (long long)blockIdx.x * kDftCols;
  if (col0 >= ncol) return;
  extern __shared__ double2 xs[];  // [L][kDftCols]
  const int tid = threadIdx.x;

  long long xbase, ybase;  // window-relative base offsets (elements)
  switch (MODE) {
    case kFA: xbase = g.tap_off * r; ybase = g.a1_off * r; break;
    case kFB: xbase = g.a1_off * r; ybase = g.a2_off * r; break;
    case kFC1: xbase = g.a2_off * r; ybase = g.a3_off * r; break;
    case kFC2: xbase = g.a3_off * r; ybase = g.c_off * r; break;
    case kFD: xbase = g.c_off * r; ybase = g.c2_off * r; break;
    default: xbase = g.c2_off * r; ybase = g.tap_off * (long long)ops * r; break;
  }
  // twiddle table of the transformed axis: T[k][l] = e^{-2 pi i k (box_lo + l) / n_g}, [K][L]
  const int axis = (MODE == kFA || MODE == kFE) ? 2 : (MODE == kFB || MODE == kFD) ? 1 : 0;
  const double2* T = tw + g.tw_off[axis];
  const int Lt = g.L[axis];  // row length of the table

  // stage the inputs X[o][l][i] of the CTA's columns (FC2: with D_op applied)
  const long long kk = (long long)g.K[1] * g.K[2];
  const long long dper = (long long)g.K[0] * kk;
  for (int idx = tid; idx < sh.L * kDftCols; idx += kDftThreads) {
    const int l = idx / kDftCols, j = idx - l * kDftCols;
    const long long col = col0 + j;
    double2 v = make_double2(0.0, 0.0);
    if (col < ncol) {
      const long long o = col / sh.I, i = col - o * sh.I;
      const long long off = xbase + o * sh.xo + (long long)l * sh.xl + i;
      if (MODE == kFA) {
        v.x = static_cast<const double*>(Xv)[off];
      } else {
        v = static_cast<const double2*>(Xv)[off];
      }
      if (MODE == kFC2) {  // multiplier D_op[k0 = l][(k1,k2) = i / r]
        const double dd = D[g.d_off + (dslot0 + o) * dper + (long long)l * kk + i / r];
        v.x *= dd;
        v.y *= dd;
      }
    }
    xs[idx] = v;
  }
  __syncthreads();

  // outputs (k, column): a warp shares k (broadcast twiddles), lanes take consecutive columns
  const int j = tid % kDftCols;
  const long long col = col0 + j;
  if (col >= ncol) return;
  const long long o = col / sh.I, i = col - o * sh.I;
  for (int k = tid / kDftCols; k < sh.K; k += kDftThreads / kDftCols) {
    // four interleaved partial sums over l (independent FMA chains)
    double re4[4] = {0.0, 0.0, 0.0, 0.0}, im4[4] = {0.0, 0.0, 0.0, 0.0};
    if (MODE == kFA || MODE == kFB || MODE == kFC1) {  // forward: M[k][l] = T[k][l]
      const double2* Tk = T + (long long)k * Lt;
      int l = 0;
      for (; l + 4 <= sh.L; l += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 t = Tk[l + q], x = xs[(l + q) * kDftCols + j];
          re4[q] = fma(t.x, x.x, fma(-t.y, x.y, re4[q]));
          im4[q] = fma(t.x, x.y, fma(t.y, x.x, im4[q]));
        }
      }
      for (; l < sh.L; ++l) {
        const double2 t = Tk[l], x = xs[l * kDftCols + j];
        re4[0] = fma(t.x, x.x, fma(-t.y, x.y, re4[0]));
        im4[0] = fma(t.x, x.y, fma(t.y, x.x, im4[0]));
      }
    } else {  // inverse: M[k][l] = conj(T[l][k]) (k indexes nodes, l frequencies)
      int l = 0;
      for (; l + 4 <= sh.L; l += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 t = T[(long long)(l + q) * Lt + k], x = xs[(l + q) * kDftCols + j];
          if (MODE == kFE) {
            const double w = (l + q == 0) ? 1.0 : 2.0;  // Hermitian half-sum, real part
            re4[q] = fma(w, fma(t.x, x.x, t.y * x.y), re4[q]);
          } else {
            re4[q] = fma(t.x, x.x, fma(t.y, x.y, re4[q]));
            im4[q] = fma(t.x, x.y, fma(-t.y, x.x, im4[q]));
          }
        }
      }
      for (; l < sh.L; ++l) {
        const double2 t = T[(long long)l * Lt + k], x = xs[l * kDftCols + j];
        if (MODE == kFE) {
          const double w = (l == 0) ? 1.0 : 2.0;
          re4[0] = fma(w, fma(t.x, x.x, t.y * x.y), re4[0]);
        } else {
          re4[0] = fma(t.x, x.x, fma(t.y, x.y, re4[0]));
          im4[0] = fma(t.x, x.y, fma(-t.y, x.x, im4[0]));
        }
      }
    }
    const double re = (re4[0] + re4[1]) + (re4[2] + re4[3]);
    const double im = (im4[0] + im4[1]) + (im4[2] + im4[3]);
    if (MODE == kFE) {
      // H[(line * L2 + l2) * ops + op][c] with o = op * lines + line
      const long long lines = (long long)g.L[0] * g.L[1];
      const long long op = o / lines, line = o - op * lines;
      static_cast<double*>(Yv)[ybase + ((line * g.L[2] + k) * ops + op) * r + i] = re;
    } else {
      static_cast<double2*>(Yv)[ybase + o * sh.yo + (long long)k * sh.yk + i] = make_double2(re, im);
    }
  }
}

// ---------------------------------------------------------------- DMMA passes (kFB, kFD)
// The complex axis-1 passes of the generic path as FP64 tensor-core GEMMs (large 2-D boxes, c3):
// Y_o[k][i] = sum_l M[k][l] X_o[l][i] with M = T (kFB) or M[k][l] = conj(T[l][k]) (kFD), computed
// as the real product C (2K x I) = A (2K x 2L) B (2L x I): A is the 2x2 real block form of M
// (rows 2k + q: component q of the output; columns 2l + p: component p of the input), B's row
// 2l + p holds component p of X[l][i].  A CTA owns 16 complex rows x 64 columns (2x2 warps of
// 2x4 DMMA tiles); the K loop stages 16 complex l per chunk, double-buffered: the global loads of
// chunk c + 1 are issued into registers before the MMAs of chunk c, so their L2 latency hides
// under the MMAs (the first version staged 8 l synchronously and stalled on every load).
constexpr int kMmaK = 16;  // complex l per staged chunk (32 real k)
constexpr int kMmaTM = 2, kMmaTN = 4;  // DMMA tiles per warp along m and n (2 x 2 warps per CTA)
constexpr int kMmaRows = 2 * kMmaTM * 8, kMmaCols = 2 * kMmaTN * 8;  // real rows / columns per CTA
constexpr int kMmaXE = kMmaK * kMmaCols / 128, kMmaME = (kMmaRows / 2) * kMmaK / 128;  // loads per thread
constexpr int kMmaLdB = kMmaCols + 4, kMmaLdA = 2 * kMmaK + 4;  // smem row strides (= 4 mod 16)
constexpr size_t kMmaSmem = sizeof(double) * (2 * 2 * kMmaK * kMmaLdB + 2 * kMmaRows * kMmaLdA);
// FUSED_D (kFD, every window without an axis 0): the input is A2 itself times the multiplier
// D_op[k0 = 0][k1][k2] (the FC1 copy and the FC2 multiply folded into the load).
template <int MODE, bool FUSED_D = false>
__global__ void __launch_bounds__(128) k_dft_mma(const WinTable* __restrict__ tabp, const double2* __restrict__ X,
                                                 double2* __restrict__ Y, const double2* __restrict__ tw, int r,
                                                 int ops, int ktiles, const double* __restrict__ D = nullptr,
                                                 int dslot0 = 0) {
  constexpr int CK = kMmaRows / 2;  // complex rows per CTA
  const WinGeom& g = tabp->w[blockIdx.z];
  const DftShape sh = dft_shape(g, MODE, r, ops);
  const int o = blockIdx.y / ktiles, kt = blockIdx.y - o * ktiles;
  const long long i0 = (long long)blockIdx.x * kMmaCols;
  const int k0 = kt * CK;
  if (o >= sh.O || i0 >= sh.I || k0 >= sh.K) return;
  const long long xbase = FUSED_D ? g.a2_off * r : (MODE == kFB ? g.a1_off : g.c_off) * r + (long long)o * sh.xo;
  const long long dbase = g.d_off + (long long)(dslot0 + o) * g.K[0] * g.K[1] * g.K[2];  // FUSED_D: o = op
  const long long ybase = (MODE == kFB ? g.a2_off : g.c2_off) * r + (long long)o * sh.yo;
  const double2* T = tw + g.tw_off[1];
  const int Lt = g.L[1];
  // operands stored in their real form, so a fragment is one 8-byte load: Br[2l + p][col] = component
  // p of X[l][col], Ar[2k + q][2l + p] = the 2x2 real block of M[k][l]; row strides = 4 (mod 16)
  extern __shared__ __align__(16) double dft_sm[];
  double* Br = dft_sm;                               // [2][2 kMmaK][kMmaLdB]
  double* Ar = dft_sm + 2 * 2 * kMmaK * kMmaLdB;     // [2][kMmaRows][kMmaLdA]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, wm = warp >> 1, wn = warp & 1;
  double acc[kMmaTM][kMmaTN][2];
#pragma unroll
  for (int a = 0; a < kMmaTM; ++a)
#pragma unroll
    for (int b = 0; b < kMmaTN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // raw values only (no arithmetic on them here: the loads stay in flight under the MMAs of the
  // current chunk; the multiplier and the conjugation are applied when they are stored)
  double2 xr[kMmaXE], mr[kMmaME];
  double dr[FUSED_D ? kMmaXE : 1];
  auto gload = [&](int l0) {
#pragma unroll
    for (int e = 0; e < kMmaXE; ++e) {
      const int idx = tid + 128 * e, l = idx / kMmaCols, j = idx - l * kMmaCols;
      const long long i = i0 + j;
      double2 v = make_double2(0.0, 0.0);
      double dd = 0.0;
      if (l0 + l < sh.L && i < sh.I) {
        v = X[xbase + (long long)(l0 + l) * sh.xl + i];
        if (FUSED_D) dd = D[dbase + (long long)(l0 + l) * g.K[2] + (int)i / r];  // D_op[k1 = l][k2 = i / r]
      }
      xr[e] = v;
      if constexpr (FUSED_D) dr[e] = dd;
    }
#pragma unroll
    for (int e = 0; e < kMmaME; ++e) {
      const int idx = tid + 128 * e, k = idx / kMmaK, l = idx - k * kMmaK;
      double2 m = make_double2(0.0, 0.0);
      if (k0 + k < sh.K && l0 + l < sh.L)
        m = (MODE == kFB) ? T[(long long)(k0 + k) * Lt + l0 + l] : T[(long long)(l0 + l) * Lt + k0 + k];
      mr[e] = m;
    }
  };
  gload(0);
  for (int l0 = 0, c = 0; l0 < sh.L; l0 += kMmaK, ++c) {
    const int buf = c & 1;
#pragma unroll
    for (int e = 0; e < kMmaXE; ++e) {
      const int idx = tid + 128 * e, l = idx / kMmaCols, j = idx - l * kMmaCols;
      double2 v = xr[e];
      if constexpr (FUSED_D) {
        v.x *= dr[e];
        v.y *= dr[e];
      }
      double* bb = Br + (buf * 2 * kMmaK + 2 * l) * kMmaLdB + j;
      bb[0] = v.x;
      bb[kMmaLdB] = v.y;
    }
#pragma unroll
    for (int e = 0; e < kMmaME; ++e) {
      const int idx = tid + 128 * e, k = idx / kMmaK, l = idx - k * kMmaK;
      const double2 m = (MODE == kFB) ? mr[e] : make_double2(mr[e].x, -mr[e].y);  // kFD: conj(T[l][k])
      double* ab = Ar + (buf * kMmaRows + 2 * k) * kMmaLdA + 2 * l;
      ab[0] = m.x;
      ab[1] = -m.y;
      ab[kMmaLdA] = m.y;
      ab[kMmaLdA + 1] = m.x;
    }
    __syncthreads();  // chunk c visible; buffer buf ^ 1 (chunk c - 1) free for the next store
    if (l0 + kMmaK < sh.L) gload(l0 + kMmaK);
#pragma unroll
    for (int ks = 0; ks < 2 * kMmaK / 4; ++ks) {
      const int kr = ks * 4 + (lane & 3);
      double af[kMmaTM], bf[kMmaTN];
#pragma unroll
      for (int mt = 0; mt < kMmaTM; ++mt)
        af[mt] = Ar[(buf * kMmaRows + (wm * kMmaTM + mt) * 8 + (lane >> 2)) * kMmaLdA + kr];
#pragma unroll
      for (int nt = 0; nt < kMmaTN; ++nt)
        bf[nt] = Br[(buf * 2 * kMmaK + kr) * kMmaLdB + (wn * kMmaTN + nt) * 8 + (lane >> 2)];
#pragma unroll
      for (int mt = 0; mt < kMmaTM; ++mt)
#pragma unroll
        for (int nt = 0; nt < kMmaTN; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
  }
  // rows 2k (real) and 2k + 1 (imaginary) sit in lanes l and l ^ 4
#pragma unroll
  for (int mt = 0; mt < kMmaTM; ++mt) {
    const int row = (wm * kMmaTM + mt) * 8 + (lane >> 2), k = k0 + (row >> 1);
#pragma unroll
    for (int nt = 0; nt < kMmaTN; ++nt) {
      const double im0 = __shfl_xor_sync(0xffffffffu, acc[mt][nt][0], 4);
      const double im1 = __shfl_xor_sync(0xffffffffu, acc[mt][nt][1], 4);
      if ((row & 1) || k >= sh.K) continue;
      const long long i = i0 + (wn * kMmaTN + nt) * 8 + 2 * (lane & 3);
      if (i < sh.I) Y[ybase + (long long)k * sh.yk + i] = make_double2(acc[mt][nt][0], im0);
      if (i + 1 < sh.I) Y[ybase + (long long)k * sh.yk + i + 1] = make_double2(acc[mt][nt][1], im1);
    }
  }
}

template <int MODE, bool FUSED_D = false>
static cudaError_t launch_dft_mma(const WinTable& tab, const WinTable* dtab, const double2* X, double2* Y,
                                  const double2* tw, int r, int ops, cudaStream_t s, const double* D = nullptr,
                                  int dslot0 = 0) {
  long long itiles = 1, O = 1;
  int ktiles = 1;
  for (int w = 0; w < tab.P; ++w) {
    const DftShape sh = dft_shape(tab.w[w], MODE, r, ops);
    itiles = std::max(itiles, (sh.I + kMmaCols - 1) / kMmaCols);
    O = std::max(O, sh.O);
    ktiles = std::max(ktiles, (sh.K + kMmaRows / 2 - 1) / (kMmaRows / 2));
  }
  static std::atomic<unsigned long long> attr{0};
  if (!optin_done(attr)) {
    cudaError_t e = cudaFuncSetAttribute(k_dft_mma<MODE, FUSED_D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kMmaSmem);
    if (e != cudaSuccess) return e;
    optin_mark(attr);
  }
  k_dft_mma<MODE, FUSED_D><<<dim3((unsigned)itiles, (unsigned)(O * ktiles), tab.P), 128, kMmaSmem, s>>>(
      dtab, X, Y, tw, r, ops, ktiles, D, dslot0);
  return cudaGetLastError();
}

// The real-side axis-2 passes (kFA: real grid -> half spectrum; kFE: half spectrum -> real H with
// the Hermitian weights) as FP64 tensor-core GEMMs over the columns (o, c):
//   kFA:  C[2k + q][(o, c)] = sum_l  {Re, Im} T[k][l] * x[o][l][c]
//   kFE:  C[l][(o, c)]      = sum_{k, p} w_k {Re, Im} T[k][l] * {Re, Im} X[o][k][c]   (w_0 = 1, else 2)
// A CTA owns 32 real rows x 64 columns (2x2 warps of 2x4 DMMA tiles); K is staged 16 (complex for
// kFE) at a time, double-buffered through registers like k_dft_mma.
constexpr int kMrK = 16, kMrCols = 64;
template <int MODE>
__global__ void __launch_bounds__(128) k_dft_mma_r(const WinTable* __restrict__ tabp, const void* __restrict__ Xv,
                                                   void* __restrict__ Yv, const double2* __restrict__ tw, int r,
                                                   int ops) {
  constexpr int XE = kMrK * kMrCols / 128, ME = 32 * kMrK / 128;
  const WinGeom& g = tabp->w[blockIdx.z];
  const DftShape sh = dft_shape(g, MODE, r, ops);
  const long long ncol = sh.O * sh.I, c0 = (long long)blockIdx.x * kMrCols;
  const int rows = (MODE == kFA) ? 2 * sh.K : sh.K;  // real output rows
  const int row0 = blockIdx.y * 32;
  if (c0 >= ncol || row0 >= rows) return;
  const double2* T = tw + g.tw_off[2];
  const int Lt = g.L[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, wm = warp >> 1, wn = warp & 1;
  __shared__ double2 Xs[2][kMrK][kMrCols];  // kFA: .x only (real input), [l][col]; kFE: [k][col]
  __shared__ double2 Ms[2][32][kMrK];  // kFA: [k (16 used)][l]; kFE: [l][k]; column swizzled by row & 7
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const long long xbase = (MODE == kFA) ? g.tap_off * r : g.c2_off * r;
  double2 xr[XE], mr[ME];
  auto gload = [&](int l0) {  // l0: kFA nodes l2, kFE frequencies k2
#pragma unroll
    for (int e = 0; e < XE; ++e) {
      const int idx = tid + 128 * e, l = idx / kMrCols, j = idx - l * kMrCols;
      const long long col = c0 + j;
      double2 v = make_double2(0.0, 0.0);
      if (l0 + l < sh.L && col < ncol) {
        const int o = (int)col / (int)sh.I, c = (int)col - o * (int)sh.I;  // 32-bit: ncol < 2^31
        const long long off = xbase + o * sh.xo + (long long)(l0 + l) * sh.xl + c;
        if (MODE == kFA) v.x = static_cast<const double*>(Xv)[off];
        else v = static_cast<const double2*>(Xv)[off];
      }
      xr[e] = v;
    }
#pragma unroll
    for (int e = 0; e < ME; ++e) {
      const int idx = tid + 128 * e, a = idx / kMrK, b = idx - a * kMrK;  // kFA: a = k, b = l; kFE: a = l, b = k
      double2 m = make_double2(0.0, 0.0);
      if (MODE == kFA) {
        const int k = row0 / 2 + a;
        if (a < 16 && k < sh.K && l0 + b < sh.L) m = T[(long long)k * Lt + l0 + b];
      } else {
        const int l = row0 + a, k = l0 + b;
        if (l < sh.K && k < sh.L) m = T[(long long)k * Lt + l];  // Hermitian weight applied at the store
      }
      mr[e] = m;
    }
  };
  gload(0);
  for (int l0 = 0, c = 0; l0 < sh.L; l0 += kMrK, ++c) {
    const int buf = c & 1;
#pragma unroll
    for (int e = 0; e < XE; ++e) {
      const int idx = tid + 128 * e, l = idx / kMrCols, j = idx - l * kMrCols;
      Xs[buf][l][j] = xr[e];
    }
#pragma unroll
    for (int e = 0; e < ME; ++e) {
      const int idx = tid + 128 * e, a = idx / kMrK, b = idx - a * kMrK;
      double2 m = mr[e];
      if (MODE != kFA && l0 + b > 0) {  // kFE: w_k = 2 for k2 > 0 (both halves of the spectrum)
        m.x *= 2.0;
        m.y *= 2.0;
      }
      Ms[buf][a][b ^ (a & 7)] = m;
    }
    __syncthreads();
    if (l0 + kMrK < sh.L) gload(l0 + kMrK);
    constexpr int KS = (MODE == kFA) ? kMrK / 4 : 2 * kMrK / 4;  // k-steps of 4 real k per chunk
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int kr = ks * 4 + (lane & 3);
      double af[2], bf[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int row = (wm * 2 + mt) * 8 + (lane >> 2);
        if (MODE == kFA) {
          const double2 m = Ms[buf][row >> 1][kr ^ ((row >> 1) & 7)];
          af[mt] = (row & 1) ? m.y : m.x;
        } else {
          const double2 m = Ms[buf][row][(kr >> 1) ^ (row & 7)];
          af[mt] = (kr & 1) ? m.y : m.x;
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int col = (wn * 4 + nt) * 8 + (lane >> 2);
        if (MODE == kFA) {
          bf[nt] = Xs[buf][kr][col].x;
        } else {
          const double2 x = Xs[buf][kr >> 1][col];
          bf[nt] = (kr & 1) ? x.y : x.x;
        }
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int row = row0 + (wm * 2 + mt) * 8 + (lane >> 2);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const long long colb = c0 + (wn * 4 + nt) * 8 + 2 * (lane & 3);
      if (MODE == kFA) {
        const double im0 = __shfl_xor_sync(0xffffffffu, acc[mt][nt][0], 4);
        const double im1 = __shfl_xor_sync(0xffffffffu, acc[mt][nt][1], 4);
        const int k = row >> 1;
        if ((row & 1) || k >= sh.K) continue;
        double2* Y = static_cast<double2*>(Yv) + g.a1_off * r;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long long col = colb + h;
          if (col >= ncol) continue;
          const int o = (int)col / (int)sh.I, c = (int)col - o * (int)sh.I;
          Y[o * sh.yo + (long long)k * sh.yk + c] = make_double2(h ? acc[mt][nt][1] : acc[mt][nt][0], h ? im1 : im0);
        }
      } else {
        if (row >= sh.K) continue;
        double* H = static_cast<double*>(Yv) + g.tap_off * (long long)ops * r;
        const long long lines = (long long)g.L[0] * g.L[1];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long long col = colb + h;
          if (col >= ncol) continue;
          const int o = (int)col / (int)sh.I, c = (int)col - o * (int)sh.I, op = o / (int)lines, line = o - op * (int)lines;
          H[((line * g.L[2] + row) * ops + op) * r + c] = acc[mt][nt][h];
        }
      }
    }
  }
}

template <int MODE>
static cudaError_t launch_dft_mma_r(const WinTable& tab, const WinTable* dtab, const void* X, void* Y,
                                    const double2* tw, int r, int ops, cudaStream_t s) {
  long long ctiles = 1;
  int rtiles = 1;
  for (int w = 0; w < tab.P; ++w) {
    const DftShape sh = dft_shape(tab.w[w], MODE, r, ops);
    ctiles = std::max(ctiles, (sh.O * sh.I + kMrCols - 1) / kMrCols);
    rtiles = std::max(rtiles, ((MODE == kFA ? 2 * sh.K : sh.K) + 31) / 32);
  }
  k_dft_mma_r<MODE><<<dim3((unsigned)ctiles, (unsigned)rtiles, tab.P), 128, 0, s>>>(dtab, X, Y, tw, r, ops);
  return cudaGetLastError();
}

static bool no_axis0(const WinTable& tab) {
  for (int w = 0; w < tab.P; ++w)
    if (tab.w[w].L[0] != 1 || tab.w[w].K[0] != 1) return false;
  return true;
}

// the DMMA passes pay off for long axes (the 2-D c3 boxes); short ones stay scalar
static bool use_dft_mma(const WinTable& tab, int mode, int r, int ops) {
  static const int env = getenv("AKM_DFT_MMA") ? atoi(getenv("AKM_DFT_MMA")) : -1;
  if (env >= 0) return env != 0;
  for (int w = 0; w < tab.P; ++w) {
    const DftShape sh = dft_shape(tab.w[w], mode, r, ops);
    if (sh.L < 64 || sh.K < 64) return false;
  }
  return true;
}

// host: grid for one pass = max over windows of the column tiles; smem = max L

// ---------------------------------------------------------------- fused plane kernels
// When a (window, l0) plane of the box fits in shared memory (the 3-D configurations), FA+FB and
// FD+FE run as one kernel per plane with 1024 threads (the intermediate A1 / C2 never leaves
// shared memory; one or a few outputs per thread) and FC1+FC2 as one kernel per column tile:
// three launches instead of six for the latency-bound small problems.
constexpr int kFuseThreads = 1024;

// FA + FB for plane (window blockIdx.y, l0 = blockIdx.x): G[l0] (L1 x L2 x r, real) -> A2[l0]
__global__ void __launch_bounds__(kFuseThreads) k_plane_fwd(const WinTable* __restrict__ tabp,
                                                            const double* __restrict__ G, double2* __restrict__ A2,
                                                            const double2* __restrict__ tw, int r) {
  const WinGeom& g = tabp->w[blockIdx.y];
  const int l0 = blockIdx.x;
  if (l0 >= g.L[0]) return;
  const int L1 = g.L[1], L2 = g.L[2], K1 = g.K[1], K2 = g.K[2];
  extern __shared__ double sm_[];
  double* gs = sm_;                                                           // [L1][L2][r]
  double2* a1 = reinterpret_cast<double2*>(gs + ((L1 * L2 * r + 1) & ~1));    // [L1][K2][r]
  double2* T2 = a1 + L1 * K2 * r;                                             // [K2][L2]
  double2* T1 = T2 + K2 * L2;                                                 // [K1][L1]
  const double* src = G + (g.tap_off + (long long)l0 * L1 * L2) * r;
  for (int idx = threadIdx.x; idx < L1 * L2 * r; idx += blockDim.x) gs[idx] = src[idx];
  for (int idx = threadIdx.x; idx < K2 * L2; idx += blockDim.x) T2[idx] = tw[g.tw_off[2] + idx];
  for (int idx = threadIdx.x; idx < K1 * L1; idx += blockDim.x) T1[idx] = tw[g.tw_off[1] + idx];
  __syncthreads();
  const int KR = K2 * r;
  for (int idx = threadIdx.x; idx < L1 * KR; idx += blockDim.x) {  // (l1, k2, c)
    const int l1 = idx / KR, rem = idx - l1 * KR, k2 = rem / r, c = rem - k2 * r;
    const double* x = gs + (l1 * L2) * r + c;
    const double2* t = T2 + (long long)k2 * L2;
    double re[2] = {0.0, 0.0}, im[2] = {0.0, 0.0};
    int l = 0;
    for (; l + 2 <= L2; l += 2) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double v = x[(l + q) * r];
        re[q] = fma(t[l + q].x, v, re[q]);
        im[q] = fma(t[l + q].y, v, im[q]);
      }
    }
    if (l < L2) {
      const double v = x[l * r];
      re[0] = fma(t[l].x, v, re[0]);
      im[0] = fma(t[l].y, v, im[0]);
    }
    a1[idx] = make_double2(re[0] + re[1], im[0] + im[1]);
  }
  __syncthreads();
  double2* dst = A2 + g.a2_off * r + (long long)l0 * K1 * KR;  // A2[l0][k1][k2][c]
  for (int idx = threadIdx.x; idx < K1 * KR; idx += blockDim.x) {  // (k1, (k2, c))
    const int k1 = idx / KR, j = idx - k1 * KR;
    const double2* t = T1 + (long long)k1 * L1;
    double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    int l = 0;
    for (; l + 2 <= L1; l += 2) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double2 v = a1[(l + q) * KR + j], tt = t[l + q];
        acc[q].x = fma(tt.x, v.x, fma(-tt.y, v.y, acc[q].x));
        acc[q].y = fma(tt.x, v.y, fma(tt.y, v.x, acc[q].y));
      }
    }
    if (l < L1) {
      const double2 v = a1[l * KR + j], tt = t[l];
      acc[0].x = fma(tt.x, v.x, fma(-tt.y, v.y, acc[0].x));
      acc[0].y = fma(tt.x, v.y, fma(tt.y, v.x, acc[0].y));
    }
    dst[idx] = make_double2(acc[0].x + acc[1].x, acc[0].y + acc[1].y);
  }
}

// FD + FE for plane (window blockIdx.y, (op, l0) = blockIdx.x): C[op][l0] (K1 x K2 x r) -> H
__global__ void __launch_bounds__(kFuseThreads) k_plane_inv(const WinTable* __restrict__ tabp,
                                                            const double2* __restrict__ C, double* __restrict__ H,
                                                            const double2* __restrict__ tw, int r, int ops) {
  const WinGeom& g = tabp->w[blockIdx.y];
  const int L0 = g.L[0];
  if ((int)blockIdx.x >= ops * L0) return;
  const int op = blockIdx.x / L0, l0 = blockIdx.x - op * L0;
  const int L1 = g.L[1], L2 = g.L[2], K1 = g.K[1], K2 = g.K[2];
  const int KR = K2 * r;
  extern __shared__ double2 smc[];
  double2* cs = smc;                 // [K1][K2][r]
  double2* c2 = smc + K1 * KR;       // [L1][K2][r]
  double2* T1 = c2 + L1 * KR;        // [K1][L1]
  double2* T2 = T1 + K1 * L1;        // [K2][L2]
  const double2* src = C + g.c_off * r + ((long long)op * L0 + l0) * K1 * KR;
  for (int idx = threadIdx.x; idx < K1 * KR; idx += blockDim.x) cs[idx] = src[idx];
  for (int idx = threadIdx.x; idx < K1 * L1; idx += blockDim.x) T1[idx] = tw[g.tw_off[1] + idx];
  for (int idx = threadIdx.x; idx < K2 * L2; idx += blockDim.x) T2[idx] = tw[g.tw_off[2] + idx];
  __syncthreads();
  for (int idx = threadIdx.x; idx < L1 * KR; idx += blockDim.x) {  // (l1, (k2, c)): sum_k1 conj(T1[k1][l1]) C[k1]
    const int l1 = idx / KR, j = idx - l1 * KR;
    double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    int k = 0;
    for (; k + 2 <= K1; k += 2) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double2 v = cs[(k + q) * KR + j], t = T1[(long long)(k + q) * L1 + l1];
        acc[q].x = fma(t.x, v.x, fma(t.y, v.y, acc[q].x));
        acc[q].y = fma(t.x, v.y, fma(-t.y, v.x, acc[q].y));
      }
    }
    if (k < K1) {
      const double2 v = cs[k * KR + j], t = T1[(long long)k * L1 + l1];
      acc[0].x = fma(t.x, v.x, fma(t.y, v.y, acc[0].x));
      acc[0].y = fma(t.x, v.y, fma(-t.y, v.x, acc[0].y));
    }
    c2[idx] = make_double2(acc[0].x + acc[1].x, acc[0].y + acc[1].y);
  }
  __syncthreads();
  // H[((l0 L1 + l1) L2 + l2) ops + op][c] = Re sum_k2 alpha conj(T2[k2][l2]) C2[l1][k2][c]
  const long long hbase = g.tap_off * (long long)ops * r;
  const int LR = L2 * r;
  for (int idx = threadIdx.x; idx < L1 * LR; idx += blockDim.x) {
    const int l1 = idx / LR, rem = idx - l1 * LR, l2 = rem / r, c = rem - l2 * r;
    const double2* x = c2 + l1 * KR + c;
    double acc[2] = {0.0, 0.0};
    for (int k = 0; k < K2; ++k) {
      const double2 t = T2[(long long)k * L2 + l2], v = x[k * r];
      const double w = (k == 0) ? 1.0 : 2.0;
      acc[k & 1] = fma(w, fma(t.x, v.x, t.y * v.y), acc[k & 1]);
    }
    const long long tap = ((long long)l0 * L1 + l1) * L2 + l2;
    H[hbase + (tap * ops + op) * r + c] = acc[0] + acc[1];
  }
}

// FC1 + FC2 for a tile of columns (k1, k2, c): A2[l0][col] -> A3 (smem) -> C[op][l0][col]
template <int COLS>
__global__ void __launch_bounds__(kDftThreads) k_pencil(const WinTable* __restrict__ tabp, const double2* __restrict__ A2,
                                                        double2* __restrict__ C, const double2* __restrict__ tw,
                                                        const double* __restrict__ D, int dslot0, int r, int ops) {
  const WinGeom& g = tabp->w[blockIdx.y];
  const int L0 = g.L[0], K0 = g.K[0];
  const long long I = (long long)g.K[1] * g.K[2] * r;
  const long long col0 = (long long)blockIdx.x * COLS;
  if (col0 >= I) return;
  extern __shared__ double2 smp[];
  double2* xs = smp;                     // [L0][COLS]
  double2* a3 = smp + L0 * COLS;         // [ops][K0][COLS]  D_op * A3
  double2* T0 = a3 + ops * K0 * COLS;    // [K0][L0]
  const int tid = threadIdx.x;
  const double2* src = A2 + g.a2_off * r;
  for (int idx = tid; idx < L0 * COLS; idx += kDftThreads) {
    const int l = idx / COLS, j = idx - l * COLS;
    xs[idx] = (col0 + j < I) ? src[(long long)l * I + col0 + j] : make_double2(0.0, 0.0);
  }
  for (int idx = tid; idx < K0 * L0; idx += kDftThreads) T0[idx] = tw[g.tw_off[0] + idx];
  __syncthreads();
  const long long kk = (long long)g.K[1] * g.K[2], dper = (long long)K0 * kk;
  for (int idx = tid; idx < K0 * COLS; idx += kDftThreads) {  // forward along l0, then D_op
    const int k = idx / COLS, j = idx - k * COLS;
    double2 acc = make_double2(0.0, 0.0);
    for (int l = 0; l < L0; ++l) {
      const double2 t = T0[k * L0 + l], v = xs[l * COLS + j];
      acc.x = fma(t.x, v.x, fma(-t.y, v.y, acc.x));
      acc.y = fma(t.x, v.y, fma(t.y, v.x, acc.y));
    }
    const long long col = col0 + j;
    for (int op = 0; op < ops; ++op) {
      const double dd = (col < I) ? D[g.d_off + (dslot0 + op) * dper + (long long)k * kk + col / r] : 0.0;
      a3[(op * K0 + k) * COLS + j] = make_double2(dd * acc.x, dd * acc.y);
    }
  }
  __syncthreads();
  double2* dst = C + g.c_off * r;
  for (int idx = tid; idx < ops * L0 * COLS; idx += kDftThreads) {  // inverse along k0
    const int j = idx % COLS, ol = idx / COLS, op = ol / L0, l = ol - op * L0;
    const long long col = col0 + j;
    if (col >= I) continue;
    const double2* av = a3 + op * K0 * COLS + j;
    double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    for (int k = 0; k < K0; ++k) {
      const double2 t = T0[k * L0 + l], v = av[k * COLS];
      acc[k & 1].x = fma(t.x, v.x, fma(t.y, v.y, acc[k & 1].x));
      acc[k & 1].y = fma(t.x, v.y, fma(-t.y, v.x, acc[k & 1].y));
    }
    dst[((long long)op * L0 + l) * I + col] = make_double2(acc[0].x + acc[1].x, acc[0].y + acc[1].y);
  }
}

static bool planes_fit(const WinTable& tab, int r, size_t& smem_fwd, size_t& smem_inv) {
  smem_fwd = smem_inv = 0;
  for (int w = 0; w < tab.P; ++w) {
    const WinGeom& g = tab.w[w];
    if (g.d < 3) return false;  // 2-D boxes are single large planes: the generic passes
    const size_t tws = sizeof(double2) * ((size_t)g.K[1] * g.L[1] + (size_t)g.K[2] * g.L[2]);
    const size_t fwd = sizeof(double) * (((size_t)g.L[1] * g.L[2] * r + 1) & ~(size_t)1) +
                       sizeof(double2) * (size_t)g.L[1] * g.K[2] * r + tws;
    const size_t inv = sizeof(double2) * ((size_t)g.K[1] + g.L[1]) * g.K[2] * r + tws;
    smem_fwd = std::max(smem_fwd, fwd);
    smem_inv = std::max(smem_inv, inv);
  }
  return smem_fwd <= 200 * 1024 && smem_inv <= 200 * 1024;
}

template <int MODE, int COLS>
static cudaError_t launch_cols(long long tiles, int P, int Lmax, const WinTable* dtab, const void* X, void* Y,
                               const double2* tw, const double* D, int dslot0, int r, int ops, cudaStream_t s) {
  const size_t smem = sizeof(double2) * (size_t)Lmax * COLS;
  static std::atomic<unsigned long long> attr_set{0};
  if (!optin_done(attr_set)) {
    cudaError_t e = cudaFuncSetAttribute(k_dft_axis<MODE, COLS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    optin_mark(attr_set);
  }
  k_dft_axis<MODE, COLS><<<dim3((unsigned)tiles, P), kDftThreads, smem, s>>>(dtab, X, Y, tw, D, dslot0, r, ops);
  return cudaGetLastError();
}

// columns per CTA: 32 when there are many columns; 8 for small passes (more CTAs, fewer outputs
// per thread -- the small configurations are latency-bound)
template <int MODE>
static cudaError_t launch_pass(const WinTable& tab, const WinTable* dtab, const void* X, void* Y, const double2* tw,
                               const double* D, int dslot0, int r, int ops, cudaStream_t s) {
  long long cols = 1, total = 0;
  int Lmax = 1, Kmax = 1;
  for (int w = 0; w < tab.P; ++w) {
    const DftShape sh = dft_shape(tab.w[w], MODE, r, ops);
    cols = std::max(cols, sh.O * sh.I);
    total += sh.O * sh.I;
    Lmax = std::max(Lmax, sh.L);
    Kmax = std::max(Kmax, sh.K);
  }
  if (Kmax <= 2)  // singleton axis (d < 3): a copy / scaling, every thread its own column
    return launch_cols<MODE, 128>((cols + 127) / 128, tab.P, Lmax, dtab, X, Y, tw, D, dslot0, r, ops, s);
  if (total >= 148LL * 4 * 32)
    return launch_cols<MODE, 32>((cols + 31) / 32, tab.P, Lmax, dtab, X, Y, tw, D, dslot0, r, ops, s);
  return launch_cols<MODE, 8>((cols + 7) / 8, tab.P, Lmax, dtab, X, Y, tw, D, dslot0, r, ops, s);
}

cudaError_t launch_fft_forward(const WinTable& tab, const WinTable* dtab, const double* grid, double2* A1, double2* A2,
                               const double2* tw, int r, cudaStream_t s) {
  size_t sf, si;
  if (planes_fit(tab, r, sf, si)) {
    int L0 = 1;
    for (int w = 0; w < tab.P; ++w) L0 = std::max(L0, tab.w[w].L[0]);
    static std::atomic<unsigned long long> attr{0};
    if (!optin_done(attr)) {
      cudaError_t e = cudaFuncSetAttribute(k_plane_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
      optin_mark(attr);
    }
    k_plane_fwd<<<dim3(L0, tab.P), kFuseThreads, sf, s>>>(dtab, grid, A2, tw, r);
    return cudaGetLastError();
  }
  cudaError_t e = use_dft_mma(tab, kFA, r, 1) ? launch_dft_mma_r<kFA>(tab, dtab, grid, A1, tw, r, 1, s)
                                               : launch_pass<kFA>(tab, dtab, grid, A1, tw, nullptr, 0, r, 1, s);
  if (e != cudaSuccess) return e;
  if (use_dft_mma(tab, kFB, r, 1)) return launch_dft_mma<kFB>(tab, dtab, A1, A2, tw, r, 1, s);
  return launch_pass<kFB>(tab, dtab, A1, A2, tw, nullptr, 0, r, 1, s);
}

cudaError_t launch_fft_multiply_inverse(const WinTable& tab, const WinTable* dtab, const double2* A2, double2* A3,
                                        double2* C, double2* C2, const double2* tw, const double* D, int ops,
                                        int dslot0, int r, double* H, cudaStream_t s) {
  size_t sf, si;
  if (planes_fit(tab, r, sf, si)) {
    int L0 = 1, K0 = 1;
    long long I = 1;
    for (int w = 0; w < tab.P; ++w) {
      L0 = std::max(L0, tab.w[w].L[0]);
      K0 = std::max(K0, tab.w[w].K[0]);
      I = std::max(I, (long long)tab.w[w].K[1] * tab.w[w].K[2] * r);
    }
    // columns per pencil CTA: 4 for few columns (r = 1: more CTAs against latency), else 8
    static std::atomic<unsigned long long> attr{0};
    if (!optin_done(attr)) {
      cudaError_t e = cudaFuncSetAttribute(k_plane_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(k_pencil<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(k_pencil<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
      optin_mark(attr);
    }
    if (I < 2048) {
      constexpr int PC = 4;
      const size_t sp = sizeof(double2) * ((size_t)(L0 + ops * K0) * PC + (size_t)K0 * L0);
      k_pencil<PC><<<dim3((unsigned)((I + PC - 1) / PC), tab.P), kDftThreads, sp, s>>>(dtab, A2, C, tw, D, dslot0, r,
                                                                                      ops);
    } else {
      constexpr int PC = 8;
      const size_t sp = sizeof(double2) * ((size_t)(L0 + ops * K0) * PC + (size_t)K0 * L0);
      k_pencil<PC><<<dim3((unsigned)((I + PC - 1) / PC), tab.P), kDftThreads, sp, s>>>(dtab, A2, C, tw, D, dslot0, r,
                                                                                      ops);
    }
    k_plane_inv<<<dim3(L0 * ops, tab.P), kFuseThreads, si, s>>>(dtab, C, H, tw, r, ops);
    return cudaGetLastError();
  }
  cudaError_t e = cudaSuccess;
  if (use_dft_mma(tab, kFD, r, ops) && no_axis0(tab)) {
    // no axis 0: FC1 is a copy and FC2 a multiply; both fold into the FD load
    e = launch_dft_mma<kFD, true>(tab, dtab, A2, C2, tw, r, ops, s, D, dslot0);
  } else {
    e = launch_pass<kFC1>(tab, dtab, A2, A3, tw, nullptr, 0, r, ops, s);
    if (e == cudaSuccess) e = launch_pass<kFC2>(tab, dtab, A3, C, tw, D, dslot0, r, ops, s);
    if (e == cudaSuccess) {
      if (use_dft_mma(tab, kFD, r, ops)) e = launch_dft_mma<kFD>(tab, dtab, C, C2, tw, r, ops, s);
      else e = launch_pass<kFD>(tab, dtab, C, C2, tw, nullptr, 0, r, ops, s);
    }
  }
  if (e == cudaSuccess) {
    if (use_dft_mma(tab, kFE, r, ops)) e = launch_dft_mma_r<kFE>(tab, dtab, C2, H, tw, r, ops, s);
    else e = launch_pass<kFE>(tab, dtab, C2, H, tw, nullptr, 0, r, ops, s);
  }
  return e;
}

// kernels launched by launch_fft_forward + launch_fft_multiply_inverse (for the launch counters)
int fft_launch_count(const WinTable& tab, int r) {
  size_t sf, si;
  if (planes_fit(tab, r, sf, si)) return 3;
  return use_dft_mma(tab, kFD, r, 1) && no_axis0(tab) ? 4 : 6;
}

cudaError_t launch_zero(double* p, long long count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  return cudaMemsetAsync(p, 0, sizeof(double) * count, s);
}

}  // namespace akm
