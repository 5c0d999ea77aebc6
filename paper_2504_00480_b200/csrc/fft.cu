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
// have one node and k = 0 with twiddle 1.  The stage is L2-resident and ~1% of the MVM.
#include "akm_internal.cuh"

namespace akm {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// Thread-per-output kernels; blockIdx.y = window.  r = number of RHS (innermost index).
__global__ void k_fa(const WinTable* __restrict__ tabp, const double* __restrict__ G, double2* __restrict__ A1,
                     const double2* __restrict__ tw, int r) {
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[blockIdx.y];
  const long long total = (long long)g.L[0] * g.L[1] * g.K[2] * r;
  const double2* T = tw + g.tw_off[2];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(idx % r);
    const long long q = idx / r;
    const int k2 = (int)(q % g.K[2]);
    const long long line = q / g.K[2];  // l0*L1 + l1
    const double* src = G + (g.tap_off + line * g.L[2]) * r + c;
    const double2* Tk = T + (long long)k2 * g.L[2];
    double re = 0.0, im = 0.0;
    for (int l = 0; l < g.L[2]; ++l) {
      const double v = src[(long long)l * r];
      const double2 t = Tk[l];
      re = fma(t.x, v, re);
      im = fma(t.y, v, im);
    }
    A1[(g.a1_off + q) * r + c] = make_double2(re, im);
  }
}

__global__ void k_fb(const WinTable* __restrict__ tabp, const double2* __restrict__ A1, double2* __restrict__ A2,
                     const double2* __restrict__ tw, int r) {
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[blockIdx.y];
  const long long total = (long long)g.L[0] * g.K[1] * g.K[2] * r;
  const double2* T = tw + g.tw_off[1];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx % ((long long)g.K[2] * r);  // (k2, c)
    const long long q = idx / ((long long)g.K[2] * r);
    const int k1 = (int)(q % g.K[1]);
    const int l0 = (int)(q / g.K[1]);
    const double2* src = A1 + (g.a1_off + (long long)l0 * g.L[1] * g.K[2]) * r + j;
    const double2* Tk = T + (long long)k1 * g.L[1];
    double2 acc = make_double2(0.0, 0.0);
    for (int l = 0; l < g.L[1]; ++l) {
      const double2 v = src[(long long)l * g.K[2] * r];
      const double2 t = Tk[l];
      acc.x = fma(t.x, v.x, fma(-t.y, v.y, acc.x));
      acc.y = fma(t.x, v.y, fma(t.y, v.x, acc.y));
    }
    A2[g.a2_off * r + idx] = acc;
  }
}

// FC1: A3[k0][k1][k2][c] = sum_l0 T0[k0][l0] A2[l0][k1][k2][c]
__global__ void k_fc1(const WinTable* __restrict__ tabp, const double2* __restrict__ A2, double2* __restrict__ A3,
                      const double2* __restrict__ tw, int r) {
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[blockIdx.y];
  const long long plane = (long long)g.K[1] * g.K[2] * r;
  const long long total = (long long)g.K[0] * plane;
  const double2* T = tw + g.tw_off[0];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx % plane;
    const int k0 = (int)(idx / plane);
    const double2* src = A2 + g.a2_off * r + j;
    const double2* Tk = T + (long long)k0 * g.L[0];
    double2 acc = make_double2(0.0, 0.0);
    for (int l = 0; l < g.L[0]; ++l) {
      const double2 v = src[(long long)l * plane];
      const double2 t = Tk[l];
      acc.x = fma(t.x, v.x, fma(-t.y, v.y, acc.x));
      acc.y = fma(t.x, v.y, fma(t.y, v.x, acc.y));
    }
    A3[g.a3_off * r + idx] = acc;
  }
}

// FC2: C[op][l0][k1][k2][c] = sum_k0 conj(T0[k0][l0]) D_op[k0][k1][k2] A3[k0][k1][k2][c]
__global__ void k_fc2(const WinTable* __restrict__ tabp, const double2* __restrict__ A3, double2* __restrict__ C,
                      const double2* __restrict__ tw, const double* __restrict__ D, int ops, int dslot0, int r) {
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[blockIdx.y];
  const long long kplane = (long long)g.K[1] * g.K[2];
  const long long plane = kplane * r;
  const long long per_op = (long long)g.L[0] * plane;
  const long long total = ops * per_op;
  const long long dper = (long long)g.K[0] * kplane;
  const double2* T = tw + g.tw_off[0];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int op = (int)(idx / per_op);
    const long long rem = idx % per_op;
    const int l0 = (int)(rem / plane);
    const long long j = rem % plane;   // (k1, k2, c)
    const long long kj = j / r;        // (k1, k2)
    const double2* src = A3 + g.a3_off * r + j;
    const double* Dk = D + g.d_off + (dslot0 + op) * dper + kj;
    double2 acc = make_double2(0.0, 0.0);
    for (int k0 = 0; k0 < g.K[0]; ++k0) {
      const double2 v = src[(long long)k0 * plane];
      const double dd = Dk[(long long)k0 * kplane];
      const double2 t = T[(long long)k0 * g.L[0] + l0];
      const double2 y = make_double2(dd * v.x, dd * v.y);
      // conj(t) * y
      acc.x = fma(t.x, y.x, fma(t.y, y.y, acc.x));
      acc.y = fma(t.x, y.y, fma(-t.y, y.x, acc.y));
    }
    C[g.c_off * r + idx] = acc;
  }
}

// FD: C2[op][l0][l1][k2][c] = sum_k1 conj(T1[k1][l1]) C[op][l0][k1][k2][c]
__global__ void k_fd(const WinTable* __restrict__ tabp, const double2* __restrict__ C, double2* __restrict__ C2,
                     const double2* __restrict__ tw, int ops, int r) {
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[blockIdx.y];
  const long long inner = (long long)g.K[2] * r;
  const long long per_op = (long long)g.L[0] * g.L[1] * inner;
  const long long total = ops * per_op;
  const double2* T = tw + g.tw_off[1];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int op = (int)(idx / per_op);
    const long long rem = idx % per_op;
    const long long j = rem % inner;
    const long long q = rem / inner;
    const int l1 = (int)(q % g.L[1]);
    const int l0 = (int)(q / g.L[1]);
    const double2* src = C + g.c_off * r + (long long)op * g.L[0] * g.K[1] * inner + (long long)l0 * g.K[1] * inner + j;
    double2 acc = make_double2(0.0, 0.0);
    for (int k1 = 0; k1 < g.K[1]; ++k1) {
      const double2 v = src[(long long)k1 * inner];
      const double2 t = T[(long long)k1 * g.L[1] + l1];
      acc.x = fma(t.x, v.x, fma(t.y, v.y, acc.x));
      acc.y = fma(t.x, v.y, fma(-t.y, v.x, acc.y));
    }
    C2[g.c2_off * r + idx] = acc;
  }
}

// FE: H[(tap_off + tap) * ops*r + op*r + c] = Re sum_k2 alpha_k2 conj(T2[k2][l2]) C2[op][l0][l1][k2][c]
__global__ void k_fe(const WinTable* __restrict__ tabp, const double2* __restrict__ C2, double* __restrict__ H,
                     const double2* __restrict__ tw, int ops, int r) {
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[blockIdx.y];
  const long long total = g.ntap * ops * r;
  const double2* T = tw + g.tw_off[2];
  const long long lines = (long long)g.L[0] * g.L[1];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(idx % r);
    const int op = (int)((idx / r) % ops);
    const long long tap = idx / ((long long)ops * r);
    const int l2 = (int)(tap % g.L[2]);
    const long long line = tap / g.L[2];
    const double2* src = C2 + (g.c2_off + ((long long)op * lines + line) * g.K[2]) * r + c;
    double acc = 0.0;
    for (int k2 = 0; k2 < g.K[2]; ++k2) {
      const double2 v = src[(long long)k2 * r];
      const double2 t = T[(long long)k2 * g.L[2] + l2];
      // Re(conj(t) v) = t.x v.x + t.y v.y
      const double re = fma(t.x, v.x, t.y * v.y);
      acc = (k2 == 0) ? re : fma(2.0, re, acc);
    }
    H[(g.tap_off + tap) * ops * r + op * r + c] = acc;
  }
}

static int blocks_for(long long total) {
  long long b = (total + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_fft_forward(const WinTable& tab, const WinTable* dtab, const double* grid, double2* A1, double2* A2, const double2* tw,
                               int r, long long maxA1, long long maxA2, cudaStream_t s) {
  k_fa<<<dim3(blocks_for(maxA1 * r), tab.P), 256, 0, s>>>(dtab, grid, A1, tw, r);
  k_fb<<<dim3(blocks_for(maxA2 * r), tab.P), 256, 0, s>>>(dtab, A1, A2, tw, r);
  return cudaGetLastError();
}

cudaError_t launch_fft_multiply_inverse(const WinTable& tab, const WinTable* dtab, const double2* A2, double2* A3, double2* C,
                                        double2* C2, const double2* tw, const double* D, int ops, int dslot0, int r, double* H,
                                        long long maxA3, long long maxC, long long maxC2, long long maxTap,
                                        cudaStream_t s) {
  k_fc1<<<dim3(blocks_for(maxA3 * r), tab.P), 256, 0, s>>>(dtab, A2, A3, tw, r);
  k_fc2<<<dim3(blocks_for(maxC * ops * r), tab.P), 256, 0, s>>>(dtab, A3, C, tw, D, ops, dslot0, r);
  k_fd<<<dim3(blocks_for(maxC2 * ops * r), tab.P), 256, 0, s>>>(dtab, C, C2, tw, ops, r);
  k_fe<<<dim3(blocks_for(maxTap * ops * r), tab.P), 256, 0, s>>>(dtab, C2, H, tw, ops, r);
  return cudaGetLastError();
}

__global__ void k_zero(double* __restrict__ p, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

cudaError_t launch_zero(double* p, long long count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  return cudaMemsetAsync(p, 0, sizeof(double) * count, s);
}

}  // namespace akm
