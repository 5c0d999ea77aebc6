// setup_kernels.cu -- device side of akm_set_points / akm_set_theta.
//
//   window_minmax / window_radius : per-window bounding box and radius R_w (reading R2)
//   scale_and_key                 : scaled grid coordinates u = (x - center) n_g / c_w,
//                                   cell index, cell histogram (the rest of the bin sort: binsort.cu)
//   kernel_samples, cos_dft_axis  : b_k of eq. (3.2) for kappa and kappa^der
//   deconv_table, multiplier      : D_k = omega_k b_k / prod_t I0(m sqrt(beta^2-(2 pi k_t/n_g)^2))^2
//                                   (App. A deconvolution; reading R5 for omega)
//   twiddles                      : e^{-2 pi i k (box_lo + l) / n_g} tables of the box-local DFTs
#include "akm_internal.cuh"

namespace akm {

// ---------------------------------------------------------------- min / max per feature
__global__ void k_window_minmax(const double* __restrict__ X, long long n, long long ldx,
                                const int* __restrict__ feat, double* __restrict__ out) {
  const int f = feat[blockIdx.x];
  double lo = INFINITY, hi = -INFINITY;
  bool bad = false;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = X[i * ldx + f];
    if (!isfinite(v)) bad = true;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  __shared__ double slo[32], shi[32];
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  if (bad) atomicOr(&sbad, 1);
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { slo[wid] = lo; shi[wid] = hi; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    lo = lane < nw ? slo[lane] : INFINITY;
    hi = lane < nw ? shi[lane] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      out[3 * blockIdx.x + 0] = lo;
      out[3 * blockIdx.x + 1] = hi;
      out[3 * blockIdx.x + 2] = sbad ? 1.0 : 0.0;
    }
  }
}

cudaError_t launch_window_minmax(const double* X, long long n, long long ldx, const int* feat_dev, int nfeat,
                                 double* minmax_dev, cudaStream_t s) {
  if (nfeat <= 0) return cudaSuccess;
  k_window_minmax<<<nfeat, 1024, 0, s>>>(X, n, ldx, feat_dev, minmax_dev);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- compact copy of the window features
__global__ void k_gather_columns(const double* __restrict__ X, long long n, long long ldx, const int* __restrict__ feat,
                                 int nf, double* __restrict__ Xc) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * nf;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / nf;
    const int j = (int)(idx % nf);
    Xc[idx] = X[i * ldx + feat[j]];
  }
}

cudaError_t launch_gather_columns(const double* X, long long n, long long ldx, const int* feat, int nf, double* Xc,
                                  cudaStream_t s) {
  if (n == 0 || nf == 0) return cudaSuccess;
  long long blocks = (n * nf + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_gather_columns<<<(int)blocks, 256, 0, s>>>(X, n, ldx, feat, nf, Xc);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- radius per window
// r2[w] = max_i sum_t (x_{i,f_t} - center_t)^2, as the bit pattern of a non-negative double
// (monotone under unsigned comparison) accumulated with atomicMax.
__global__ void k_window_radius(const double* __restrict__ X, long long n, long long ldx, const WinTable* __restrict__ tabp,
                                unsigned long long* __restrict__ r2bits) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y;
  const WinGeom& g = tab.w[w];
  double best = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double rr = 0.0;
    for (int a = 3 - g.d; a < 3; ++a) {
      const double t = X[i * ldx + g.feat[a]] - g.center[a];
      rr += t * t;
    }
    best = fmax(best, rr);
  }
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(r2bits + w, (unsigned long long)__double_as_longlong(best));
}

cudaError_t launch_window_radius(const double* X, long long n, long long ldx, const WinTable& tab, const WinTable* dtab, double* r2_dev,
                                 cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(r2_dev, 0, sizeof(double) * tab.P, s);
  if (e != cudaSuccess) return e;
  if (n == 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  k_window_radius<<<dim3((unsigned)blocks, tab.P), 256, 0, s>>>(X, n, ldx, dtab, (unsigned long long*)r2_dev);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- scaling + cell histogram
__device__ __forceinline__ long long cell_linear(const WinGeom& g, const int c[3]) {
  return ((long long)c[0] * g.ncell[1] + c[1]) * g.ncell[2] + c[2];
}

// Histogram key = (cell, class): class 1 marks the rows i >= n_split (the targets of a cross
// product, akm_kernel_cross_mvm), so the two classes can be laid out apart inside every bin.
// One thread per point for all windows: the point's row of X is read once (the later windows hit L1).
__global__ void k_scale_and_key(const double* __restrict__ X, long long n, long long ldx, const WinTable* __restrict__ tabp,
                                double* __restrict__ u_tmp, int* __restrict__ hist,
                                const long long* __restrict__ hist_off, int* __restrict__ err_flag, long long n_split) {
  const WinTable& tab = *tabp;
  const int m = tab.m;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    for (int w = 0; w < tab.P; ++w) {
      const WinGeom& g = tab.w[w];
      int c[3] = {0, 0, 0};
      bool ok = true;
      for (int a = 3 - g.d; a < 3; ++a) {
        const double u = (__ldg(X + i * ldx + g.feat[a]) - g.center[a]) * g.scale;
        u_tmp[((long long)w * 3 + a) * n + i] = u;
        const int cc = (int)floor(u) - (g.box_lo[a] + m - 1);
        ok = ok && cc >= 0 && cc < g.ncell[a];
        c[a] = cc;
      }
      if (!ok) atomicOr(err_flag, 1);
      // warp-level aggregation: lanes with the same (cell, class) key elect one leader that adds the
      // group's size (points concentrate in few cells, up to 2.5e4 per cell: contended atomics otherwise)
      const long long key = ok ? hist_off[w] + 2 * cell_linear(g, c) + (i >= n_split ? 1 : 0) : -1;
      const unsigned act = __activemask();
      const unsigned peers = __match_any_sync(act, key);
      const int leader = __ffs(peers) - 1;
      if (ok && (int)(threadIdx.x & 31) == leader) atomicAdd(hist + key, __popc(peers));
    }
  }
}

cudaError_t launch_scale_and_key(const double* X, long long n, long long ldx, const WinTable& tab, const WinTable* dtab, double* u_tmp,
                                 int* /*key*/, int* hist, const long long* hist_off, int* err_flag, long long n_split,
                                 cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_scale_and_key<<<(unsigned)blocks, 256, 0, s>>>(X, n, ldx, dtab, u_tmp, hist, hist_off, err_flag, n_split);
  return cudaGetLastError();
}


// ---------------------------------------------------------------- b_k (eq. 3.2)
// samples s[l] = kappa(l/N; ell_eff) (or kappa^der) for l in I_N^d, stored at index (l + N/2).
__global__ void k_kernel_samples(int family, int d, int N, double ell, int deriv, double* __restrict__ out) {
  long long total = 1;
  for (int t = 0; t < d; ++t) total *= N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long rem = idx;
    double rr = 0.0;
    for (int t = 0; t < d; ++t) {
      const int li = (int)(rem % N) - N / 2;
      rem /= N;
      const double x = (double)li / (double)N;
      rr += x * x;
    }
    double v;
    if (family == 0) {  // Gaussian, eq. (2.2) / (2.3)
      const double k = exp(-rr / (2.0 * ell * ell));
      v = deriv ? rr / (ell * ell * ell) * k : k;
    } else {            // Matern(1/2)
      const double rn = sqrt(rr);
      const double k = exp(-rn / ell);
      v = deriv ? rn / (ell * ell) * k : k;
    }
    out[idx] = v;
  }
}

cudaError_t launch_kernel_samples(int family, int d, int N, double ell_eff, int deriv, double* out, cudaStream_t s) {
  long long total = 1;
  for (int t = 0; t < d; ++t) total *= N;
  int blocks = (int)((total + 255) / 256);
  k_kernel_samples<<<blocks, 256, 0, s>>>(family, d, N, ell_eff, deriv, out);
  return cudaGetLastError();
}

// One axis of the real cosine DFT  out[k] = (1/N) sum_{l in I_N} cos(2 pi k l / N) in[l].
// The samples are even in every axis separately (kappa depends on |l_t| and the node -N/2 is its
// own mirror on the torus), so the sine parts of eq. (3.2) vanish axis by axis and b_k is real.
// Axis index t counts from the fastest-varying (t = 0) dimension of the flat array.
// The N cosines cos(2 pi j / N) are computed once per CTA into shared memory (cospi, exact phase
// reduction j = k l mod N as before); each term is then a table lookup (N <= kCosTabMax; larger N
// evaluate cospi per term).
constexpr int kCosTabMax = 4096;
__global__ void k_cos_dft_axis(int d, int N, int axis, const double* __restrict__ in, double* __restrict__ out) {
  extern __shared__ double cos_tab[];
  const bool tab = N <= kCosTabMax;
  if (tab)
    for (int j = threadIdx.x; j < N; j += blockDim.x) cos_tab[j] = cospi(2.0 * (double)j / (double)N);
  __syncthreads();
  long long total = 1;
  for (int t = 0; t < d; ++t) total *= N;
  long long stride = 1;
  for (int t = 0; t < axis; ++t) stride *= N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int ki = (int)((idx / stride) % N);
    const long long base = idx - (long long)ki * stride;
    const int k = ki - N / 2;
    int j = (int)(((long long)k * (-N / 2)) % N);  // k l mod N for l = -N/2, then += k per step
    if (j < 0) j += N;
    const int kstep = ((k % N) + N) % N;
    double acc = 0.0;
    for (int li = 0; li < N; ++li) {
      acc += (tab ? cos_tab[j] : cospi(2.0 * (double)j / (double)N)) * in[base + (long long)li * stride];
      j += kstep;
      if (j >= N) j -= N;
    }
    out[idx] = acc / (double)N;
  }
}

cudaError_t launch_cos_dft_axis(int d, int N, int axis, const double* in, double* out, cudaStream_t s) {
  long long total = 1;
  for (int t = 0; t < d; ++t) total *= N;
  int blocks = (int)((total + 255) / 256);
  k_cos_dft_axis<<<blocks, 256, N <= kCosTabMax ? sizeof(double) * N : 0, s>>>(d, N, axis, in, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- multiplier tables
// D[op][k0][k1][k2] for the box-local spectrum of window `win`:
//   k_a in {-N/2..N/2} on real leading axes (index k+N/2), {0..N/2} on the last axis, {0} on
//   singleton axes.  With unnormalised forward/backward DFTs on the n_g^d grid,
//   h = IDFT( D . DFT(g) ),  D_k = omega_k b_k / prod_t (n_g c_{k_t}(phi))^2,
//   n_g c_k(phi) = I0(m sqrt(beta^2 - (2 pi k / n_g)^2))   (reading R4),
//   omega_k = (1[k in I_N^d] + 1[-k in I_N^d]) / 2          (reading R5: real part of eq. 3.3),
// and for the ell-derivative table the joint-scaling factor 1/c_w (reading R7).
// i0sq[a * (N + 1) + ki] = I0(m sqrt(beta^2 - (2 pi k / n_g)^2))^2, k = ki (a = 2) or ki - N/2: the
// per-axis factors of the deconvolution; they depend on (N, n_g, m, sigma) only (set_points)
__global__ void k_deconv_table(int N, int n_g, int m, double beta, double* __restrict__ i0sq) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 3 * (N + 1); idx += gridDim.x * blockDim.x) {
    const int a = idx / (N + 1), ki = idx % (N + 1);
    const int k = (a == 2) ? ki : ki - N / 2;
    const double wk = 2.0 * kPi * (double)k / (double)n_g;
    const double i0 = bessel_i0((double)m * sqrt(beta * beta - wk * wk));
    i0sq[idx] = i0 * i0;
  }
}

cudaError_t launch_deconv_table(int N, int n_g, int m, double sigma_over, double* i0sq, cudaStream_t s) {
  const double beta = kPi * (2.0 - 1.0 / sigma_over);
  k_deconv_table<<<(3 * (N + 1) + 255) / 256, 256, 0, s>>>(N, n_g, m, beta, i0sq);
  return cudaGetLastError();
}

__global__ void k_multiplier(const WinTable* __restrict__ tabp, int win, const double* __restrict__ bK, const double* __restrict__ bL,
                             int ops_mask, double inv_c, const double* __restrict__ i0sq, double* __restrict__ D) {
  const WinTable& tab = *tabp;
  const WinGeom& g = tab.w[win];
  const int N = tab.N, n_g = tab.n_g, m = tab.m, d = g.d;
  const long long per = (long long)g.K[0] * g.K[1] * g.K[2];
  // the deconvolution factorises over the axes: I0(.)^2 per axis and frequency (k_deconv_table)
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < per;
       idx += (long long)gridDim.x * blockDim.x) {
    int kk[3];
    kk[2] = (int)(idx % g.K[2]);                 // 0..N/2
    kk[1] = (int)((idx / g.K[2]) % g.K[1]);
    kk[0] = (int)(idx / ((long long)g.K[2] * g.K[1]));
    int k[3];
    k[2] = kk[2];
    k[1] = (g.K[1] == 1) ? 0 : kk[1] - N / 2;
    k[0] = (g.K[0] == 1) ? 0 : kk[0] - N / 2;
    bool inI = true, negInI = true;
    double deconv = 1.0;
    long long bidx = 0;
    for (int a = 3 - d; a < 3; ++a) {
      inI = inI && (k[a] >= -N / 2) && (k[a] <= N / 2 - 1);
      negInI = negInI && (-k[a] >= -N / 2) && (-k[a] <= N / 2 - 1);
      deconv *= i0sq[a * (N + 1) + kk[a]];
      int km = k[a] % N;  // periodic index of b: k mod N in I_N
      if (km >= N / 2) km -= N;
      if (km < -N / 2) km += N;
      bidx = bidx * N + (km + N / 2);
    }
    const double omega = 0.5 * ((inI ? 1.0 : 0.0) + (negInI ? 1.0 : 0.0));
    int slot = 0;
    if (ops_mask & 1) D[g.d_off + (slot++) * per + idx] = omega * bK[bidx] / deconv;
    if (ops_mask & 2) D[g.d_off + (slot++) * per + idx] = omega * bL[bidx] * inv_c / deconv;
  }
}

cudaError_t launch_multiplier(const WinTable& tab, const WinTable* dtab, int win, const double* bK, const double* bL, int ops_mask,
                              double inv_c, const double* i0sq, double* D, cudaStream_t s) {
  const WinGeom& g = tab.w[win];
  const long long per = (long long)g.K[0] * g.K[1] * g.K[2];
  int blocks = (int)std::min<long long>((per + 255) / 256, 148 * 4);
  k_multiplier<<<blocks, 256, 0, s>>>(dtab, win, bK, bL, ops_mask, inv_c, i0sq, D);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- twiddles
// tw[tw_off[a] + k_index * L_a + l] = exp(-2 pi i k (box_lo_a + l) / n_g), exact phase reduction mod n_g.
__global__ void k_twiddles(const WinTable* __restrict__ tabp, double2* __restrict__ tw) {
  const WinTable& tab = *tabp;
  const int win = blockIdx.y;
  const WinGeom& g = tab.w[win];
  const int N = tab.N, n_g = tab.n_g;
  for (int a = 0; a < 3; ++a) {
    const long long cnt = (long long)g.K[a] * g.L[a];
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < cnt;
         idx += (long long)gridDim.x * blockDim.x) {
      const int ki = (int)(idx / g.L[a]);
      const int l = (int)(idx % g.L[a]);
      int k;
      if (a == 2) k = ki;
      else k = (g.K[a] == 1) ? 0 : ki - N / 2;
      long long j = ((long long)k * (long long)(g.box_lo[a] + l)) % n_g;
      if (j < 0) j += n_g;
      double sn, cs;
      sincospi(-2.0 * (double)j / (double)n_g, &sn, &cs);
      tw[g.tw_off[a] + idx] = make_double2(cs, sn);
    }
  }
}

cudaError_t launch_twiddles(const WinTable& tab, const WinTable* dtab, double2* tw, cudaStream_t s) {
  k_twiddles<<<dim3(16, tab.P), 256, 0, s>>>(dtab, tw);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- window polynomials
// One thread per tap o: Chebyshev interpolation of f_o(t) = phi(t + m - 1 - o), t in [0,1], at
// kPolyLen Chebyshev nodes (exact sinh form of App. A), converted to monomials in
// x = 2t - 1.  f_o is sampled with the analytic (untruncated) window: on t in [0,1] the distance
// |delta| never exceeds m, so this is the window itself.
__global__ void k_window_poly(int m, double beta, double* __restrict__ coef) {
  const int o = threadIdx.x;
  if (o >= 2 * m) return;
  constexpr int L = kPolyLen;
  double f[L], a[L], c[L], Tp[L], Tc[L], Tn[L];
  for (int j = 0; j < L; ++j) {
    const double xn = cospi(((double)j + 0.5) / L);
    const double delta = 0.5 * (xn + 1.0) + (double)(m - 1 - o);
    const double s = (double)m * m - delta * delta;
    if (s > 0.0) {
      const double q = sqrt(s);
      f[j] = sinh(beta * q) / (kPi * q);
    } else {
      f[j] = beta / kPi;  // limit q -> 0
    }
  }
  for (int k = 0; k < L; ++k) {
    double acc = 0.0;
    for (int j = 0; j < L; ++j) acc += f[j] * cospi((double)k * ((double)j + 0.5) / L);
    a[k] = acc * 2.0 / L;
  }
  a[0] *= 0.5;
  for (int k = 0; k < L; ++k) { c[k] = 0.0; Tp[k] = 0.0; Tc[k] = 0.0; }
  Tp[0] = 1.0;  // T_0
  Tc[1] = 1.0;  // T_1
  c[0] += a[0];
  c[1] += a[1];
  for (int k = 2; k < L; ++k) {
    Tn[0] = -Tp[0];
    for (int q = 1; q < L; ++q) Tn[q] = 2.0 * Tc[q - 1] - Tp[q];
    for (int q = 0; q < L; ++q) c[q] += a[k] * Tn[q];
    for (int q = 0; q < L; ++q) { Tp[q] = Tc[q]; Tc[q] = Tn[q]; }
  }
  for (int k = 0; k < L; ++k) coef[o * L + k] = c[k];
}

cudaError_t launch_window_poly(int m, double beta, double* coef, cudaStream_t s) {
  k_window_poly<<<1, 32, 0, s>>>(m, beta, coef);
  return cudaGetLastError();
}

}  // namespace akm
