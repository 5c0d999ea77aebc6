// krylov.cu -- the config-5 driver: one evaluation of the preconditioned
// objective Z~(theta) of eq. (1.4) with M = diag(Khat) = c I (reading R11):
//   CG for alpha = Khat^{-1} y from x0 = 0, fixed iteration count;
//   SLQ for tr logm(M^{-1} Khat): Lanczos on S = Khat / c from q_1 = z_i / ||z_i|| with
//   full reorthogonalisation (classical Gram-Schmidt twice), breakdown rule of reading R14, and
//   Gauss quadrature ||z||^2 sum_j tau_j^2 log theta_j from the tridiagonal T.
// Every Krylov step applies Khat to one n x R block (R = 1 + n_z; column 0 the CG direction,
// columns 1.. the Lanczos vectors) through the NFFT path (plan.cu run_mvm); the vector work here
// is O(n R) per step plus O(j n R) for the reorthogonalisation, all in fixed-order reductions.
//
// Layout: every vector block is n x R row-major (like V); Q holds one n x R slab per Lanczos step
// (column 0 unused).  KrylovState (device) carries every scalar, so the whole evaluation is
// enqueued without host synchronisation.
#include "akm_internal.cuh"

namespace akm {

// ---------------------------------------------------------------- column sums
// part[blk][c][0] = sum_k A[k][c] B[k][c],  part[blk][c][1] = sum_k B[k][c]^2 over the rows of this
// block (grid-stride).  blockDim = 32 * R: thread t owns column c = t % R and row slot t / R.
__global__ void k_col2_partial(long long n, int R, const double* __restrict__ A, const double* __restrict__ B,
                               double* __restrict__ part) {
  extern __shared__ double sm[];  // [2][32][R]
  const int t = threadIdx.x, c = t % R, slot = t / R;
  double s0 = 0.0, s1 = 0.0;
  for (long long k = (long long)blockIdx.x * 32 + slot; k < n; k += (long long)gridDim.x * 32) {
    const double b = B[k * R + c];
    s0 = fma(A[k * R + c], b, s0);
    s1 = fma(b, b, s1);
  }
  sm[slot * R + c] = s0;
  sm[32 * R + slot * R + c] = s1;
  __syncthreads();
  if (t < 2 * R) {
    const int q = t / R, cc = t % R;
    double acc = 0.0;
    for (int s = 0; s < 32; ++s) acc += sm[q * 32 * R + s * R + cc];
    part[((long long)blockIdx.x * R + cc) * 2 + q] = acc;
  }
}

// sum over the nblk partials of the 2R column sums; one warp per output, lanes over blocks in a
// fixed order and a fixed butterfly (deterministic)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ void col2_final(const double* __restrict__ part, int nblk, int R, double* out /* [R][2] */) {
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int idx = threadIdx.x >> 5; idx < 2 * R; idx += nw) {
    double acc = 0.0;
    for (int b = lane; b < nblk; b += 32) acc += part[(long long)b * 2 * R + idx];
    acc = warp_sum(acc);
    if (lane == 0) out[idx] = acc;
  }
}

// ---------------------------------------------------------------- scalar bookkeeping
struct KrylovState {
  int t;                // current step
  int cg_on;            // CG still iterating
  double c, s2;         // M = c I; S = Khat / c -> s2 = 1/c
  double rz;            // r^T M^{-1} r
  double cg_a, cg_beta;
  double ynorm;
  double sums[2 * kKrMaxR];  // scratch for the column sums
  double alpha[kKrMaxR], wn[kKrMaxR], beta_prev[kKrMaxR], beta_new[kKrMaxR];
  int live[kKrMaxR];    // probe still in the Lanczos recurrence
  int cont[kKrMaxR];    // probe builds q_{t+1} this step
  int steps[kKrMaxR];
  double Ta[kKrMaxR][kKrMaxSteps], Tb[kKrMaxR][kKrMaxSteps];
  double znorm2[kKrMaxR];
  double cg_hist[kKrMaxIters];
  double quad, samples[kKrMaxR];
};

// init: state from the column sums of B = [y | Z] (part of k_col2_partial(B, B)): ||y||^2, ||z_i||^2
__global__ void k_kr_init(KrylovState* st, const double* __restrict__ part, int nblk, int R, double c) {
  col2_final(part, nblk, R, st->sums);
  __syncthreads();
  if (threadIdx.x == 0) {
    const double yy = st->sums[1];
    st->t = 0;
    st->cg_on = yy > 0.0;
    st->c = c;
    st->s2 = 1.0 / c;
    st->rz = yy / c;
    st->ynorm = sqrt(yy);
    st->quad = 0.0;
    st->cg_a = st->cg_beta = 0.0;
  }
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    st->znorm2[i] = st->sums[2 * i + 1];
    st->live[i] = (i > 0) && st->sums[2 * i + 1] > 0.0;
    st->cont[i] = 0;
    st->steps[i] = 0;
    st->beta_prev[i] = 0.0;
    st->alpha[i] = 0.0;
    st->samples[i] = 0.0;
  }
  for (int t = threadIdx.x; t < kKrMaxIters; t += blockDim.x) st->cg_hist[t] = -1.0;  // not run
}

// B = [y | Z] (row-major n x R); y also kept in ybuf
__global__ void k_kr_load(long long n, int R, const double* __restrict__ y, const double* __restrict__ Z, long long ldz,
                          double* __restrict__ B, double* __restrict__ ybuf) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const long long k = e / R;
    const int c = (int)(e % R);
    if (c == 0) {
      B[e] = y[k];
      ybuf[k] = y[k];
    } else {
      B[e] = Z[k * ldz + (c - 1)];
    }
  }
}

// in place on B: column 0 becomes p0 = M^{-1} r0 = y / c (W[:,0] = r0 = y, x = 0); probe columns
// become q_1 = z_i / ||z_i|| (also into Q_0)
__global__ void k_kr_start(long long n, int R, const KrylovState* __restrict__ st, double* __restrict__ B,
                           double* __restrict__ W, double* __restrict__ Q0, double* __restrict__ x) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const long long k = e / R;
    const int c = (int)(e % R);
    const double b = B[e];
    if (c == 0) {
      B[e] = b / st->c;
      W[e] = b;
      Q0[e] = 0.0;
      x[k] = 0.0;
    } else {
      const double q = st->live[c] ? b / sqrt(st->znorm2[c]) : 0.0;
      B[e] = q;
      Q0[e] = q;
      W[e] = 0.0;
    }
  }
}

// after the product KB = Khat B: CG step length and Lanczos alpha_t, ||S q_t||
__global__ void k_kr_after_dots(KrylovState* st, const double* __restrict__ part, int nblk, int R, int cg_iters,
                                int lanczos_steps) {
  col2_final(part, nblk, R, st->sums);
  __syncthreads();
  const int t = st->t;
  if (threadIdx.x == 0) {
    const int on = st->cg_on && t < cg_iters;
    st->cg_on = on;
    st->cg_a = on ? st->rz / st->sums[0] : 0.0;
  }
  for (int i = 1 + threadIdx.x; i < R; i += blockDim.x) {
    int cont = 0;
    if (st->live[i] && t < lanczos_steps) {
      const double a = st->s2 * st->sums[2 * i];
      st->alpha[i] = a;
      st->wn[i] = st->s2 * sqrt(st->sums[2 * i + 1]);
      st->Ta[i][t] = a;
      st->steps[i] = t + 1;
      cont = (t + 1 < lanczos_steps);
      if (!cont) st->live[i] = 0;   // T complete
    } else {
      st->live[i] = 0;
    }
    st->cont[i] = cont;
  }
}

// x += a p; r -= a A p (column 0);  w = S q_t - alpha q_t - beta_{t-1} q_{t-1} (probes)
__global__ void k_kr_update(long long n, int R, const KrylovState* __restrict__ st, const double* __restrict__ B,
                            const double* __restrict__ KB, double* __restrict__ W, const double* __restrict__ Qt,
                            const double* __restrict__ Qtm1, double* __restrict__ x) {
  const double a = st->cg_a, s2 = st->s2;
  const int on = st->cg_on;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const long long k = e / R;
    const int c = (int)(e % R);
    if (c == 0) {
      if (on) {
        x[k] = fma(a, B[e], x[k]);
        W[e] = fma(-a, KB[e], W[e]);
      }
    } else if (st->cont[c]) {
      double w = fma(s2, KB[e], -st->alpha[c] * Qt[e]);
      if (Qtm1) w = fma(-st->beta_prev[c], Qtm1[e], w);
      W[e] = w;
    }
  }
}

// h[j][c] partials: sum_k Q_j[k][c] W[k][c] for j in [j0, j0 + JC) (blockIdx.y = chunk), probes only
constexpr int kProjJC = 8;
__global__ void k_kr_proj_partial(long long n, int R, int nq, const double* __restrict__ Q, long long slab,
                                  const double* __restrict__ W, double* __restrict__ part) {
  extern __shared__ double sm[];  // [JC][S][R], S = blockDim.x / R row slots
  const int t = threadIdx.x, c = t % R, slot = t / R, S = blockDim.x / R;
  const int j0 = blockIdx.y * kProjJC;
  const int jn = min(kProjJC, nq - j0);
  double acc[kProjJC];
#pragma unroll
  for (int jj = 0; jj < kProjJC; ++jj) acc[jj] = 0.0;
  // two rows per iteration: 2 kProjJC independent loads in flight per thread (the kernel is
  // latency-bound at the occupancy its registers allow)
  const long long stride = (long long)gridDim.x * S;
  long long k = (long long)blockIdx.x * S + slot;
  for (; k + stride < n; k += 2 * stride) {
    const long long e0 = k * R + c, e1 = e0 + stride * R;
    const double w0 = W[e0], w1 = W[e1];
    double q0[kProjJC], q1[kProjJC];
#pragma unroll
    for (int jj = 0; jj < kProjJC; ++jj) {
      q0[jj] = jj < jn ? Q[(long long)(j0 + jj) * slab + e0] : 0.0;
      q1[jj] = jj < jn ? Q[(long long)(j0 + jj) * slab + e1] : 0.0;
    }
#pragma unroll
    for (int jj = 0; jj < kProjJC; ++jj) acc[jj] = fma(q1[jj], w1, fma(q0[jj], w0, acc[jj]));
  }
  for (; k < n; k += stride) {
    const long long e = k * R + c;
    const double w = W[e];
#pragma unroll
    for (int jj = 0; jj < kProjJC; ++jj)
      if (jj < jn) acc[jj] = fma(Q[(long long)(j0 + jj) * slab + e], w, acc[jj]);
  }
#pragma unroll
  for (int jj = 0; jj < kProjJC; ++jj) sm[(jj * S + slot) * R + c] = acc[jj];
  __syncthreads();
  for (int idx = t; idx < jn * R; idx += blockDim.x) {
    const int jj = idx / R, cc = idx % R;
    double s = 0.0;
    for (int q = 0; q < S; ++q) s += sm[(jj * S + q) * R + cc];
    part[((long long)blockIdx.x * nq + j0 + jj) * R + cc] = s;
  }
}

// one warp per output h[j][c] (fixed order, as col2_final)
__global__ void k_kr_proj_final(const double* __restrict__ part, int nblk, int nq, int R, double* __restrict__ h) {
  const int lane = threadIdx.x & 31;
  const int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (idx >= nq * R) return;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += part[(long long)b * nq * R + idx];
  s = warp_sum(s);
  if (lane == 0) h[idx] = s;
}

// W[:, c] -= sum_j Q_j[:, c] h[j][c] for probes that continue
__global__ void k_kr_orth_update(long long n, int R, int nq, const KrylovState* __restrict__ st,
                                 const double* __restrict__ Q, long long slab, const double* __restrict__ h,
                                 double* __restrict__ W) {
  extern __shared__ double hs[];  // [nq][R]
  for (int idx = threadIdx.x; idx < nq * R; idx += blockDim.x) hs[idx] = h[idx];
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % R);
    if (c == 0 || !st->cont[c]) continue;
    double w = W[e];
    for (int j = 0; j < nq; ++j) w = fma(-Q[(long long)j * slab + e], hs[j * R + c], w);
    W[e] = w;
  }
}

// norms: ||r||^2 (column 0) and ||w_i||^2 -> CG beta, Lanczos beta_t / breakdown (reading R14)
__global__ void k_kr_after_norms(KrylovState* st, const double* __restrict__ part, int nblk, int R) {
  col2_final(part, nblk, R, st->sums);
  __syncthreads();
  const int t = st->t;
  if (threadIdx.x == 0 && st->cg_on) {
    const double rr = st->sums[1];
    const double rz_new = rr / st->c;
    st->cg_beta = (st->rz > 0.0) ? rz_new / st->rz : 0.0;
    st->rz = rz_new;
    st->cg_hist[t] = sqrt(rr) / st->ynorm;
    if (rz_new == 0.0) st->cg_on = 0;
  }
  for (int i = 1 + threadIdx.x; i < R; i += blockDim.x) {
    if (!st->cont[i]) continue;
    const double b = sqrt(st->sums[2 * i + 1]);
    if (b <= 1e-12 * st->wn[i]) {
      st->cont[i] = 0;
      st->live[i] = 0;
    } else {
      st->Tb[i][t] = b;
      st->beta_new[i] = b;
    }
  }
}

// p = M^{-1} r + beta p into B[:,0]; q_{t+1} = w / beta into Q_{t+1} and B; dead columns zero
__global__ void k_kr_finalize(long long n, int R, KrylovState* __restrict__ st, double* __restrict__ B,
                              const double* __restrict__ W, double* __restrict__ Qn) {
  const double invc = 1.0 / st->c, beta = st->cg_beta;
  const int on = st->cg_on;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % R);
    if (c == 0) {
      B[e] = on ? fma(beta, B[e], W[e] * invc) : 0.0;
    } else if (st->cont[c]) {
      const double q = W[e] / st->beta_new[c];
      B[e] = q;
      Qn[e] = q;
    } else {
      B[e] = 0.0;
    }
  }
}

__global__ void k_kr_advance(KrylovState* st, int R) {
  if (threadIdx.x == 0) st->t += 1;
  for (int i = 1 + threadIdx.x; i < R; i += blockDim.x) {
    if (st->cont[i]) st->beta_prev[i] = st->beta_new[i];
  }
}

// ---------------------------------------------------------------- SLQ quadrature
// Symmetric tridiagonal eigenproblem by implicit QL with Wilkinson-type shifts, tracking only the
// first row of the eigenvector matrix (tau_j); one thread per probe.  This is the textbook implicit
// QL iteration (EISPACK tql2, Bowdler, Martin, Reinsch and Wilkinson 1968; the same loop as the
// widely reprinted "tqli" routine), restated here with the eigenvector update reduced to row 0.
__device__ bool tridiag_eig_first_row(int k, double* d, double* e, double* z) {
  for (int i = 0; i < k; ++i) z[i] = (i == 0) ? 1.0 : 0.0;
  e[k - 1] = 0.0;
  for (int l = 0; l < k; ++l) {
    int iter = 0, mm;
    do {
      for (mm = l; mm < k - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= 2.2e-16 * dd) break;
      }
      if (mm != l) {
        if (iter++ == 100) return false;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool early = false;
        for (i = mm - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          f = z[i + 1];
          z[i + 1] = s * z[i] + c * f;
          z[i] = c * z[i] - s * f;
        }
        if (early) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  return true;
}

__global__ void k_kr_slq(KrylovState* st, int R, int* __restrict__ err) {
  const int i = 1 + threadIdx.x;
  if (i >= R) return;
  const int k = st->steps[i];
  double d[kKrMaxSteps], e[kKrMaxSteps], z[kKrMaxSteps];
  if (k == 0) {
    st->samples[i] = 0.0;
    return;
  }
  for (int j = 0; j < k; ++j) {
    d[j] = st->Ta[i][j];
    e[j] = (j + 1 < k) ? st->Tb[i][j] : 0.0;
  }
  if (!tridiag_eig_first_row(k, d, e, z)) atomicOr(err, 1);
  double s = 0.0;
  for (int j = 0; j < k; ++j) {
    if (!(d[j] > 0.0)) atomicOr(err, 2);
    s += z[j] * z[j] * log(d[j]);
  }
  st->samples[i] = st->znorm2[i] * s;
}

__global__ void k_kr_quad(KrylovState* st, const double* __restrict__ part, int nblk) {
  // part from k_col2_partial with R = 1 over (y, x): sum y x in slot 0
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += part[(long long)b * 2];
    st->quad = acc;
  }
}

// ---------------------------------------------------------------- launchers
static const int kKrBlocks = 296;

size_t kr_state_bytes() { return sizeof(KrylovState); }

cudaError_t launch_kr_col2(long long n, int R, const double* A, const double* B, double* part, cudaStream_t s) {
  k_col2_partial<<<kKrBlocks, 32 * R, sizeof(double) * 64 * R, s>>>(n, R, A, B, part);
  return cudaGetLastError();
}

int kr_blocks() { return kKrBlocks; }

cudaError_t launch_kr_init(void* st, const double* part, int R, double c, cudaStream_t s) {
  k_kr_init<<<1, 256, 0, s>>>((KrylovState*)st, part, kKrBlocks, R, c);
  return cudaGetLastError();
}

static int grid_for(long long total) {
  long long b = (total + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return (int)(b < 1 ? 1 : b);
}

cudaError_t launch_kr_load(long long n, int R, const double* y, const double* Z, long long ldz, double* B,
                           double* ybuf, cudaStream_t s) {
  k_kr_load<<<grid_for(n * R), 256, 0, s>>>(n, R, y, Z, ldz, B, ybuf);
  return cudaGetLastError();
}

cudaError_t launch_kr_start(long long n, int R, const void* st, double* B, double* W, double* Q0, double* x,
                            cudaStream_t s) {
  k_kr_start<<<grid_for(n * R), 256, 0, s>>>(n, R, (const KrylovState*)st, B, W, Q0, x);
  return cudaGetLastError();
}

cudaError_t launch_kr_after_dots(void* st, const double* part, int R, int cg_iters, int lanczos_steps, cudaStream_t s) {
  k_kr_after_dots<<<1, 256, 0, s>>>((KrylovState*)st, part, kKrBlocks, R, cg_iters, lanczos_steps);
  return cudaGetLastError();
}

cudaError_t launch_kr_update(long long n, int R, const void* st, const double* B, const double* KB, double* W,
                             const double* Qt, const double* Qtm1, double* x, cudaStream_t s) {
  k_kr_update<<<grid_for(n * R), 256, 0, s>>>(n, R, (const KrylovState*)st, B, KB, W, Qt, Qtm1, x);
  return cudaGetLastError();
}

cudaError_t launch_kr_reorth(long long n, int R, int nq, const void* st, const double* Q, long long slab, double* W,
                             double* part, double* h, cudaStream_t s) {
  const int chunks = (nq + kProjJC - 1) / kProjJC;
  static std::atomic<unsigned long long> attr_set{0};  // R up to kKrMaxR needs more than the default 48 KB
  if (!optin_done(attr_set)) {
    cudaError_t e = cudaFuncSetAttribute(k_kr_proj_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(double) * kProjJC * 32 * kKrMaxR));
    if (e != cudaSuccess) return e;
    optin_mark(attr_set);
  }
  const int slots = R <= 16 ? 32 : 16;  // block <= 512 threads: the registers of 2 rows in flight fit
  k_kr_proj_partial<<<dim3(kKrBlocks, chunks), slots * R, sizeof(double) * kProjJC * slots * R, s>>>(n, R, nq, Q, slab, W,
                                                                                                  part);
  k_kr_proj_final<<<(nq * R + 7) / 8, 256, 0, s>>>(part, kKrBlocks, nq, R, h);
  k_kr_orth_update<<<grid_for(n * R), 256, sizeof(double) * nq * R, s>>>(n, R, nq, (const KrylovState*)st, Q, slab, h,
                                                                         W);
  return cudaGetLastError();
}

cudaError_t launch_kr_after_norms(void* st, const double* part, int R, cudaStream_t s) {
  k_kr_after_norms<<<1, 256, 0, s>>>((KrylovState*)st, part, kKrBlocks, R);
  return cudaGetLastError();
}

cudaError_t launch_kr_finalize(long long n, int R, void* st, double* B, const double* W, double* Qn, cudaStream_t s) {
  k_kr_finalize<<<grid_for(n * R), 256, 0, s>>>(n, R, (KrylovState*)st, B, W, Qn);
  return cudaGetLastError();
}

cudaError_t launch_kr_advance(void* st, int R, cudaStream_t s) {
  k_kr_advance<<<1, 64, 0, s>>>((KrylovState*)st, R);
  return cudaGetLastError();
}

cudaError_t launch_kr_slq_quad(void* st, int R, const double* part_yx, int* err, cudaStream_t s) {
  k_kr_slq<<<1, 32, 0, s>>>((KrylovState*)st, R, err);
  k_kr_quad<<<1, 32, 0, s>>>((KrylovState*)st, part_yx, kKrBlocks);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- gradient
// eq. (div) needs alpha = Khat^{-1} y and Khat^{-1} z_i: fixed-iteration PCG with
// M = c I from x0 = 0 on every column of the n x R block [y | Z] at once (one block product per
// iteration; the columns are independent recurrences with their own scalars).
struct BcgState {
  double c;
  double rz[kKrMaxR], a[kKrMaxR], beta[kKrMaxR];
  double bnorm[kKrMaxR];                  // ||b_c|| (relative residuals)
  double sums[2 * kKrMaxR];
  double hist[kKrMaxIters];               // column 0 relative residual per iteration
  double out[3][2 * kKrMaxR];             // the gradient dot products (col2 finals)
};

size_t bcg_state_bytes() { return sizeof(BcgState); }

__global__ void k_bcg_init(BcgState* st, const double* __restrict__ part, int nblk, int R, double c) {
  col2_final(part, nblk, R, st->sums);
  __syncthreads();
  if (threadIdx.x == 0) st->c = c;
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    st->rz[i] = st->sums[2 * i + 1] / c;
    st->bnorm[i] = sqrt(st->sums[2 * i + 1]);
    st->a[i] = st->beta[i] = 0.0;
  }
  for (int t = threadIdx.x; t < kKrMaxIters; t += blockDim.x) st->hist[t] = -1.0;
}

// R (residual) = B, P = B / c, X = 0
__global__ void k_bcg_start(long long n, int R, const BcgState* __restrict__ st, const double* __restrict__ B,
                            double* __restrict__ Rr, double* __restrict__ P, double* __restrict__ X) {
  const double invc = 1.0 / st->c;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const double b = B[e];
    Rr[e] = b;
    P[e] = b * invc;
    X[e] = 0.0;
  }
}

// a_c = rz_c / (p_c^T Khat p_c) for live columns (rz_c > 0)
__global__ void k_bcg_after_dots(BcgState* st, const double* __restrict__ part, int nblk, int R) {
  col2_final(part, nblk, R, st->sums);
  __syncthreads();
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const double pkp = st->sums[2 * i];
    st->a[i] = (st->rz[i] > 0.0 && pkp != 0.0) ? st->rz[i] / pkp : 0.0;
  }
}

// X += a P;  R -= a KP
__global__ void k_bcg_update(long long n, int R, const BcgState* __restrict__ st, const double* __restrict__ P,
                             const double* __restrict__ KP, double* __restrict__ Rr, double* __restrict__ X) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e - (e / R) * R);
    const double a = st->a[c];
    X[e] = fma(a, P[e], X[e]);
    Rr[e] = fma(-a, KP[e], Rr[e]);
  }
}

// rz_new = ||r||^2 / c, beta = rz_new / rz; column 0 relative residual into the history
__global__ void k_bcg_after_norms(BcgState* st, const double* __restrict__ part, int nblk, int R, int t) {
  col2_final(part, nblk, R, st->sums);
  __syncthreads();
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    if (!(st->rz[i] > 0.0)) {
      st->beta[i] = 0.0;
      continue;
    }
    const double rr = st->sums[2 * i + 1], rz_new = rr / st->c;
    st->beta[i] = rz_new / st->rz[i];
    st->rz[i] = rz_new;
    if (i == 0) st->hist[t] = sqrt(rr) / st->bnorm[0];
  }
}

// P = R / c + beta P
__global__ void k_bcg_dir(long long n, int R, const BcgState* __restrict__ st, const double* __restrict__ Rr,
                          double* __restrict__ P) {
  const double invc = 1.0 / st->c;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e - (e / R) * R);
    P[e] = fma(st->beta[c], P[e], Rr[e] * invc);
  }
}

// B2 = [alpha | Z]: column 0 from X, the probe columns from B (the original block)
__global__ void k_bcg_grad_rhs(long long n, int R, const double* __restrict__ X, const double* __restrict__ B,
                               double* __restrict__ B2) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * R; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e - (e / R) * R);
    B2[e] = (c == 0) ? X[e] : B[e];
  }
}

__global__ void k_bcg_store(BcgState* st, const double* __restrict__ part, int nblk, int R, int slot) {
  col2_final(part, nblk, R, st->out[slot]);
}

cudaError_t launch_bcg_init(void* st, const double* part, int R, double c, cudaStream_t s) {
  k_bcg_init<<<1, 256, 0, s>>>((BcgState*)st, part, kKrBlocks, R, c);
  return cudaGetLastError();
}
cudaError_t launch_bcg_start(long long n, int R, const void* st, const double* B, double* Rr, double* P, double* X,
                             cudaStream_t s) {
  k_bcg_start<<<grid_for(n * R), 256, 0, s>>>(n, R, (const BcgState*)st, B, Rr, P, X);
  return cudaGetLastError();
}
cudaError_t launch_bcg_after_dots(void* st, const double* part, int R, cudaStream_t s) {
  k_bcg_after_dots<<<1, 256, 0, s>>>((BcgState*)st, part, kKrBlocks, R);
  return cudaGetLastError();
}
cudaError_t launch_bcg_update(long long n, int R, const void* st, const double* P, const double* KP, double* Rr,
                              double* X, cudaStream_t s) {
  k_bcg_update<<<grid_for(n * R), 256, 0, s>>>(n, R, (const BcgState*)st, P, KP, Rr, X);
  return cudaGetLastError();
}
cudaError_t launch_bcg_after_norms(void* st, const double* part, int R, int t, cudaStream_t s) {
  k_bcg_after_norms<<<1, 256, 0, s>>>((BcgState*)st, part, kKrBlocks, R, t);
  return cudaGetLastError();
}
cudaError_t launch_bcg_dir(long long n, int R, const void* st, const double* Rr, double* P, cudaStream_t s) {
  k_bcg_dir<<<grid_for(n * R), 256, 0, s>>>(n, R, (const BcgState*)st, Rr, P);
  return cudaGetLastError();
}
cudaError_t launch_bcg_grad_rhs(long long n, int R, const double* X, const double* B, double* B2, cudaStream_t s) {
  k_bcg_grad_rhs<<<grid_for(n * R), 256, 0, s>>>(n, R, X, B, B2);
  return cudaGetLastError();
}
cudaError_t launch_bcg_store(void* st, const double* part, int R, int slot, cudaStream_t s) {
  k_bcg_store<<<1, 256, 0, s>>>((BcgState*)st, part, kKrBlocks, R, slot);
  return cudaGetLastError();
}
void bcg_offsets(size_t* off_hist, size_t* off_out, size_t* off_bnorm) {
  *off_hist = offsetof(BcgState, hist);
  *off_out = offsetof(BcgState, out);
  *off_bnorm = offsetof(BcgState, bnorm);
}

// host-readable summary (offsets into KrylovState)
void kr_summary_offsets(size_t* off_quad, size_t* off_samples, size_t* off_steps, size_t* off_hist, size_t* off_znorm) {
  *off_quad = offsetof(KrylovState, quad);
  *off_samples = offsetof(KrylovState, samples);
  *off_steps = offsetof(KrylovState, steps);
  *off_hist = offsetof(KrylovState, cg_hist);
  *off_znorm = offsetof(KrylovState, znorm2);
}

}  // namespace akm
