// interp.cu -- dispatch of the NFFT interpolation kernels (kernel template in
// interp_impl.cuh) and the epilogue S7: Y = sigma_f^2 S + sigma_eps^2 V, dY_ell = sigma_f^2 S^ell,
// dY_sf = 2 sigma_f S, with the windows summed in a fixed order.
#include <cstdlib>

#include "akm_internal.cuh"

namespace akm {

cudaError_t launch_interp_d1_t8(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);
cudaError_t launch_interp_d1_t12(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);
cudaError_t launch_interp_d1_t16(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);
cudaError_t launch_interp_d2_t8(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);
cudaError_t launch_interp_d2_t12(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);
cudaError_t launch_interp_d2_t16(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);
cudaError_t launch_interp_d3_t8(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);
cudaError_t launch_interp_d3_t12(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);
cudaError_t launch_interp_d3_t16(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s);


// Largest instantiated RHS chunk not exceeding r_remaining.
int interp_rc_for(int r_remaining) {
  if (r_remaining >= 11) return 11;
  if (r_remaining >= 4) return 4;
  if (r_remaining >= 2) return 2;
  return 1;
}

cudaError_t launch_interp(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                          int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm, const double* H,
                          int d, int taps, int ops, int r, int r0, int rc, double* part, long long n, const void* tma,
                          cudaStream_t s) {
  if (n_items <= 0 && n_items_bin <= 0) return cudaSuccess;
  if (d == 1 && taps == 8)
    return launch_interp_d1_t8(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  if (d == 1 && taps == 12)
    return launch_interp_d1_t12(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  if (d == 1 && taps == 16)
    return launch_interp_d1_t16(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  if (d == 2 && taps == 8)
    return launch_interp_d2_t8(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  if (d == 2 && taps == 12)
    return launch_interp_d2_t12(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  if (d == 2 && taps == 16)
    return launch_interp_d2_t16(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  if (d == 3 && taps == 8)
    return launch_interp_d3_t8(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  if (d == 3 && taps == 12)
    return launch_interp_d3_t12(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  if (d == 3 && taps == 16)
    return launch_interp_d3_t16(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops,
                                   r, r0, rc, part, n, tma, s);
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- TMA tensor maps of H (k_interp_mma)
// Per 3-D window w < kTmaWin: a 3-D map over the window's box of H with dims (values per node V,
// axis-2 nodes L2, (axis-0, axis-1) rows L0*L1), element pitch 8 bytes, node pitch 8V bytes (V even:
// 16-byte multiples), box (LDH, 2m, 2m) with LDH the kernel's padded plane row (values past V are
// outside the tensor: TMA writes zeros there).  The driver entry point is looked up at run time.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

size_t interp_tma_maps_bytes() { return sizeof(TmaMaps); }

bool interp_tma_build(const WinTable& tab, const double* H, int ops, int r, void* maps) {
  static const bool off = getenv("AKM_INTERP_TMA") && atoi(getenv("AKM_INTERP_TMA")) == 0;
  const int V = ops * r;
  if (off || (V % 2) != 0 || tab.P > kTmaWin) return false;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  TmaMaps* tm = static_cast<TmaMaps*>(maps);
  const int taps = 2 * tab.m;
  const cuuint32_t ldh = (cuuint32_t)mma_ld(((V + 7) / 8) * 8);
  for (int w = 0; w < tab.P; ++w) {
    const WinGeom& g = tab.w[w];
    if (g.d != 3) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)V, (cuuint64_t)g.L[2], (cuuint64_t)g.L[0] * g.L[1]};
    const cuuint64_t strides[2] = {(cuuint64_t)V * 8, (cuuint64_t)g.L[2] * V * 8};
    const cuuint32_t box[3] = {ldh, (cuuint32_t)taps, (cuuint32_t)taps};
    const cuuint32_t estr[3] = {1, 1, 1};
    void* base = const_cast<double*>(H + g.tap_off * (long long)V);
    if (enc(&tm->m[w], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

// ---------------------------------------------------------------- epilogue (S7)
// part[(w*n + i)*ops + slot][r] holds S^{w,op}; sums over windows in fixed order (deterministic).
__global__ void k_epilogue(long long n, int P, int r, int ops, const double* __restrict__ part,
                           const double* __restrict__ V, long long ldv, double sigma_f, double sigma_eps,
                           double* __restrict__ Y, double* __restrict__ dYl, double* __restrict__ dYsf,
                           long long ldy, int slotK, int slotL) {
  const long long total = n * r;
  const double sf2 = sigma_f * sigma_f, se2 = sigma_eps * sigma_eps;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / r;
    const int c = (int)(idx % r);
    double sK = 0.0, sL = 0.0;
    for (int w = 0; w < P; ++w) {
      const double* pp = part + (((long long)w * n + i) * ops) * r + c;
      if (slotK >= 0) sK += pp[(long long)slotK * r];
      if (slotL >= 0) sL += pp[(long long)slotL * r];
    }
    if (Y) Y[i * ldy + c] = sf2 * sK + se2 * V[i * ldv + c];
    if (dYl) dYl[i * ldy + c] = sf2 * sL;
    if (dYsf) dYsf[i * ldy + c] = 2.0 * sigma_f * sK;
  }
}

cudaError_t launch_epilogue(long long n, int P, int r, int ops, const double* part, const double* V, long long ldv,
                            double sigma_f, double sigma_eps, double* Y, double* dYl, double* dYsf, long long ldy,
                            int slotK, int slotL, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  long long blocks = (n * r + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_epilogue<<<(int)blocks, 256, 0, s>>>(n, P, r, ops, part, V, ldv, sigma_f, sigma_eps, Y, dYl, dYsf, ldy, slotK,
                                         slotL);
  return cudaGetLastError();
}

// cross product (akm_kernel_cross_mvm): Yt[i - n_src][c] = sigma_f^2 sum_w S^w[i][c] for the target
// rows i >= n_src (no noise term: a target is not a training point), windows in a fixed order
__global__ void k_epilogue_cross(long long n, long long n_src, int P, int r, int ops, int slotK,
                                 const double* __restrict__ part, double sigma_f, double* __restrict__ Yt,
                                 long long ldy) {
  const long long total = (n - n_src) * r;
  const double sf2 = sigma_f * sigma_f;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long t = idx / r, i = n_src + t;
    const int c = (int)(idx - t * r);
    double sK = 0.0;
    for (int w = 0; w < P; ++w) sK += part[(((long long)w * n + i) * ops + slotK) * r + c];
    Yt[t * ldy + c] = sf2 * sK;
  }
}

cudaError_t launch_epilogue_cross(long long n, long long n_src, int P, int r, int ops, int slotK, const double* part,
                                  double sigma_f, double* Yt, long long ldy, cudaStream_t s) {
  const long long total = (n - n_src) * r;
  if (total <= 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_epilogue_cross<<<(int)blocks, 256, 0, s>>>(n, n_src, P, r, ops, slotK, part, sigma_f, Yt, ldy);
  return cudaGetLastError();
}

__global__ void k_scaled_copy(long long n, int r, double alpha, const double* __restrict__ V, long long ldv,
                              double* __restrict__ Y, long long ldy) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * r;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / r;
    const int c = (int)(idx % r);
    Y[i * ldy + c] = alpha * V[i * ldv + c];
  }
}

cudaError_t launch_scaled_copy(long long n, int r, double alpha, const double* V, long long ldv, double* Y,
                               long long ldy, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  long long blocks = (n * r + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_scaled_copy<<<(int)blocks, 256, 0, s>>>(n, r, alpha, V, ldv, Y, ldy);
  return cudaGetLastError();
}

}  // namespace akm
