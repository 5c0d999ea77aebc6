// Instantiations of the interpolation kernels for d = 2, 2m = 16 (see interp_impl.cuh).
#include "interp_impl.cuh"

namespace akm {
cudaError_t launch_interp_d2_t16(const WinTable* dtab, const WorkItem* items, int n_items, const WorkItem* items_bin,
                              int n_items_bin, int Fb1, int Fb2, bool sparse, const double* u_sorted, const int* perm,
                              const double* H, int ops, int r, int r0, int rc, double* part, long long n,
                              const void* tma, cudaStream_t s) {
  return launch_interp_dt<2, 16>(dtab, items, n_items, items_bin, n_items_bin, Fb1, Fb2, sparse, u_sorted, perm, H, ops, r,
                                 r0, rc, part, n, tma, s);
}
}  // namespace akm
