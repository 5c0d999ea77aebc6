// spread_det.cu -- deterministic spreading (akm_set_deterministic; SURVEY.md §4 tier 3 "determinism").
//
// The footprint flushes of the spreading kernels are the only order-dependent sums on the product
// path (reading R13: float64 atomics).  In deterministic mode they add v * 2^S_c as three signed
// 40-bit limbs (akm_internal.cuh det_add) with 64-bit integer atomics: integer addition is exact and
// associative, so the limb sums do not depend on the order the work items finish in.
//   S_wc = 112 - ceil(log2(n * max_j |v_jc| * W^d_w)) per window w, W >= max |window tap| (the Kaiser-Bessel taps
//   reach ~1e12 per axis at m = 6; W is bounded by the sum of |coefficients| of the tap polynomials):
//   every grid value and every single contribution is at most n max|v| W^d, so |v w| 2^S_c < 2^112
//   fits the three limbs (< 2^119) with room; a limb sum stays below 2^63 for up to 2^23
//   contributions per node.  The resolution 2^-S_c = n max|v| W^d 2^-112 is ~1e-34 of the largest
//   possible node value, far below float64 rounding of the outputs.
// The conversion adds the three limb sums in a fixed order (deterministic; its rounding error is
// ~1e-16 of the node value).
#include <cuda_runtime.h>

#include <algorithm>

#include "akm_internal.cuh"

namespace akm {

// column max |v| as the bit pattern of a non-negative double (monotone as unsigned): atomicMax is
// order-independent
__global__ void k_det_colmax(const double* __restrict__ V, long long ldv, long long n, int r,
                             unsigned long long* __restrict__ colmax) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * r;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / r;
    const int c = (int)(idx - i * r);
    const double a = fabs(V[i * ldv + c]);
    if (a > 0.0) atomicMax(colmax + c, (unsigned long long)__double_as_longlong(a));
  }
}

// S[w * r + c] = 112 - ceil(log2(n max|v_c|)) - wbits_w
__global__ void k_det_scale(long long n, int r, DetWin dw, const unsigned long long* __restrict__ colmax,
                            int* __restrict__ S) {
  for (int q = threadIdx.x; q < dw.P * r; q += blockDim.x) {
    const int w = q / r, c = q - w * r;
    const double m = __longlong_as_double((long long)colmax[c]);
    int e = 0;
    if (m > 0.0 && isfinite(m)) {
      int ex;
      frexp(m * (double)n, &ex);  // m n < 2^ex
      e = 112 - ex - dw.wbits[w];
    }
    S[q] = e;
  }
}

__global__ void k_det_to_double(const unsigned long long* __restrict__ limbs, const int* __restrict__ S, long long stride,
                                int r, DetWin dw, double* __restrict__ grid) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < stride;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long tap = idx / r;
    const int c = (int)(idx - tap * r);
    int w = 0;
    while (w + 1 < dw.P && tap >= dw.tap_off[w + 1]) ++w;
    const long long l0 = (long long)limbs[idx], l1 = (long long)limbs[stride + idx],
                    l2 = (long long)limbs[2 * stride + idx];
    const int e = S[w * r + c];
    grid[idx] = ldexp((double)l2, 80 - e) + ldexp((double)l1, 40 - e) + ldexp((double)l0, -e);
  }
}

cudaError_t launch_det_prepare(const double* V, long long ldv, long long n, int r, const DetWin& dw,
                               unsigned long long* colmax, int* S, unsigned long long* limbs, long long stride,
                               cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * r, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(limbs, 0, sizeof(unsigned long long) * 3 * (size_t)stride, s);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    const long long blocks = std::min<long long>((n * r + 255) / 256, 148 * 8);
    k_det_colmax<<<(unsigned)blocks, 256, 0, s>>>(V, ldv, n, r, colmax);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_det_scale<<<1, 256, 0, s>>>(n, r, dw, colmax, S);
  return cudaGetLastError();
}

cudaError_t launch_det_finish(const unsigned long long* limbs, const int* S, long long stride, int r,
                              const DetWin& dw, double* grid, cudaStream_t s) {
  if (stride <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>((stride + 255) / 256, 148 * 8);
  k_det_to_double<<<(unsigned)blocks, 256, 0, s>>>(limbs, S, stride, r, dw, grid);
  return cudaGetLastError();
}

}  // namespace akm
