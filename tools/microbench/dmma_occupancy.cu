// DMMA (mma.sync.m8n8k4.f64) throughput vs warps per SM and independent accumulators per warp,
// and the cost of DFMA chains issued next to DMMA traffic.  Informs the spreading / interpolation
// kernels' warp layout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_occupancy dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ACC>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

// warps [0, nmma) run DMMAs, the rest run CH independent DFMA chains of length iters*16
template <int ACC, int CH>
__global__ void mixed_kernel(double* out, int iters, int nmma_warps) {
  const int warp = threadIdx.x >> 5;
  if (warp < nmma_warps) {
    double a = threadIdx.x * 1e-3, b = 0.5;
    double c[ACC][2];
#pragma unroll
    for (int i = 0; i < ACC; ++i) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < ACC; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[0] = s;
  } else {
    double v[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) v[q] = threadIdx.x * 1e-9 + q;
    for (int it = 0; it < iters * 4; ++it)
#pragma unroll
      for (int q = 0; q < CH; ++q) v[q] = fma(v[q], 1.0000001, 1e-7);
    double s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += v[q];
    if (s == 1234.5) out[1] = s;
  }
}

template <int ACC>
int run_dmma(int sms, int threads, int blocks_per_sm, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  const int iters = 2000;
  dim3 g(sms * blocks_per_sm), b(threads);
  dmma_kernel<ACC><<<g, b>>>(out, 10);
  cudaEventRecord(e0);
  dmma_kernel<ACC><<<g, b>>>(out, iters);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 256 * ACC * (double)iters * g.x * (b.x / 32);
  printf("DMMA acc/warp %2d  warps/SM %2d: %.2f TFLOP/s\n", ACC, threads / 32 * blocks_per_sm, fl / ms / 1e9);
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 16));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    run_dmma<8>(sms, 128, 1, out, e0, e1);
    run_dmma<16>(sms, 128, 1, out, e0, e1);
    run_dmma<32>(sms, 128, 1, out, e0, e1);
    run_dmma<36>(sms, 128, 1, out, e0, e1);
    run_dmma<8>(sms, 256, 1, out, e0, e1);
    run_dmma<16>(sms, 256, 1, out, e0, e1);
    run_dmma<32>(sms, 256, 1, out, e0, e1);
    run_dmma<16>(sms, 512, 1, out, e0, e1);
    run_dmma<8>(sms, 512, 2, out, e0, e1);
  }
  // DMMA warps + DFMA-chain warps in one CTA of 8 warps
  for (int nm : {4, 8}) {
    const int iters = 2000;
    mixed_kernel<32, 4><<<sms, 256>>>(out, 10, nm);
    cudaEventRecord(e0);
    mixed_kernel<32, 4><<<sms, 256>>>(out, iters, nm);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dm = 2.0 * 256 * 32 * (double)iters * sms * nm;
    const double df = 2.0 * 4 * 4 * (double)iters * sms * (8 - nm) * 32;
    printf("mixed: %d DMMA warps (32 acc) + %d DFMA warps (4 chains): %.3f ms, DMMA %.2f TF/s, DFMA %.2f TF/s\n", nm,
           8 - nm, ms, dm / ms / 1e9, df / ms / 1e9);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
