// FP64 pipe / FP64 tensor (DMMA) / L2 RED.ADD.F64 / smem throughput probes on sm_100a.
// Used once to derive the "alu" roofline denominator reported by bench.py.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void red_kernel(double* buf, size_t nbuf, int iters) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it) {
    size_t idx = (tid + it * stride) % nbuf;
    atomicAdd(buf + idx, 1.0);
  }
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clockRate %d kHz smemPerBlockOptin %zu L2 %d\n", p.name, p.multiProcessorCount, clk_khz,
         p.sharedMemPerBlockOptin, p.l2CacheSize);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    for (int blocksPerSM : {4, 8}) {
      int iters = 20000; const int CH = 8;
      dim3 g(sms * blocksPerSM), b(256);
      dfma_kernel<CH><<<g, b>>>(out, 100, 1.0000001, 1e-7);
      cudaEventRecord(e0);
      dfma_kernel<CH><<<g, b>>>(out, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * CH * (double)iters * g.x * b.x;
      printf("DFMA  blocks/SM %d: %.3f ms  %.2f TFLOP/s  (%.1f DFMA/clk/SM at %d MHz nominal)\n", blocksPerSM, ms,
             fl / ms / 1e9, fl / 2 / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
    }
    for (int blocksPerSM : {4, 8}) {
      int iters = 4000;
      dim3 g(sms * blocksPerSM), b(256);
      dmma_kernel<<<g, b>>>(out, 100);
      cudaEventRecord(e0);
      dmma_kernel<<<g, b>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 256 * 8 * (double)iters * g.x * (b.x / 32);
      printf("DMMA  blocks/SM %d: %.3f ms  %.2f TFLOP/s\n", blocksPerSM, ms, fl / ms / 1e9);
    }
    {
      size_t nbuf = (size_t)1 << 22;  // 32 MB of doubles, L2-resident
      double* buf; CK(cudaMalloc(&buf, nbuf * 8)); cudaMemset(buf, 0, nbuf * 8);
      int iters = 64; dim3 g(sms * 8), b(256);
      red_kernel<<<g, b>>>(buf, nbuf, 4);
      cudaEventRecord(e0);
      red_kernel<<<g, b>>>(buf, nbuf, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)iters * g.x * b.x;
      printf("RED.F64 spread addresses: %.3f ms  %.2f Gop/s  (%.1f per clk chip-wide at nominal)\n", ms, ops / ms / 1e6,
             ops / (ms * 1e-3) / (clk_khz * 1e3));
      cudaFree(buf);
    }
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
