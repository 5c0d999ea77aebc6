// Verifies the register fragment layout of mma.sync.aligned.m8n8k4.row.col.f64 on sm_100a:
//   A (8x4, row):  a = A[lane >> 2][lane & 3]
//   B (4x8, col):  b = B[lane & 3][lane >> 2]
//   C (8x8):       c{0,1} = C[lane >> 2][2 * (lane & 3) + {0,1}]
// and measures DMMA vs DFMA co-issue.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_layout.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k_layout(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x;
  double a = A[(lane >> 2) * 4 + (lane & 3)];
  double b = B[(lane & 3) * 8 + (lane >> 2)];
  double c0 = 0.0, c1 = 0.0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  C[(lane >> 2) * 8 + 2 * (lane & 3)] = c0;
  C[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = c1;
}

__global__ void k_mixed(double* out, int iters, int mode) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
  double f[8];
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; f[i] = i; }
  for (int it = 0; it < iters; ++it) {
    if (mode & 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    if (mode & 2) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
  if (s == 1234.5) out[0] = s;
}

int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i; hB[i] = 0.5 * i - 3.0; }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += hA[i * 4 + k] * hB[k * 8 + j];
      ref[i * 8 + j] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  k_layout<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("layout max abs err = %g (%s)\n", err, err == 0 ? "OK" : "MISMATCH");
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* out; cudaMalloc(&out, 8);
  for (int mode = 1; mode <= 3; ++mode) {
    int iters = 4000;
    k_mixed<<<148 * 4, 256>>>(out, 10, mode);
    cudaEventRecord(e0);
    k_mixed<<<148 * 4, 256>>>(out, iters, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 0;
    if (mode & 1) fl += 2.0 * 256 * 8 * iters * (148.0 * 4 * 8);
    if (mode & 2) fl += 2.0 * 64 * iters * (148.0 * 4 * 256);
    printf("mode %d (1=DMMA 2=DFMA 3=both): %.3f ms  %.2f TFLOP/s\n", mode, ms, fl / ms / 1e9);
  }
  return 0;
}
