// Microbenchmark: SM throughput of F2F.F64.F32 (exact float -> double) and
// DADD on B200, elements per clock per SM (K1 pooling sums bf16 rows in f64).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(const float* in, double* out, int iters, long long* cyc) {
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = in[(threadIdx.x + i) & 255];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("" : "+f"(f[i]));
      if (MODE == 0) acc[i] += static_cast<double>(f[i]);    // F2F + DADD
      if (MODE == 1) acc[i] += static_cast<double>(i) * 0.5;  // DADD only (constant)
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* in; double* out; long long* cyc;
  cudaMalloc(&in, 4096); cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 8);
  cudaMemset(in, 0, 4096);
  for (int mode = 0; mode < 2; ++mode) {
    const int iters = 4000, threads = 1024;
    for (int r = 0; r < 2; ++r) {
      if (mode == 0) kern<0><<<148, threads>>>(in, out, iters, cyc); else kern<1><<<148, threads>>>(in, out, iters, cyc);
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.1f elements/clk/SM\n", mode == 0 ? "F2F.F64.F32 + DADD" : "DADD", (double)iters * 8 * threads / c);
  }
  return 0;
}
