// Microbenchmark: per-SM throughput of MUFU ex2, the FMA-pipe exp2
// polynomial and FFMA2 on B200.  Each thread runs a long unrolled loop of
// independent operations on 16 registers; we report elements per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float2 poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f); x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 q = __ffma2_rn(make_float2(0.0551f, 0.0551f), f, make_float2(0.2426f, 0.2426f));
  q = __ffma2_rn(q, f, make_float2(0.6932f, 0.6932f));
  q = __ffma2_rn(q, f, make_float2(0.99993f, 0.99993f));
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}

__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }

template <int MODE>
__global__ void kern(float* out, int iters, long long* cyc) {
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) { v[i] = ex2a(v[i]) - 1.0f; v[i + 1] = ex2a(v[i + 1]) - 1.0f; }
      if (MODE == 1) { float2 r = poly2(make_float2(v[i], v[i + 1])); v[i] = r.x - 1.0f; v[i + 1] = r.y - 1.0f; }
      if (MODE == 2) { float2 r = __ffma2_rn(make_float2(v[i], v[i + 1]), make_float2(0.999f, 0.999f), make_float2(-0.001f, -0.001f)); v[i] = r.x; v[i + 1] = r.y; }
      if (MODE == 4) {  // pack fp32 pair -> bf16x2, ex2.bf16x2 (P stays packed)
        __nv_bfloat162 hb = __floats2bfloat162_rn(v[i], v[i + 1]);
        uint32_t y = ex2bf2(*reinterpret_cast<uint32_t*>(&hb));
        v[i] = __uint_as_float(y) ; v[i + 1] = v[i + 1] * 0.5f;
      }
      if (MODE == 5) {
        __half2 hh = __floats2half2_rn(v[i], v[i + 1]);
        uint32_t y = ex2h2(*reinterpret_cast<uint32_t*>(&hh));
        v[i] = __uint_as_float(y) ; v[i + 1] = v[i + 1] * 0.5f;
      }
      if (MODE == 3) {  // 3 MUFU : 1 poly mix per 4 pairs (the p14 softmax mix)
        if ((i >> 1) % 4 == 3) { float2 r = poly2(make_float2(v[i], v[i + 1])); v[i] = r.x - 1.0f; v[i + 1] = r.y - 1.0f; }
        else { v[i] = ex2a(v[i]) - 1.0f; v[i + 1] = ex2a(v[i + 1]) - 1.0f; }
      }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4 * 4); cudaMalloc(&cyc, 8);
  const char* names[] = {"MUFU ex2", "poly ex2 (pair)", "FFMA2", "3:1 mix", "bf16x2 ex2", "f16x2 ex2"};
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 6; ++mode) {
      int iters = 2000;
      auto launch = [&]() {
        if (mode == 0) kern<0><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 1) kern<1><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 2) kern<2><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 3) kern<3><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 4) kern<4><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 5) kern<5><<<148, warps * 32>>>(out, iters, cyc);
      };
      launch(); cudaDeviceSynchronize();
      launch(); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double elems = (double)iters * 16 * warps * 32;  // per SM
      printf("warps/SM %2d  %-16s %7.2f elements/clk/SM\n", warps, names[mode], elems / c);
    }
  }
  return 0;
}
