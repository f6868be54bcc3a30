// Microbenchmark: SM throughput of the K2 softmax element sequence and of
// its parts on B200 (elements per clock per SM).  One CTA per SM, 16 warps
// (the softmax warps of sparse_attn_tc_kernel).  Each element: s*scale - m
// (FFMA2), exp2 (3 MUFU : 1 FMA-pipe polynomial per 4 pairs), running sum
// (FADD2), bf16x2 pack (F2FP); variants drop or replace one part.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../paper_2605_20659_b200/csrc/sm100_ptx.cuh"
using namespace ropeslr::sm100;

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
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
// round-to-nearest-even-ish bf16x2 pack on the integer pipe: add 0x7fff +
// lsb, keep the high halves (PRMT)
__device__ __forceinline__ uint32_t pack_int(float a, float b) {
  uint32_t ua = __float_as_uint(a) + 0x8000u, ub = __float_as_uint(b) + 0x8000u;
  return __byte_perm(ua, ub, 0x7632);
}

template <int MODE>
__global__ void kern(const float* in, uint32_t* out, int iters, long long* cyc) {
  uint32_t s[32];
  for (int i = 0; i < 32; ++i) s[i] = __float_as_uint(in[(threadIdx.x + i) & 255]);
  float sc = in[300], m = in[301];
  __shared__ uint32_t holder;
  if (threadIdx.x < 32) {
    tmem_alloc(&holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // P goes to TMEM as in the kernel: lane = row of this warp, 16 columns per
  // warp slot (16 warps -> 4 column slots per lane quarter)
  const uint32_t taddr = holder + (((threadIdx.x >> 5) & 3) * 32 << 16) + (threadIdx.x >> 7) * 16;
  float2 sum2 = make_float2(0.f, 0.f);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    m = fmaf(m, 0.99999994f, 1e-7f);  // loop-carried: the element work cannot be hoisted
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float2 x2 = __ffma2_rn(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])),
                             make_float2(sc, sc), make_float2(-m, -m));
      float2 e2;
      if (MODE == 6) {
        e2 = x2;  // no exp
      } else if ((i % 4) < (MODE == 5 ? 0 : 1)) {
        e2 = poly2(x2);
      } else {
        e2.x = ex2a(x2.x);
        e2.y = ex2a(x2.y);
      }
      if (MODE != 2) sum2 = __fadd2_rn(sum2, e2);
      if (MODE == 1) {
        pk[i] = __float_as_uint(e2.x) ^ __float_as_uint(e2.y);
      } else if (MODE == 3) {
        pk[i] = pack_int(e2.x, e2.y);
      } else {
        __nv_bfloat162 hb = __floats2bfloat162_rn(e2.x, e2.y);
        pk[i] = *reinterpret_cast<uint32_t*>(&hb);
      }
    }
    tmem_st16(taddr, pk);
  }
  long long t1 = clock64();
  tmem_wait_st();
  uint32_t back[16];
  tmem_ld16(taddr, back);
  tmem_wait_ld();
  acc = back[threadIdx.x & 15];
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(holder, 512);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(sum2.x + sum2.y);
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* in;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&in, 4096);
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  float h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = -0.01f * (i % 97);
  h[300] = 0.127f;
  h[301] = 1.5f;
  cudaMemcpy(in, h, 4096, cudaMemcpyHostToDevice);
  const char* names[] = {"full (F2FP pack)", "no pack", "no sum", "int pack", "-", "all MUFU", "no exp"};
  for (int warps : {8, 16}) {
    for (int mode : {0, 1, 2, 3, 5, 6}) {
      int iters = 2000;
      auto launch = [&]() {
        switch (mode) {
          case 0: kern<0><<<148, warps * 32>>>(in, out, iters, cyc); break;
          case 1: kern<1><<<148, warps * 32>>>(in, out, iters, cyc); break;
          case 2: kern<2><<<148, warps * 32>>>(in, out, iters, cyc); break;
          case 3: kern<3><<<148, warps * 32>>>(in, out, iters, cyc); break;
          case 5: kern<5><<<148, warps * 32>>>(in, out, iters, cyc); break;
          case 6: kern<6><<<148, warps * 32>>>(in, out, iters, cyc); break;
        }
      };
      launch();
      cudaDeviceSynchronize();
      launch();
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double elems = (double)iters * 32 * warps * 32;  // per SM
      printf("warps/SM %2d  %-18s %7.2f elements/clk/SM  (%.0f clk per 128x128 tile)\n", warps, names[mode],
             elems / c, 16384.0 / (elems / c));
    }
  }
  return 0;
}
