// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion time per
// instruction for M = 128 vs M = 64 (cta_group::1, N = 128 / 64, K = 16, A and
// B from shared memory), one CTA per SM, one issuing thread, all 148 SMs.
// Question: does an M = 64 MMA take half the tensor-pipe time of M = 128
// (block 64 leaves half of a 128-row tile idle)?
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_2605_20659_b200/csrc/sm100_ptx.cuh"
using namespace ropeslr::sm100;

template <int MM, int NN>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  if (threadIdx.x < 32) {
    tmem_alloc(&holder, 256);
    tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  constexpr uint32_t idesc = idesc_bf16_f32(MM, NN, false, false);
  const uint64_t da = desc_sw128(smem_u32(smem), 16, 1024);
  const uint64_t db = desc_sw128(smem_u32(smem + 32768), 16, 1024);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_bf16_ss(tmem, da + kk * 2, db + kk * 2, idesc, kk > 0 ? 1u : 0u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

template <int MM, int NN>
void run(long long* cyc) {
  auto k = mma_loop<MM, NN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 4000;
  k<<<148, 128, 65536>>>(iters, cyc);
  cudaDeviceSynchronize();
  k<<<148, 128, 65536>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (long long v : c) mx = v > mx ? v : mx;
  const double per = (double)mx / (iters * 8.0);
  printf("M=%3d N=%3d K=16: %.1f cycles per MMA, %.0f FLOP/clk/SM (%s)\n", MM, NN, per, 2.0 * MM * NN * 16 / per,
         cudaGetErrorString(e));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<128, 128>(cyc);
  run<64, 128>(cyc);
  run<128, 64>(cyc);
  run<64, 64>(cyc);
  run<128, 256>(cyc);
  return 0;
}
