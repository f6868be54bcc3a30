// Microbenchmark: L2 -> SM bandwidth of the K2 access pattern on B200.
// 148 persistent CTAs each stream 32 KiB K/V block tiles (two 128x64 bf16
// TMA boxes, 128-byte swizzle) of one head's [L, 128] slab, in a random
// block order, through a ring of NST stages with no compute: the ceiling
// that K/V re-reads put on the sparse-attention kernel.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_2605_20659_b200/csrc/sm100_ptx.cuh"
using namespace ropeslr::sm100;

constexpr int BLK = 128;
constexpr int TILE = BLK * 128 * 2;

template <int NST>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const int* order,
                                                      int tiles_per_cta, int nb, int heads, long long* cyc,
                                                      int evict_last) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * TILE);
  uint64_t* empty = full + NST;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = evict_last ? policy_evict_last() : policy_evict_normal();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < tiles_per_cta; ++i) {
      const int s = i % NST;
      mbar_wait(&empty[s], ((i / NST) & 1) ^ 1);
      const int g = blockIdx.x * tiles_per_cta + i;
      const int head = (g / (tiles_per_cta * 4)) % heads;  // ~4 CTAs' worth of tiles per head window
      const int kb = order[g % (1 << 20)] % nb;
      mbar_arrive_expect_tx(&full[s], TILE);
      tma_load_3d_hint(smem + s * TILE, &tm, &full[s], 0, kb * BLK, head, pol);
      tma_load_3d_hint(smem + s * TILE + BLK * 128, &tm, &full[s], 64, kb * BLK, head, pol);
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < tiles_per_cta; ++i) {
      const int s = i % NST;
      mbar_wait(&full[s], (i / NST) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const int heads = 8, L = 118912, nb = L / BLK;
  void* buf;
  cudaMalloc(&buf, (size_t)heads * L * 128 * 2);
  cudaMemset(buf, 0, (size_t)heads * L * 128 * 2);
  std::vector<int> h(1 << 20);
  srand(1);
  for (auto& x : h) x = rand();
  int* order;
  cudaMalloc(&order, h.size() * 4);
  cudaMemcpy(order, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  CUtensorMap tm;
  cuuint64_t dims[3] = {128, (cuuint64_t)L, (cuuint64_t)heads};
  cuuint64_t strides[2] = {256, (cuuint64_t)L * 256};
  cuuint32_t box[3] = {64, BLK, 1}, es[3] = {1, 1, 1};
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  int evict_last = 1;
  auto encode = [&]() {
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  encode();
  const int tiles = 4000;
  auto run = [&](auto kern, int nst) {
    const int smem = nst * TILE + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<148, 64, smem>>>(tm, order, tiles, nb, heads, cyc, evict_last);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> c(148);
      cudaMemcpy(c.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (auto v : c) mx = v > mx ? v : mx;
      const double bytes = 148.0 * tiles * TILE;
      printf("promo %d evict_last %d NST %d rep %d: %.3f ms  %.2f TB/s  %.0f B/clk (SM clk)  %.0f clk per 32 KiB tile per SM\n", (int)promo, evict_last, nst, rep, ms,
             bytes / ms / 1e9, bytes / mx, (double)mx / tiles);
    }
  };
  run(stream_kernel<2>, 2);
  run(stream_kernel<3>, 3);
  run(stream_kernel<4>, 4);
  run(stream_kernel<6>, 6);
  evict_last = 0;
  run(stream_kernel<4>, 4);
  for (auto pr : {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B}) {
    promo = pr;
    encode();
    evict_last = 1;
    run(stream_kernel<4>, 4);
  }
  return 0;
}
