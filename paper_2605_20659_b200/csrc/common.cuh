// Shared helpers for the RoPeSLR sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ropeslr_b200.h"

namespace ropeslr {

constexpr double kMassSlack = 1e-12;     // decomposition.py:102
constexpr float kLinearFloor = 1e-8f;    // mechanism.py:347

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Real token count of flat block `b` (the last block is ragged).
__host__ __device__ inline int block_size(int64_t L, int block, int64_t b) {
  int64_t r = L - b * block;
  return (int)(r < block ? r : block);
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Numerically stable logistic, mechanism.py:27-30.
__device__ __forceinline__ float sigmoidf_stable(float x) {
  float t = __expf(-fabsf(x));
  return x >= 0.f ? 1.f / (1.f + t) : t / (1.f + t);
}

// Load 8 consecutive elements as float.
__device__ __forceinline__ void load8(const float* p, float* o) {
  float4 a = *reinterpret_cast<const float4*>(p);
  float4 b = *reinterpret_cast<const float4*>(p + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* o) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}

__device__ __forceinline__ void store8(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* v) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

template <typename T>
__device__ __forceinline__ float warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Host: map a CUDA error to a status; the error is kept per thread for
// ropeslr_last_cuda_error().
void note_cuda_error(cudaError_t e);  // abi.cu
inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) note_cuda_error(e);
  return e == cudaSuccess ? ROPESLR_OK : ROPESLR_ERR_LAUNCH;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int num_sms();  // cached per device (abi.cu)

// ORs `bit` into *flag (stream-ordered) when any of the n values is NaN or
// infinite; no-op for a NULL flag (abi.cu).
int scan_nonfinite(const void* a, bool f64, int64_t n, uint32_t* flag, uint32_t bit, cudaStream_t st);

// The A/B switches of the kernel experiments, read
// from the environment once per process (abi.cu), not on every call.
struct Tuning {
  bool k2_online;      // ROPESLR_K2=online: the running-max K2 kernel
  bool pair64;         // ROPESLR_PAIR64=0 turns the paired block-64 tiles off
  bool schedule;       // ROPESLR_SCHEDULE=0 turns the longest-first unit schedule off
  bool kv_evict_last;  // ROPESLR_KV_EVICT_LAST=0 drops the K/V L2 evict-last hint
  char scores;         // ROPESLR_SCORES: 'f' CUDA-core f64, 'd' unpipelined DMMA, 0 default
  bool rope_tma;       // ROPESLR_ROPE_TMA=0: the row-bulk-copy RoPE kernel
  bool linear_simt;    // ROPESLR_LINEAR=simt: the CUDA-core linear compensator
  bool screen;         // ROPESLR_SCREEN=0: K1 top-k from float64 scores of every pair (no screening)
  bool keep_bitonic;   // ROPESLR_KEEP_SORT=bitonic: the round-1 keep-mode selection (bitonic sort per row)
  bool pairs64;        // ROPESLR_PAIRS64=0: block-64 K2 units of one query block (no query-block pairs)
};
const Tuning& tuning();

inline bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

}  // namespace ropeslr
