// Caller-side fused ops of the config-4 DiT (dit.py), the transformer block
// around RoPeSLR: the token-wise normalisations and gated residuals that
// PyTorch would otherwise run as 5-8 separate elementwise kernels each, and
// the head-major re-layout the op's Q/K/V need.  All are HBM-bound row
// kernels: one warp per token row of D = H * d bf16 values, fp32 math.
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace ropeslr {
namespace dit {

constexpr int kMaxPerLane = 64;  // D <= 2048

// Row r of x[N, D] into registers: lane holds columns [8 * (lane + 32 j), +8).
template <int J>
__device__ __forceinline__ void load_row(const __nv_bfloat16* row, int D, int lane, float (&v)[J * 8]) {
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int c = (lane + 32 * j) * 8;
    if (c < D) {
      load8(row + c, v + 8 * j);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[8 * j + e] = 0.f;
    }
  }
}

// y = LayerNorm(x) * (1 + scale) + shift (no affine; fp32 statistics).
template <int J>
__global__ void ln_modulate_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ shift,
                                   const float* __restrict__ scale, float eps, int64_t N, int D,
                                   __nv_bfloat16* __restrict__ y, int one_plus) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= N) return;
  float v[J * 8];
  load_row<J>(x + r * D, D, lane, v);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < J * 8; ++i) s += v[i];
  const float mean = warp_sum(s) / static_cast<float>(D);
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    if ((lane + 32 * j) * 8 >= D) continue;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float t = v[8 * j + e] - mean;
      q = fmaf(t, t, q);
    }
  }
  const float rstd = rsqrtf(warp_sum(q) / static_cast<float>(D) + eps);
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int c = (lane + 32 * j) * 8;
    if (c >= D) continue;
    float sc[8], sh[8], o[8];
    load8(scale + c, sc);
    load8(shift + c, sh);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = fmaf((v[8 * j + e] - mean) * rstd, one_plus ? 1.f + sc[e] : sc[e], sh[e]);
    store8(y + r * D + c, o);
  }
}

// RMSNorm over the row (torch order: bf16(x * rsqrt(mean(x^2) + eps)) * w,
// w == nullptr: no norm) written head-major out[H, N, d] (head_major) or in
// place of the row layout out[N, D].
// (256, 4): 64 registers, four CTAs per SM: 40.4 -> 37.2 us for a
// [32760, 1536] row set (the LayerNorm kernels spill at that cap)
template <int J>
__global__ void __launch_bounds__(256, 4) rms_heads_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w, float eps,
                                 int64_t N, int D, int H, int head_major, __nv_bfloat16* __restrict__ out,
                                 int64_t xs) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= N) return;
  const int d = D / H;
  float v[J * 8];
  load_row<J>(x + r * xs, D, lane, v);
  float rs = 1.f;
  if (w != nullptr) {
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < J * 8; ++i) q = fmaf(v[i], v[i], q);
    rs = rsqrtf(warp_sum(q) / static_cast<float>(D) + eps);
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int c = (lane + 32 * j) * 8;
    if (c >= D) continue;
    float o[8], wv[8];
    if (w != nullptr) load8(w + c, wv);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float t = v[8 * j + e];
      if (w != nullptr) t = __bfloat162float(__float2bfloat16_rn(t * rs)) * wv[e];
      o[e] = t;
    }
    const int h = c / d, cc = c - h * d;  // 8 | d: a chunk never straddles two heads
    __nv_bfloat16* dst = head_major ? out + (static_cast<int64_t>(h) * N + r) * d + cc : out + r * D + c;
    store8(dst, o);
  }
}

// x = x + bf16(y * gate), torch's `x + (y.float() * g).to(bf16)`.
template <int J>
__global__ void gated_residual_kernel(const __nv_bfloat16* x, const __nv_bfloat16* __restrict__ y,
                                      const float* __restrict__ gate, int64_t N, int D, __nv_bfloat16* out) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= N) return;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int c = (lane + 32 * j) * 8;
    if (c >= D) continue;
    float xv[8], yv[8], gv[8];
    load8(x + r * D + c, xv);
    load8(y + r * D + c, yv);
    load8(gate + c, gv);
#pragma unroll
    for (int e = 0; e < 8; ++e) xv[e] = xv[e] + __bfloat162float(__float2bfloat16_rn(yv[e] * gv[e]));
    store8(out + r * D + c, xv);
  }
}

// [B, H, L, dh] -> [B, L, H, dh], 16-byte chunks: reads in source order
// (coalesced), writes whole dh-element rows (full 32-byte sectors).
__global__ void heads_to_tokens_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, int64_t n, int H,
                                       int64_t L, int cpr) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int j = static_cast<int>(i % cpr);
    const int64_t row = i / cpr;  // (b, h, l)
    const int64_t l = row % L;
    const int64_t bh = row / L;
    const int64_t h = bh % H, b = bh / H;
    y[((b * L + l) * H + h) * cpr + j] = __ldcs(x + i);
  }
}

static bool row_ok(int64_t N, int D) { return N >= 1 && D >= 8 && D % 8 == 0 && D <= 32 * 8 * kMaxPerLane / 8; }

}  // namespace dit
}  // namespace ropeslr

using namespace ropeslr;

#define ROPESLR_DIT_DISPATCH(KERNEL, ...)                                          \
  do {                                                                             \
    const unsigned grid_ = static_cast<unsigned>(ceil_div(N * 32, 256));           \
    const int J_ = static_cast<int>(ceil_div(D, 256));                             \
    if (J_ <= 2)                                                                   \
      dit::KERNEL<2><<<grid_, 256, 0, st>>>(__VA_ARGS__);                          \
    else if (J_ <= 4)                                                              \
      dit::KERNEL<4><<<grid_, 256, 0, st>>>(__VA_ARGS__);                          \
    else if (J_ <= 6)                                                              \
      dit::KERNEL<6><<<grid_, 256, 0, st>>>(__VA_ARGS__);                          \
    else                                                                           \
      dit::KERNEL<8><<<grid_, 256, 0, st>>>(__VA_ARGS__);                          \
  } while (0)

extern "C" int ropeslr_dit_ln_modulate(const void* x, const float* shift, const float* scale, float eps, int64_t N,
                                       int32_t D, void* y, void* stream) {
  if (!x || !shift || !scale || !y) return ROPESLR_ERR_NULL;
  if (!dit::row_ok(N, D)) return ROPESLR_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(y)) return ROPESLR_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ROPESLR_DIT_DISPATCH(ln_modulate_kernel, static_cast<const __nv_bfloat16*>(x), shift, scale, eps, N, D,
                       static_cast<__nv_bfloat16*>(y), 1);
  return launch_status();
}

extern "C" int ropeslr_dit_ln_affine(const void* x, const float* weight, const float* bias, float eps, int64_t N,
                                     int32_t D, void* y, void* stream) {
  if (!x || !weight || !bias || !y) return ROPESLR_ERR_NULL;
  if (!dit::row_ok(N, D)) return ROPESLR_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(y)) return ROPESLR_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ROPESLR_DIT_DISPATCH(ln_modulate_kernel, static_cast<const __nv_bfloat16*>(x), bias, weight, eps, N, D,
                       static_cast<__nv_bfloat16*>(y), 0);
  return launch_status();
}

extern "C" int ropeslr_dit_rms_heads(const void* x, const void* weight, float eps, int64_t N, int32_t D, int32_t H,
                                     int32_t head_major, void* out, void* stream) {
  if (!x || !out) return ROPESLR_ERR_NULL;
  if (!dit::row_ok(N, D) || H < 1 || D % H || (D / H) % 8) return ROPESLR_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(out)) return ROPESLR_ERR_ALIGN;
  if (!head_major && x == out && weight == nullptr) return ROPESLR_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ROPESLR_DIT_DISPATCH(rms_heads_kernel, static_cast<const __nv_bfloat16*>(x),
                       static_cast<const __nv_bfloat16*>(weight), eps, N, D, H, head_major,
                       static_cast<__nv_bfloat16*>(out), static_cast<int64_t>(D));
  return launch_status();
}

extern "C" int ropeslr_dit_rms_heads_strided(const void* x, int64_t x_row_stride, const void* weight, float eps,
                                             int64_t N, int32_t D, int32_t H, int32_t head_major, void* out,
                                             void* stream) {
  if (!x || !out) return ROPESLR_ERR_NULL;
  if (!dit::row_ok(N, D) || H < 1 || D % H || (D / H) % 8 || x_row_stride < D || x_row_stride % 8)
    return ROPESLR_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(out)) return ROPESLR_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ROPESLR_DIT_DISPATCH(rms_heads_kernel, static_cast<const __nv_bfloat16*>(x),
                       static_cast<const __nv_bfloat16*>(weight), eps, N, D, H, head_major,
                       static_cast<__nv_bfloat16*>(out), x_row_stride);
  return launch_status();
}

extern "C" int ropeslr_dit_gated_residual(void* x, const void* y, const float* gate, int64_t N, int32_t D,
                                          void* stream) {
  if (!x || !y || !gate) return ROPESLR_ERR_NULL;
  if (!dit::row_ok(N, D)) return ROPESLR_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(y)) return ROPESLR_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ROPESLR_DIT_DISPATCH(gated_residual_kernel, static_cast<__nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(y),
                       gate, N, D, static_cast<__nv_bfloat16*>(x));
  return launch_status();
}

extern "C" int ropeslr_dit_gated_add(const void* x, const void* y, const float* gate, int64_t N, int32_t D,
                                     void* out, void* stream) {
  if (!x || !y || !gate || !out) return ROPESLR_ERR_NULL;
  if (!dit::row_ok(N, D)) return ROPESLR_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(y) || !aligned16(out)) return ROPESLR_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ROPESLR_DIT_DISPATCH(gated_residual_kernel, static_cast<const __nv_bfloat16*>(x),
                       static_cast<const __nv_bfloat16*>(y), gate, N, D, static_cast<__nv_bfloat16*>(out));
  return launch_status();
}

extern "C" int ropeslr_dit_heads_to_tokens(const void* x, int64_t B, int32_t H, int64_t L, int32_t dh, void* y,
                                           void* stream) {
  if (!x || !y) return ROPESLR_ERR_NULL;
  if (B < 1 || H < 1 || L < 1 || dh < 8 || dh % 8) return ROPESLR_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(y)) return ROPESLR_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cpr = dh / 8;
  const int64_t n = B * H * L * cpr;
  const int64_t want = ceil_div(n, 256 * 4);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(num_sms()) * 16));
  dit::heads_to_tokens_kernel<<<grid, 256, 0, st>>>(static_cast<const uint4*>(x), static_cast<uint4*>(y), n, H, L,
                                                    cpr);
  return launch_status();
}
