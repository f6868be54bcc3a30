// Stage-I training step (SURVEY.md 8f "next" #3): the per-row chains of the
// fused forward / backward of mechanism.py:426-488 (mechanism._fused_forward,
// _rms_backward, _fused_backward) around the float32 GEMMs of training.py.
//
// Rows are head-major float32 [H, L, d] (row = h * L + l); one warp per row,
// V = d / 32 values per lane (lane-major, so every load is one coalesced
// 128-byte line per value slot).  Parameter-gradient reductions over tokens
// are written as per-CTA partial vectors and summed in a fixed order by
// ropeslr_stage1_reduce, so a step is deterministic.
//
//   pre:      x_hat = x + alpha_h * pe (mechanism.py:429-432), and the
//             per-head partial gate logit x_hat . w_g (mechanism.py:434)
//   gate:     g = sigmoid(sum_h partial + b_g)
//   rows:     o = sigmoid(z2); y_lr = RMS(o) * rms_lr; y_sp = RMS(o_sp) * rms_sp;
//             diff = y_sp + g * y_lr - target; loss; d rms_sparse, d rms_lowrank,
//             d g (per row), d z2 (in place of z2) (mechanism.py:437-488, 519-526)
//   gate_bwd: d_zg = (sum_h d g) * g * (1 - g) and its sum (d b_g)
//   dsig:     t *= h * (1 - h)               (the sigmoid derivative of H1)
//   xgrad:    d_x_hat += d_zg * w_g (with PE); d alpha = sum d_x_hat * pe;
//             d w_g = sum x_hat * d_zg   (per head)
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "ropeslr_b200.h"

namespace ropeslr {
namespace s1 {

constexpr int kWarps = 8;  // rows in flight per CTA

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float sigm(float z) { return 1.f / (1.f + __expf(-z)); }

template <int V>
__global__ void __launch_bounds__(kWarps * 32) pre_kernel(const float* __restrict__ x, const float* __restrict__ pe,
                                                          const float* __restrict__ alpha,
                                                          const float* __restrict__ w_g, int64_t L, int64_t rows,
                                                          float* __restrict__ xh, float* __restrict__ gpart) {
  constexpr int d = V * 32;
  const int lane = threadIdx.x & 31;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5); row < rows;
       row += static_cast<int64_t>(gridDim.x) * kWarps) {
    const int64_t h = row / L;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + 32 * i;
      float v = x[row * d + c];
      if (pe) v = v + alpha[h * d + c] * pe[row * d + c];
      xh[row * d + c] = v;
      s += v * w_g[h * d + c];
    }
    s = warp_sum(s);
    if (lane == 0) gpart[row] = s;
  }
}

// b_g from the argument, or from device memory when b_g_dev is set (a
// captured training step reads the current bias).
__global__ void gate_kernel(const float* __restrict__ gpart, int H, int64_t L, float b_g,
                            const double* __restrict__ b_g_dev, float* __restrict__ g) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const float b = b_g_dev != nullptr ? static_cast<float>(*b_g_dev) : b_g;
  float s = 0.f;
  for (int h = 0; h < H; ++h) s += gpart[h * L + l];
  g[l] = sigm(s + b);
}

// Per-CTA partials: red[blockIdx][0][d] = sum gh * u_sp (d rms_sparse),
// red[blockIdx][1][d] = sum dy * u_lr (d rms_lowrank); loss_part[blockIdx] =
// sum diff^2 (float64).
template <int V>
__global__ void __launch_bounds__(kWarps * 32) rows_kernel(float* __restrict__ z2, const float* __restrict__ o_sp,
                                                           const float* __restrict__ target,
                                                           const float* __restrict__ g,
                                                           const float* __restrict__ rms_sp,
                                                           const float* __restrict__ rms_lr, float eps, float gscale,
                                                           int64_t L, int64_t rows, float* __restrict__ dgpart,
                                                           float* __restrict__ red, double* __restrict__ loss_part) {
  constexpr int d = V * 32;
  __shared__ float sred[kWarps][2][d];
  __shared__ double sloss[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float a_sp[V], a_lr[V], wsp[V], wlr[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    a_sp[i] = a_lr[i] = 0.f;
    wsp[i] = rms_sp[lane + 32 * i];
    wlr[i] = rms_lr[lane + 32 * i];
  }
  double loss = 0.0;
  // one row in flight ahead: the next row's z2 / o_sp / target loads are
  // issued before this row's reductions
  const int64_t rstep = static_cast<int64_t>(gridDim.x) * kWarps;
  int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  float nz[V], ns[V], nt[V];
  if (row < rows) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      nz[i] = z2[row * d + lane + 32 * i];
      ns[i] = o_sp[row * d + lane + 32 * i];
      nt[i] = target[row * d + lane + 32 * i];
    }
  }
  for (; row < rows; row += rstep) {
    const int64_t l = row % L;
    const float gl = g[l];
    float o[V], os[V], tg[V];
    float so = 0.f, ss = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      o[i] = sigm(nz[i]);
      os[i] = ns[i];
      tg[i] = nt[i];
      so += o[i] * o[i];
      ss += os[i] * os[i];
    }
    if (row + rstep < rows) {
      const int64_t nr = row + rstep;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        nz[i] = z2[nr * d + lane + 32 * i];
        ns[i] = o_sp[nr * d + lane + 32 * i];
        nt[i] = target[nr * d + lane + 32 * i];
      }
    }
    const float inv_lr = rsqrtf(warp_sum(so) / d + eps);
    const float inv_sp = rsqrtf(warp_sum(ss) / d + eps);
    float dg = 0.f, dot = 0.f, dsq = 0.f;
    float dy[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + 32 * i;
      const float u_lr = o[i] * inv_lr, u_sp = os[i] * inv_sp;
      const float y_lr = u_lr * wlr[i];
      const float diff = u_sp * wsp[i] + gl * y_lr - tg[i];
      dsq += diff * diff;
      const float gh = diff * gscale;
      a_sp[i] += gh * u_sp;
      dg += gh * y_lr;
      dy[i] = gh * gl;
      a_lr[i] += dy[i] * u_lr;
      dot += dy[i] * wlr[i] * o[i];
    }
    loss += warp_sum_d(static_cast<double>(dsq));
    dg = warp_sum(dg);
    dot = warp_sum(dot);
    if (lane == 0) dgpart[row] = dg;
    const float k3 = inv_lr * inv_lr * inv_lr * dot / d;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + 32 * i;
      const float d_o = dy[i] * wlr[i] * inv_lr - o[i] * k3;
      z2[row * d + c] = d_o * o[i] * (1.f - o[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    sred[warp][0][lane + 32 * i] = a_sp[i];
    sred[warp][1][lane + 32 * i] = a_lr[i];
  }
  if (lane == 0) sloss[warp] = loss;
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * d; e += blockDim.x) {
    const int k = e / d, c = e % d;
    float s = 0.f;
    for (int w = 0; w < kWarps; ++w) s += sred[w][k][c];
    red[(static_cast<int64_t>(blockIdx.x) * 2 + k) * d + c] = s;
  }
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s += sloss[w];
    loss_part[blockIdx.x] = s;
  }
}

__global__ void gate_bwd_kernel(const float* __restrict__ dgpart, const float* __restrict__ g, int H, int64_t L,
                                float* __restrict__ dzg, double* __restrict__ bg_part) {
  __shared__ double sb[256 / 32];
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (l < L) {
    float s = 0.f;
    for (int h = 0; h < H; ++h) s += dgpart[h * L + l];
    const float gl = g[l];
    const float z = s * gl * (1.f - gl);
    dzg[l] = z;
    v = z;
  }
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += sb[w];
    bg_part[blockIdx.x] = s;
  }
}

__global__ void dsig_kernel(float* __restrict__ t, const float* __restrict__ hh, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n / 4; e += stride) {
    float4 a = reinterpret_cast<float4*>(t)[e];
    const float4 b = reinterpret_cast<const float4*>(hh)[e];
    a.x *= b.x * (1.f - b.x);
    a.y *= b.y * (1.f - b.y);
    a.z *= b.z * (1.f - b.z);
    a.w *= b.w * (1.f - b.w);
    reinterpret_cast<float4*>(t)[e] = a;
  }
  for (int64_t e = (n / 4) * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride)
    t[e] *= hh[e] * (1.f - hh[e]);
}

// grid (nblk, H): CTA (b, h) walks rows of head h.  red[h][b][0][d] = sum
// d_x_hat * pe (d alpha), red[h][b][1][d] = sum x_hat * d_zg (d w_g).
template <int V>
__global__ void __launch_bounds__(kWarps * 32) xgrad_kernel(const float* __restrict__ dxh,
                                                            const float* __restrict__ xh,
                                                            const float* __restrict__ pe,
                                                            const float* __restrict__ dzg,
                                                            const float* __restrict__ w_g, int64_t L,
                                                            float* __restrict__ red) {
  constexpr int d = V * 32;
  __shared__ float sred[kWarps][2][d];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t h = blockIdx.y;
  float a_al[V], a_wg[V], wg[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    a_al[i] = a_wg[i] = 0.f;
    wg[i] = w_g[h * d + lane + 32 * i];
  }
  const int64_t lstep = static_cast<int64_t>(gridDim.x) * kWarps;
  int64_t l = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  float nx[V] = {}, nd[V] = {}, np[V] = {}, nzg = 0.f;
  auto fetch = [&](int64_t ll) {
    const int64_t row = h * L + ll;
    nzg = dzg[ll];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + 32 * i;
      nx[i] = xh[row * d + c];
      if (pe) {
        nd[i] = dxh[row * d + c];
        np[i] = pe[row * d + c];
      }
    }
  };
  if (l < L) fetch(l);
  for (; l < L; l += lstep) {
    const float z = nzg;
    float cx[V], cd[V], cp[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      cx[i] = nx[i];
      cd[i] = nd[i];
      cp[i] = np[i];
    }
    if (l + lstep < L) fetch(l + lstep);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      a_wg[i] += cx[i] * z;
      if (pe) a_al[i] += (cd[i] + z * wg[i]) * cp[i];
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    sred[warp][0][lane + 32 * i] = a_al[i];
    sred[warp][1][lane + 32 * i] = a_wg[i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * d; e += blockDim.x) {
    const int k = e / d, c = e % d;
    float s = 0.f;
    for (int w = 0; w < kWarps; ++w) s += sred[w][k][c];
    red[((h * gridDim.x + blockIdx.x) * 2 + k) * d + c] = s;
  }
}

// out[(o * groups + j) * width + c] += sum over p of parts[((o * nparts + p) * groups + j) * width + c]
// (the per-CTA partials of rows_kernel: outer 1; of xgrad_kernel: outer H).
// A CTA owns 32 outputs; warp w sums parts w, w + 8, ... in order, then the
// eight warp sums are added in warp order: a fixed order, so deterministic.
__global__ void __launch_bounds__(256) reduce_kernel(const float* __restrict__ parts, int outer, int nparts,
                                                     int groups, int width, float* __restrict__ out) {
  __shared__ float sp[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const int total = outer * groups * width;
  float s = 0.f;
  if (e < total) {
    const int o = e / (groups * width), j = (e / width) % groups, c = e % width;
    const float* src = parts + (static_cast<int64_t>(o) * nparts * groups + j) * width + c;
    const int64_t step = static_cast<int64_t>(groups) * width;
#pragma unroll 4
    for (int p = warp; p < nparts; p += 8) s += src[p * step];
  }
  sp[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && e < total) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += sp[w][lane];
    out[e] += t;
  }
}

int vec_of(int64_t d) { return d == 32 ? 1 : d == 64 ? 2 : d == 128 ? 4 : 0; }  // the op's head dims

}  // namespace s1
}  // namespace ropeslr

using namespace ropeslr;

#define S1_SWITCH(V_, CALL)  \
  switch (V_) {              \
    case 1: {                \
      constexpr int V = 1;   \
      CALL;                  \
    } break;                 \
    case 2: {                \
      constexpr int V = 2;   \
      CALL;                  \
    } break;                 \
    case 4: {                \
      constexpr int V = 4;   \
      CALL;                  \
    } break;                 \
    default:                 \
      break;                 \
  }

static unsigned row_grid(int64_t rows) {
  const int64_t want = ceil_div(rows, s1::kWarps);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;  // grid-stride: 64 warps per SM
  return static_cast<unsigned>(want < cap ? want : cap);
}

extern "C" int ropeslr_stage1_supported(int64_t d) { return s1::vec_of(d) != 0; }

extern "C" int ropeslr_stage1_rows_blocks(int64_t H, int64_t L) { return static_cast<int>(row_grid(H * L)); }

static int stage1_pre(int64_t H, int64_t L, int64_t d, const float* x, const float* pe, const float* alpha,
                      const float* w_g, float b_g, const double* b_g_dev, float* xh, float* gpart, float* g,
                      void* stream) {
  const int V = s1::vec_of(d);
  if (V == 0 || H < 1 || L < 1) return ROPESLR_ERR_SHAPE;
  if (!x || !w_g || !xh || !gpart || !g || (pe && !alpha)) return ROPESLR_ERR_NULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t rows = H * L;
  S1_SWITCH(V, (s1::pre_kernel<V><<<row_grid(rows), s1::kWarps * 32, 0, st>>>(x, pe, alpha, w_g, L, rows, xh,
                                                                                gpart)));
  s1::gate_kernel<<<static_cast<unsigned>(ceil_div(L, 256)), 256, 0, st>>>(gpart, static_cast<int>(H), L, b_g,
                                                                            b_g_dev, g);
  return launch_status();
}

extern "C" int ropeslr_stage1_pre(int64_t H, int64_t L, int64_t d, const float* x, const float* pe,
                                  const float* alpha, const float* w_g, float b_g, float* xh, float* gpart,
                                  float* g, void* stream) {
  return stage1_pre(H, L, d, x, pe, alpha, w_g, b_g, nullptr, xh, gpart, g, stream);
}

extern "C" int ropeslr_stage1_pre_dev(int64_t H, int64_t L, int64_t d, const float* x, const float* pe,
                                      const float* alpha, const float* w_g, const double* b_g, float* xh,
                                      float* gpart, float* g, void* stream) {
  if (!b_g) return ROPESLR_ERR_NULL;
  return stage1_pre(H, L, d, x, pe, alpha, w_g, 0.f, b_g, xh, gpart, g, stream);
}

extern "C" int ropeslr_stage1_rows(int64_t H, int64_t L, int64_t d, float* z2, const float* o_sp,
                                   const float* target, const float* g, const float* rms_sp, const float* rms_lr,
                                   float eps, float gscale, float* dgpart, float* red, double* loss_part,
                                   void* stream) {
  const int V = s1::vec_of(d);
  if (V == 0 || H < 1 || L < 1) return ROPESLR_ERR_SHAPE;
  if (!z2 || !o_sp || !target || !g || !rms_sp || !rms_lr || !dgpart || !red || !loss_part) return ROPESLR_ERR_NULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t rows = H * L;
  S1_SWITCH(V, (s1::rows_kernel<V><<<row_grid(rows), s1::kWarps * 32, 0, st>>>(
                   z2, o_sp, target, g, rms_sp, rms_lr, eps, gscale, L, rows, dgpart, red, loss_part)));
  return launch_status();
}

extern "C" int ropeslr_stage1_gate_bwd(int64_t H, int64_t L, const float* dgpart, const float* g, float* dzg,
                                       double* bg_part, void* stream) {
  if (H < 1 || L < 1) return ROPESLR_ERR_SHAPE;
  if (!dgpart || !g || !dzg || !bg_part) return ROPESLR_ERR_NULL;
  s1::gate_bwd_kernel<<<static_cast<unsigned>(ceil_div(L, 256)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dgpart, g, static_cast<int>(H), L, dzg, bg_part);
  return launch_status();
}

extern "C" int ropeslr_stage1_dsig(float* t, const float* h1, int64_t n, void* stream) {
  if (n < 0) return ROPESLR_ERR_SHAPE;
  if (n == 0) return ROPESLR_OK;
  if (!t || !h1) return ROPESLR_ERR_NULL;
  if (!aligned16(t) || !aligned16(h1)) return ROPESLR_ERR_ALIGN;
  const int64_t want = ceil_div(ceil_div(n, 4), 256);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  s1::dsig_kernel<<<static_cast<unsigned>(want < cap ? want : cap), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      t, h1, n);
  return launch_status();
}

extern "C" int ropeslr_stage1_xgrad_blocks(int64_t H, int64_t L) {
  const int64_t per = ceil_div(static_cast<int64_t>(num_sms()) * 8, H);
  const int64_t want = ceil_div(L, s1::kWarps);
  return static_cast<int>(per < want ? per : want);
}

extern "C" int ropeslr_stage1_xgrad(int64_t H, int64_t L, int64_t d, const float* dxh, const float* xh,
                                    const float* pe, const float* dzg, const float* w_g, float* red, void* stream) {
  const int V = s1::vec_of(d);
  if (V == 0 || H < 1 || L < 1) return ROPESLR_ERR_SHAPE;
  if (!dxh || !xh || !dzg || !w_g || !red) return ROPESLR_ERR_NULL;
  dim3 grid(static_cast<unsigned>(ropeslr_stage1_xgrad_blocks(H, L)), static_cast<unsigned>(H));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  S1_SWITCH(V, (s1::xgrad_kernel<V><<<grid, s1::kWarps * 32, 0, st>>>(dxh, xh, pe, dzg, w_g, L, red)));
  return launch_status();
}

extern "C" int ropeslr_stage1_reduce(const float* parts, int32_t outer, int32_t nparts, int32_t groups,
                                     int32_t width, float* out, void* stream) {
  if (outer < 1 || nparts < 1 || groups < 1 || width < 1) return ROPESLR_ERR_SHAPE;
  if (!parts || !out) return ROPESLR_ERR_NULL;
  const int n = outer * groups * width;
  s1::reduce_kernel<<<static_cast<unsigned>(ceil_div(n, 32)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      parts, outer, nparts, groups, width, out);
  return launch_status();
}
