// K2 (CUDA-core variant): exact softmax attention of each query block over
// the tokens of its selected key blocks (mechanism.py:321-326).
//
// Used for float32 inputs (BASELINE config 0), head dims / block sizes the
// tcgen05 kernel does not cover, and as an independent cross-check of the
// tensor-core kernel in the GPU tests.  One CTA per (bh, query block); each
// warp owns up to 16 query rows and keeps an online-softmax state per row;
// key/value tiles are staged in shared memory in float32.
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"

namespace ropeslr {

template <typename T, int DPL>
__global__ void __launch_bounds__(256) sparse_attn_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                               const T* __restrict__ v, const int32_t* __restrict__ idx,
                                                               int kmax, const int32_t* __restrict__ cnt, int64_t L,
                                                               int block, int nb, const int32_t* __restrict__ perm,
                                                               float scale, float* __restrict__ o_sparse) {
  constexpr int D = DPL * 32;
  constexpr int MAXR = 16;  // rows per warp (block <= 128)
  extern __shared__ float sm[];
  const int blk = block;
  float* Qs = sm;                    // [blk][D]
  float* Ks = Qs + blk * D;          // [blk][D+1]
  float* Vs = Ks + blk * (D + 1);    // [blk][D]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qb = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const int64_t row = bh * nb + qb;
  const int qrows = block_size(L, blk, qb);
  const T* qbase = q + (bh * L + static_cast<int64_t>(qb) * blk) * D;
  for (int e = tid; e < qrows * D; e += 256) Qs[e] = to_f(qbase[e]);

  float m[MAXR], l[MAXR], o[MAXR][DPL];
#pragma unroll
  for (int i = 0; i < MAXR; ++i) {
    m[i] = -INFINITY;
    l[i] = 0.f;
#pragma unroll
    for (int c = 0; c < DPL; ++c) o[i][c] = 0.f;
  }
  const int n = cnt[row];
  const int32_t* irow = idx + row * kmax;
  for (int jb = 0; jb < n; ++jb) {
    const int kb = irow[jb];
    const int krows = block_size(L, blk, kb);
    const T* kbase = k + (bh * L + static_cast<int64_t>(kb) * blk) * D;
    const T* vbase = v + (bh * L + static_cast<int64_t>(kb) * blk) * D;
    __syncthreads();
    for (int e = tid; e < krows * D; e += 256) {
      const int rr = e / D, cc = e % D;
      Ks[rr * (D + 1) + cc] = to_f(kbase[e]);
      Vs[e] = to_f(vbase[e]);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MAXR; ++i) {
      const int r = warp + 8 * i;
      if (r >= qrows) break;
      float s[4];
      float mloc = -INFINITY;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = lane + 32 * u;
        float acc = -INFINITY;
        if (kk < krows) {
          acc = 0.f;
          const float* kr = Ks + kk * (D + 1);
          const float* qr = Qs + r * D;
#pragma unroll 8
          for (int c = 0; c < D; ++c) acc = fmaf(qr[c], kr[c], acc);
          acc *= scale;
        }
        s[u] = acc;
        mloc = fmaxf(mloc, acc);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, off));
      const float mnew = fmaxf(m[i], mloc);
      const float corr = expf(m[i] - mnew);  // 0 on the first block (m = -inf)
      float psum = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s[u] = (lane + 32 * u < krows) ? expf(s[u] - mnew) : 0.f;
        psum += s[u];
      }
      psum = warp_sum(psum);
      l[i] = l[i] * corr + psum;
#pragma unroll
      for (int c = 0; c < DPL; ++c) o[i][c] *= corr;
#pragma unroll 1
      for (int u = 0; u < 4; ++u) {
#pragma unroll 4
        for (int t = 0; t < 32; ++t) {
          const int kk = 32 * u + t;
          if (kk >= krows) break;
          const float p = __shfl_sync(0xffffffffu, s[u], t);
          const float* vr = Vs + kk * D;
#pragma unroll
          for (int c = 0; c < DPL; ++c) o[i][c] = fmaf(p, vr[lane + 32 * c], o[i][c]);
        }
      }
      m[i] = mnew;
    }
  }
#pragma unroll
  for (int i = 0; i < MAXR; ++i) {
    const int r = warp + 8 * i;
    if (r >= qrows) break;
    const int64_t flat = static_cast<int64_t>(qb) * blk + r;
    const int64_t tok = perm ? perm[flat] : flat;
    float* dst = o_sparse + (bh * L + tok) * D;
    const float inv = 1.f / l[i];
#pragma unroll
    for (int c = 0; c < DPL; ++c) dst[lane + 32 * c] = o[i][c] * inv;
  }
}

template <typename T>
static int launch_simt_t(const ropeslr_shape* s, const T* q, const T* k, const T* v, const int32_t* idx, int kmax,
                         const int32_t* cnt, const int32_t* perm, float* o_sparse, cudaStream_t st) {
  const int d = static_cast<int>(s->d);
  const int blk = s->block;
  const int nb = static_cast<int>(ceil_div(s->L, blk));
  dim3 grid(nb, static_cast<unsigned>(s->B * s->H));
  const size_t sm = sizeof(float) * (static_cast<size_t>(blk) * d * 2 + static_cast<size_t>(blk) * (d + 1));
  const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(d)));
#define ROPESLR_SIMT_CASE(DPL_)                                                                                     \
  case DPL_: {                                                                                                      \
    auto kfn = sparse_attn_simt_kernel<T, DPL_>;                                                                    \
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)) != cudaSuccess) \
      return ROPESLR_ERR_LAUNCH;                                                                                    \
    kfn<<<grid, 256, sm, st>>>(q, k, v, idx, kmax, cnt, s->L, blk, nb, perm, scale, o_sparse);                     \
    break;                                                                                                          \
  }
  switch (d / 32) {
    ROPESLR_SIMT_CASE(1)
    ROPESLR_SIMT_CASE(2)
    ROPESLR_SIMT_CASE(3)
    ROPESLR_SIMT_CASE(4)
    default:
      return ROPESLR_ERR_SHAPE;
  }
#undef ROPESLR_SIMT_CASE
  return launch_status();
}

int launch_sparse_attention_simt(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                                 const int32_t* idx, int kmax, const int32_t* cnt, const int32_t* perm,
                                 float* o_sparse, cudaStream_t st) {
  if (s->d % 32 || s->d < 32 || s->d > 128) return ROPESLR_ERR_SHAPE;
  if (s->block > 128) return ROPESLR_ERR_SHAPE;
  if (s->dtype == ROPESLR_BF16)
    return launch_simt_t(s, static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
                         static_cast<const __nv_bfloat16*>(v), idx, kmax, cnt, perm, o_sparse, st);
  return launch_simt_t(s, static_cast<const float*>(q), static_cast<const float*>(k), static_cast<const float*>(v),
                       idx, kmax, cnt, perm, o_sparse, st);
}

}  // namespace ropeslr
