// K3: the compensator branch, the token gate and the standalone fused
// epilogue (K4 for the CUDA-core attention path).
//
//   lowrank   x_hat_h = X_h + alpha_h * PE_h (mechanism.py:212-218, 429-432),
//             o_lr = sigmoid(sigmoid(x_hat_h W_A[h]) W_B[h]) (mechanism.py:225-235,
//             441-446), y_lr = RMSNorm(o_lr) * rms_lowrank (mechanism.py:238-246,
//             450); the gate logit x_hat . w_g (mechanism.py:434) is fused in
//             because the kernel already holds x_hat for every local column.
//   linear    phi = elu + 1; S = phi(k)^T v, z = sum phi(k) reduced over L in a
//             fixed chunk order; o = phi(q) S / max(phi(q).z, 1e-8)
//             (mechanism.py:33-36, 350-362).
//   fuse      out = RMS(o_sparse) * rms_sparse + sigmoid(g_logit + b_g) * y_lr
//             (mechanism.py:435-451).
#include <cuda_runtime.h>
#include <math.h>

#include <stdlib.h>

#include "common.cuh"

namespace ropeslr {

struct TokenCtx {
  int64_t L, x_row_stride, head_offset, d_model;
  int64_t tok0;  // grid index of local token 0 (the PE coordinates)
  int grid_h, grid_w, use_pe;
  const float *pe_t, *pe_x, *pe_y, *alpha, *w_g;
};

// x_hat for 4 consecutive local columns starting at global column gc.
template <typename T>
__device__ __forceinline__ void xhat4(const TokenCtx& c, const T* xrow, int64_t tok, int64_t gc, int lc, float* o) {
#pragma unroll
  for (int i = 0; i < 4; ++i) o[i] = to_f(xrow[lc + i]);
  if (c.use_pe) {
    const int64_t hw = static_cast<int64_t>(c.grid_h) * c.grid_w;
    const int64_t gt = tok + c.tok0;
    const int64_t tt = gt / hw, rem = gt % hw, xx = rem / c.grid_w, yy = rem % c.grid_w;
    const float* pt = c.pe_t + tt * c.d_model + gc;
    const float* px = c.pe_x + xx * c.d_model + gc;
    const float* py = c.pe_y + yy * c.d_model + gc;
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = fmaf(c.alpha[gc + i], (pt[i] + px[i]) + py[i], o[i]);
  }
}

constexpr int kTok = 32;  // tokens per CTA in the compensator kernels

// grid (ceil(L/32), B), block 256.
template <typename T>
__global__ void __launch_bounds__(256) lowrank_kernel(TokenCtx c, const T* __restrict__ x, int H, int d, int r,
                                                     const float* __restrict__ w_a, const float* __restrict__ w_b,
                                                     const float* __restrict__ rms_lr, float eps, T* __restrict__ y_lr,
                                                     float* __restrict__ o_lr, float* __restrict__ g_logit) {
  extern __shared__ float sm[];
  const int dp = d + 1, rp = r + 1;
  float* xs = sm;                 // [kTok][d+1]
  float* wa = xs + kTok * dp;     // [d][r]
  float* h1 = wa + d * r;         // [kTok][r+1]
  float* wb = h1 + kTok * rp;     // [r][d]
  float* gacc = wb + r * d;       // [kTok]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.y;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kTok;
  if (tid < kTok) gacc[tid] = 0.f;
  __syncthreads();

  for (int h = 0; h < H; ++h) {
    const float* wah = w_a + static_cast<int64_t>(h) * d * r;
    const float* wbh = w_b + static_cast<int64_t>(h) * r * d;
    for (int e = tid; e < d * r; e += 256) {
      wa[e] = wah[e];
      wb[e] = wbh[e];
    }
    // x_hat tile + gate partial; warp w owns tokens w, w+8, w+16, w+24
    for (int t = warp; t < kTok; t += 8) {
      const int64_t tok = t0 + t;
      float gp = 0.f;
      for (int j = lane * 4; j < d; j += 128) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (tok < c.L) {
          const int64_t gc = (c.head_offset + h) * d + j;
          const T* xrow = x + (b * c.L + tok) * c.x_row_stride + static_cast<int64_t>(h) * d;
          xhat4(c, xrow, tok, gc, j, v);
#pragma unroll
          for (int i = 0; i < 4; ++i) gp = fmaf(v[i], c.w_g[gc + i], gp);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) xs[t * dp + j + i] = v[i];
      }
      gp = warp_sum(gp);
      if (lane == 0) gacc[t] += gp;
    }
    __syncthreads();
    // layer 1: h1 = sigmoid(x_hat W_A)
    {
      const int t = tid >> 3, cg = tid & 7;
      for (int c0 = cg; c0 < r; c0 += 8) {
        float acc = 0.f;
        for (int j = 0; j < d; ++j) acc = fmaf(xs[t * dp + j], wa[j * r + c0], acc);
        h1[t * rp + c0] = sigmoidf_stable(acc);
      }
    }
    __syncthreads();
    // layer 2 + RMSNorm: each token is handled by 8 consecutive lanes
    {
      const int t = tid >> 3, jg = tid & 7;
      const int64_t tok = t0 + t;
      float o[16];
      float ss = 0.f;
      const int nj = d / 8;
      for (int m = 0; m < nj; ++m) {
        const int j = jg + 8 * m;
        float acc = 0.f;
        for (int cc = 0; cc < r; ++cc) acc = fmaf(h1[t * rp + cc], wb[cc * d + j], acc);
        float s = sigmoidf_stable(acc);
        o[m] = s;
        ss = fmaf(s, s, ss);
      }
      ss += __shfl_xor_sync(0xffffffffu, ss, 1);
      ss += __shfl_xor_sync(0xffffffffu, ss, 2);
      ss += __shfl_xor_sync(0xffffffffu, ss, 4);
      const float inv = 1.f / sqrtf(ss / static_cast<float>(d) + eps);
      if (tok < c.L) {
        T* yrow = y_lr + ((b * c.L + tok) * H + h) * d;
        float* orow = o_lr ? o_lr + ((b * H + h) * c.L + tok) * d : nullptr;
        for (int m = 0; m < nj; ++m) {
          const int j = jg + 8 * m;
          yrow[j] = from_f<T>(o[m] * inv * rms_lr[j]);
          if (orow) orow[j] = o[m];
        }
      }
    }
    __syncthreads();
  }
  if (g_logit != nullptr && tid < kTok && t0 + tid < c.L) g_logit[b * c.L + t0 + tid] = gacc[tid];
}

// One warp per token: g_logit = sum_c x_hat[c] * w_g[c] over the local columns.
template <typename T>
__global__ void __launch_bounds__(256) gate_kernel(TokenCtx c, const T* __restrict__ x, int H, int d,
                                                   float* __restrict__ g_logit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = blockIdx.y;
  const int64_t tok = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (tok >= c.L) return;
  const T* xrow = x + (b * c.L + tok) * c.x_row_stride;
  const int ncol = H * d;
  float gp = 0.f;
  for (int j = lane * 4; j < ncol; j += 128) {
    float v[4];
    xhat4(c, xrow, tok, c.head_offset * d + j, j, v);
#pragma unroll
    for (int i = 0; i < 4; ++i) gp = fmaf(v[i], c.w_g[c.head_offset * d + j + i], gp);
  }
  gp = warp_sum(gp);
  if (lane == 0) g_logit[b * c.L + tok] = gp;
}

__device__ __forceinline__ float elu1(float v) { return v > 0.f ? v + 1.f : __expf(fminf(v, 0.f)); }

constexpr int kLinChunk = 1024;  // tokens per partial state

// grid (nchunks, BH); partial[bh][chunk] = {S (d*d), z (d)}.
template <typename T>
__global__ void __launch_bounds__(256) linear_state_kernel(const T* __restrict__ k, const T* __restrict__ v, int64_t L,
                                                           int d, int nchunks, float* __restrict__ partial) {
  extern __shared__ float sm[];
  float* pk = sm;               // [32][d]
  float* vv = pk + 32 * d;      // [32][d]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t bh = blockIdx.y;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kLinChunk;
  const int64_t c1 = c0 + kLinChunk < L ? c0 + kLinChunk : L;
  const T* kb = k + bh * L * d;
  const T* vb = v + bh * L * d;
  const int na = d / 16;
  float acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int bb = 0; bb < 8; ++bb) acc[a][bb] = 0.f;
  float zacc = 0.f;
  for (int64_t l0 = c0; l0 < c1; l0 += 32) {
    for (int e = tid; e < 32 * d; e += 256) {
      const int64_t l = l0 + e / d;
      const int j = e % d;
      const bool ok = l < c1;
      pk[e] = ok ? elu1(to_f(kb[l * d + j])) : 0.f;
      vv[e] = ok ? to_f(vb[l * d + j]) : 0.f;
    }
    __syncthreads();
    for (int l = 0; l < 32; ++l) {
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        if (a >= na) break;
        const float p = pk[l * d + ty + 16 * a];
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) {
          if (bb >= na) break;
          acc[a][bb] = fmaf(p, vv[l * d + tx + 16 * bb], acc[a][bb]);
        }
      }
    }
    if (tid < d)
      for (int l = 0; l < 32; ++l) zacc += pk[l * d + tid];
    __syncthreads();
  }
  float* out = partial + (bh * nchunks + blockIdx.x) * static_cast<int64_t>(d * d + d);
  for (int a = 0; a < na; ++a)
    for (int bb = 0; bb < na; ++bb) out[(ty + 16 * a) * d + tx + 16 * bb] = acc[a][bb];
  if (tid < d) out[d * d + tid] = zacc;
}

// Fixed-order reduction over chunks: state[bh] = sum_chunk partial[bh][chunk].
__global__ void linear_reduce_kernel(const float* __restrict__ partial, int nchunks, int n, float* __restrict__ state) {
  const int64_t bh = blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  float s = 0.f;
  for (int c = 0; c < nchunks; ++c) s += partial[(bh * nchunks + c) * static_cast<int64_t>(n) + e];
  state[bh * n + e] = s;
}

// grid (ceil(L/32), B); per local head: o = phi(q) S / max(phi(q).z, 1e-8), RMSNorm.
template <typename T>
__global__ void __launch_bounds__(256) linear_apply_kernel(const T* __restrict__ q, const float* __restrict__ state,
                                                           int64_t L, int H, int d, const float* __restrict__ rms_lr,
                                                           float eps, T* __restrict__ y_lr, float* __restrict__ o_lr) {
  extern __shared__ float sm[];
  const int dp = d + 1;
  float* S = sm;              // [d][d]
  float* z = S + d * d;       // [d]
  float* pq = z + d;          // [kTok][d+1]
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.y;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kTok;
  for (int h = 0; h < H; ++h) {
    const int64_t bh = b * H + h;
    const float* st = state + bh * static_cast<int64_t>(d * d + d);
    for (int e = tid; e < d * d + d; e += 256) S[e] = st[e];
    for (int e = tid; e < kTok * d; e += 256) {
      const int t = e / d, j = e % d;
      const int64_t tok = t0 + t;
      pq[t * dp + j] = tok < L ? elu1(to_f(q[(bh * L + tok) * d + j])) : 0.f;
    }
    __syncthreads();
    const int t = tid >> 3, jg = tid & 7;
    const int64_t tok = t0 + t;
    float den = 0.f;
    for (int i = 0; i < d; ++i) den = fmaf(pq[t * dp + i], z[i], den);
    den = fmaxf(den, kLinearFloor);
    float o[16];
    float ss = 0.f;
    const int nj = d / 8;
    for (int m = 0; m < nj; ++m) {
      const int j = jg + 8 * m;
      float acc = 0.f;
      for (int i = 0; i < d; ++i) acc = fmaf(pq[t * dp + i], S[i * d + j], acc);
      o[m] = acc / den;
      ss = fmaf(o[m], o[m], ss);
    }
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    ss += __shfl_xor_sync(0xffffffffu, ss, 4);
    const float inv = 1.f / sqrtf(ss / static_cast<float>(d) + eps);
    if (tok < L) {
      T* yrow = y_lr + ((b * L + tok) * H + h) * d;
      float* orow = o_lr ? o_lr + (bh * L + tok) * d : nullptr;
      for (int m = 0; m < nj; ++m) {
        const int j = jg + 8 * m;
        yrow[j] = from_f<T>(o[m] * inv * rms_lr[j]);
        if (orow) orow[j] = o[m];
      }
    }
    __syncthreads();
  }
}

// One warp per (b, token, head) row.
template <typename T, typename TO = T>
__global__ void __launch_bounds__(256) fuse_output_kernel(const float* __restrict__ o_sparse, const T* __restrict__ y_lr,
                                                          const float* __restrict__ g_logit, float b_g,
                                                          const float* __restrict__ rms_sp, float eps, int64_t B,
                                                          int64_t L, int H, int d, TO* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);  // (b*L + tok)*H + h
  if (row >= B * L * H) return;
  const int h = static_cast<int>(row % H);
  const int64_t bt = row / H;  // b*L + tok
  const int64_t b = bt / L, tok = bt % L;
  const float* o = o_sparse + ((b * H + h) * L + tok) * d;
  float ov[8];
  float ss = 0.f;
  const int nm = d / 32;
  for (int m = 0; m < nm; ++m) {
    ov[m] = o[lane + 32 * m];
    ss = fmaf(ov[m], ov[m], ss);
  }
  ss = warp_sum(ss);
  const float inv = 1.f / sqrtf(ss / static_cast<float>(d) + eps);
  const float g = sigmoidf_stable(g_logit[bt] + b_g);
  const T* y = y_lr + row * d;
  TO* dst = out + row * d;
  for (int m = 0; m < nm; ++m) {
    const int j = lane + 32 * m;
    dst[j] = from_f<TO>(fmaf(g, to_f(y[j]), ov[m] * inv * rms_sp[j]));
  }
}

size_t lowrank_tc_workspace_bytes(int64_t B, int64_t H, int64_t L, int r, int T, int Hg, int Wg);
bool lowrank_tc_eligible(const ropeslr_shape* s, int r);
bool lowrank_umma_eligible(const ropeslr_shape* s, const ropeslr_token_args* t, int r);
size_t lowrank_umma_workspace_bytes(const ropeslr_shape* s, const ropeslr_token_args* t, int r);
size_t lowrank_umma_tables_bytes(const ropeslr_shape* s, const ropeslr_token_args* t, int r);
int lowrank_umma_fold(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b, int r,
                      void* tables, cudaStream_t st);
int lowrank_umma_folded(const ropeslr_shape* s, const ropeslr_token_args* t, int r, const void* tables,
                        const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* g_logit, float* g_part,
                        cudaStream_t st);
int launch_lowrank_umma(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b,
                        int r, const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* g_logit,
                        void* ws, cudaStream_t st);
int launch_lowrank_tc(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b,
                      int r, const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* g_logit, void* ws,
                      cudaStream_t st);

static TokenCtx make_ctx(const ropeslr_shape* s, const ropeslr_token_args* t) {
  TokenCtx c;
  c.L = s->L;
  c.tok0 = t->token_offset;
  c.x_row_stride = t->x_row_stride;
  c.head_offset = t->head_offset;
  c.d_model = t->d_model;
  c.grid_h = t->grid_h;
  c.grid_w = t->grid_w;
  c.use_pe = t->use_pe;
  c.pe_t = t->pe_t;
  c.pe_x = t->pe_x;
  c.pe_y = t->pe_y;
  c.alpha = t->alpha;
  c.w_g = t->w_g;
  return c;
}

// token_range: the call covers grid tokens [token_offset, token_offset + L)
// (the gate of a sequence shard); otherwise the whole grid, offset 0.
static int check_token_args(const ropeslr_shape* s, const ropeslr_token_args* t, bool token_range = false) {
  if (!t || !t->x || !t->w_g) return ROPESLR_ERR_NULL;
  if (t->use_pe && (!t->pe_t || !t->pe_x || !t->pe_y || !t->alpha)) return ROPESLR_ERR_NULL;
  const int64_t gsize = static_cast<int64_t>(t->grid_t) * t->grid_h * t->grid_w;
  if (token_range) {
    if (t->token_offset < 0 || t->token_offset + s->L > gsize) return ROPESLR_ERR_SHAPE;
  } else if (gsize != s->L || t->token_offset != 0) {
    return ROPESLR_ERR_SHAPE;
  }
  if (t->grid_t < 1 || t->grid_h < 1 || t->grid_w < 1) return ROPESLR_ERR_SHAPE;
  if (t->head_offset < 0 || (t->head_offset + s->H) * s->d > t->d_model) return ROPESLR_ERR_SHAPE;
  if (t->x_row_stride < s->H * s->d || t->x_row_stride % 4) return ROPESLR_ERR_SHAPE;
  return ROPESLR_OK;
}

static int check_shape(const ropeslr_shape* s) {
  if (!s) return ROPESLR_ERR_NULL;
  if (s->B < 1 || s->H < 1 || s->L < 1) return ROPESLR_ERR_SHAPE;
  if (s->dtype != ROPESLR_F32 && s->dtype != ROPESLR_BF16) return ROPESLR_ERR_DTYPE;
  return ROPESLR_OK;
}

}  // namespace ropeslr

using namespace ropeslr;

extern "C" size_t ropeslr_lowrank_workspace_bytes(const ropeslr_shape* s, const ropeslr_token_args* t,
                                                  int32_t rank) {
  if (!s || !t) return 0;
  if (lowrank_umma_eligible(s, t, rank)) return lowrank_umma_workspace_bytes(s, t, rank);
  if (!lowrank_tc_eligible(s, rank)) return 0;
  return lowrank_tc_workspace_bytes(s->B, s->H, s->L, rank, t->grid_t, t->grid_h, t->grid_w);
}

extern "C" int ropeslr_lowrank_branch(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a,
                                      const float* w_b, int32_t rank, const float* rms_lowrank, float eps, void* y_lr,
                                      float* o_lr, float* g_logit, void* ws, size_t ws_bytes, void* stream) {
  int st = check_shape(s);
  if (st) return st;
  if ((st = check_token_args(s, t))) return st;
  if (!w_a || !w_b || !rms_lowrank || !y_lr) return ROPESLR_ERR_NULL;
  if (s->d < 8 || s->d > 128 || s->d % 8) return ROPESLR_ERR_SHAPE;
  if (rank < 1 || rank > 256) return ROPESLR_ERR_SHAPE;
  if (!(eps > 0.f)) return ROPESLR_ERR_VALUE;
  if (lowrank_umma_eligible(s, t, rank)) {
    // tcgen05 / TMA path (bf16, d = 128, r in {16, 32, 48, 64}); y_lr rows leave by 256-bit stores
    if (t->x_row_stride % 8 || !aligned16(t->x) || !aligned32(y_lr)) return ROPESLR_ERR_ALIGN;
    if (o_lr && !aligned16(o_lr)) return ROPESLR_ERR_ALIGN;
    if (!ws || ws_bytes < ropeslr_lowrank_workspace_bytes(s, t, rank)) return ROPESLR_ERR_WORKSPACE;
    if (int e = launch_lowrank_umma(s, t, w_a, w_b, rank, rms_lowrank, eps, y_lr, o_lr, g_logit, ws,
                                    static_cast<cudaStream_t>(stream)))
      return e;
    return scan_nonfinite(g_logit, false, g_logit ? s->B * s->L : 0, t->nonfinite, ROPESLR_NONFINITE_X,
                          static_cast<cudaStream_t>(stream));
  }
  if (lowrank_tc_eligible(s, rank)) {
    if (t->x_row_stride % 8 || !aligned16(t->x) || !aligned16(y_lr)) return ROPESLR_ERR_ALIGN;
    if (!ws || ws_bytes < ropeslr_lowrank_workspace_bytes(s, t, rank)) return ROPESLR_ERR_WORKSPACE;
    if (int e = launch_lowrank_tc(s, t, w_a, w_b, rank, rms_lowrank, eps, y_lr, o_lr, g_logit, ws,
                                  static_cast<cudaStream_t>(stream)))
      return e;
    return scan_nonfinite(g_logit, false, g_logit ? s->B * s->L : 0, t->nonfinite, ROPESLR_NONFINITE_X,
                          static_cast<cudaStream_t>(stream));
  }
  const int d = static_cast<int>(s->d), r = rank;
  size_t sm = sizeof(float) * (static_cast<size_t>(kTok) * (d + 1) + d * r + kTok * (r + 1) + r * d + kTok);
  dim3 grid(static_cast<unsigned>(ceil_div(s->L, kTok)), static_cast<unsigned>(s->B));
  cudaStream_t stream_ = static_cast<cudaStream_t>(stream);
  TokenCtx c = make_ctx(s, t);
  if (s->dtype == ROPESLR_BF16) {
    auto kfn = lowrank_kernel<__nv_bfloat16>;
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    kfn<<<grid, 256, sm, stream_>>>(c, static_cast<const __nv_bfloat16*>(t->x), static_cast<int>(s->H), d, r, w_a,
                                    w_b, rms_lowrank, eps, static_cast<__nv_bfloat16*>(y_lr), o_lr, g_logit);
  } else {
    auto kfn = lowrank_kernel<float>;
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    kfn<<<grid, 256, sm, stream_>>>(c, static_cast<const float*>(t->x), static_cast<int>(s->H), d, r, w_a, w_b,
                                    rms_lowrank, eps, static_cast<float*>(y_lr), o_lr, g_logit);
  }
  if (int e = launch_status()) return e;
  return scan_nonfinite(g_logit, false, g_logit ? s->B * s->L : 0, t->nonfinite, ROPESLR_NONFINITE_X, stream_);
}

extern "C" size_t ropeslr_lowrank_tables_bytes(const ropeslr_shape* s, const ropeslr_token_args* t, int32_t rank) {
  if (!s || !t || !lowrank_umma_eligible(s, t, rank)) return 0;
  return lowrank_umma_tables_bytes(s, t, rank);
}

extern "C" int ropeslr_lowrank_tables(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a,
                                      const float* w_b, int32_t rank, void* tables, size_t tables_bytes,
                                      void* stream) {
  int st = check_shape(s);
  if (st) return st;
  if ((st = check_token_args(s, t))) return st;
  if (!w_a || !w_b || !tables) return ROPESLR_ERR_NULL;
  if (!lowrank_umma_eligible(s, t, rank)) return ROPESLR_ERR_SHAPE;
  if (!aligned16(tables)) return ROPESLR_ERR_ALIGN;
  if (tables_bytes < lowrank_umma_tables_bytes(s, t, rank)) return ROPESLR_ERR_WORKSPACE;
  return lowrank_umma_fold(s, t, w_a, w_b, rank, tables, static_cast<cudaStream_t>(stream));
}

extern "C" int ropeslr_lowrank_branch_folded(const ropeslr_shape* s, const ropeslr_token_args* t, int32_t rank,
                                             const void* tables, size_t tables_bytes, const float* rms_lowrank,
                                             float eps, void* y_lr, float* o_lr, float* g_logit, void* ws,
                                             size_t ws_bytes, void* stream) {
  int st = check_shape(s);
  if (st) return st;
  if ((st = check_token_args(s, t))) return st;
  if (!tables || !rms_lowrank || !y_lr) return ROPESLR_ERR_NULL;
  if (!(eps > 0.f)) return ROPESLR_ERR_VALUE;
  if (!lowrank_umma_eligible(s, t, rank)) return ROPESLR_ERR_SHAPE;
  if (t->x_row_stride % 8 || !aligned16(t->x) || !aligned32(y_lr) || !aligned16(tables)) return ROPESLR_ERR_ALIGN;
  if (o_lr && !aligned16(o_lr)) return ROPESLR_ERR_ALIGN;
  if (tables_bytes < lowrank_umma_tables_bytes(s, t, rank)) return ROPESLR_ERR_WORKSPACE;
  const size_t need = static_cast<size_t>(s->B * s->H * s->L) * sizeof(float);
  if (g_logit != nullptr && (!ws || ws_bytes < need)) return ROPESLR_ERR_WORKSPACE;
  cudaStream_t stream_ = static_cast<cudaStream_t>(stream);
  if (int e = lowrank_umma_folded(s, t, rank, tables, rms_lowrank, eps, y_lr, o_lr, g_logit,
                                  static_cast<float*>(ws), stream_))
    return e;
  return scan_nonfinite(g_logit, false, g_logit ? s->B * s->L : 0, t->nonfinite, ROPESLR_NONFINITE_X, stream_);
}

extern "C" int ropeslr_gate_logits(const ropeslr_shape* s, const ropeslr_token_args* t, float* g_logit,
                                   void* stream) {
  int st = check_shape(s);
  if (st) return st;
  if ((st = check_token_args(s, t, true))) return st;
  if (!g_logit) return ROPESLR_ERR_NULL;
  if (s->d % 4) return ROPESLR_ERR_SHAPE;
  dim3 grid(static_cast<unsigned>(ceil_div(s->L, 8)), static_cast<unsigned>(s->B));
  cudaStream_t stream_ = static_cast<cudaStream_t>(stream);
  TokenCtx c = make_ctx(s, t);
  if (s->dtype == ROPESLR_BF16)
    gate_kernel<__nv_bfloat16><<<grid, 256, 0, stream_>>>(c, static_cast<const __nv_bfloat16*>(t->x),
                                                          static_cast<int>(s->H), static_cast<int>(s->d), g_logit);
  else
    gate_kernel<float><<<grid, 256, 0, stream_>>>(c, static_cast<const float*>(t->x), static_cast<int>(s->H),
                                                  static_cast<int>(s->d), g_logit);
  if (int e = launch_status()) return e;
  return scan_nonfinite(g_logit, false, s->B * s->L, t->nonfinite, ROPESLR_NONFINITE_X, stream_);
}

static int64_t lin_nchunks(int64_t L) { return ceil_div(L, kLinChunk); }

extern "C" size_t ropeslr_linear_workspace_bytes(const ropeslr_shape* s) {
  if (!s) return 0;
  const int64_t n = s->d * s->d + s->d;
  const int64_t BH = s->B * s->H;
  return static_cast<size_t>(BH * (lin_nchunks(s->L) + 1) * n) * sizeof(float);
}

namespace ropeslr {
int linear_branch_tc(const ropeslr_shape* s, const void* q_lin, const void* k_lin, const void* v_lin,
                     const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* partial, float* state,
                     int nchunks, cudaStream_t st);
// Fixed-order chunk reduction of the linear state (also used by linear_tc.cu).
int linear_reduce(const float* partial, int nchunks, int n, float* state, int64_t BH, cudaStream_t st) {
  dim3 g2(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(BH));
  linear_reduce_kernel<<<g2, 256, 0, st>>>(partial, nchunks, n, state);
  return cudaGetLastError() == cudaSuccess ? ROPESLR_OK : ROPESLR_ERR_LAUNCH;
}
}  // namespace ropeslr

extern "C" int ropeslr_linear_branch(const ropeslr_shape* s, const void* q_lin, const void* k_lin, const void* v_lin,
                                     const float* rms_lowrank, float eps, void* y_lr, float* o_lr, void* ws,
                                     size_t ws_bytes, void* stream) {
  int st = check_shape(s);
  if (st) return st;
  if (!q_lin || !k_lin || !v_lin || !rms_lowrank || !y_lr) return ROPESLR_ERR_NULL;
  if (s->d < 16 || s->d > 128 || s->d % 16) return ROPESLR_ERR_SHAPE;
  if (!(eps > 0.f)) return ROPESLR_ERR_VALUE;
  if (!ws || ws_bytes < ropeslr_linear_workspace_bytes(s)) return ROPESLR_ERR_WORKSPACE;
  const int d = static_cast<int>(s->d);
  const int64_t BH = s->B * s->H;
  const int nch = static_cast<int>(lin_nchunks(s->L));
  const int n = d * d + d;
  float* partial = static_cast<float*>(ws);
  float* state = partial + BH * nch * static_cast<int64_t>(n);
  cudaStream_t stream_ = static_cast<cudaStream_t>(stream);
  // bf16, d = 128: the tensor-core passes (linear_tc.cu)
  if (s->dtype == ROPESLR_BF16 && d == 128 && !tuning().linear_simt && aligned16(q_lin) &&
      aligned16(k_lin) && aligned16(v_lin) && aligned16(y_lr))
    return linear_branch_tc(s, q_lin, k_lin, v_lin, rms_lowrank, eps, y_lr, o_lr, partial, state, nch, stream_);
  size_t sm1 = sizeof(float) * 2 * 32 * d;
  size_t sm3 = sizeof(float) * (static_cast<size_t>(n) + kTok * (d + 1));
  dim3 g1(nch, static_cast<unsigned>(BH));
  dim3 g2(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(BH));
  dim3 g3(static_cast<unsigned>(ceil_div(s->L, kTok)), static_cast<unsigned>(s->B));
  if (s->dtype == ROPESLR_BF16) {
    using T = __nv_bfloat16;
    linear_state_kernel<T><<<g1, 256, sm1, stream_>>>(static_cast<const T*>(k_lin), static_cast<const T*>(v_lin), s->L,
                                                      d, nch, partial);
    linear_reduce_kernel<<<g2, 256, 0, stream_>>>(partial, nch, n, state);
    if (cudaFuncSetAttribute(linear_apply_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm3)) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    linear_apply_kernel<T><<<g3, 256, sm3, stream_>>>(static_cast<const T*>(q_lin), state, s->L,
                                                      static_cast<int>(s->H), d, rms_lowrank, eps,
                                                      static_cast<T*>(y_lr), o_lr);
  } else {
    using T = float;
    linear_state_kernel<T><<<g1, 256, sm1, stream_>>>(static_cast<const T*>(k_lin), static_cast<const T*>(v_lin), s->L,
                                                      d, nch, partial);
    linear_reduce_kernel<<<g2, 256, 0, stream_>>>(partial, nch, n, state);
    if (cudaFuncSetAttribute(linear_apply_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm3)) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    linear_apply_kernel<T><<<g3, 256, sm3, stream_>>>(static_cast<const T*>(q_lin), state, s->L,
                                                      static_cast<int>(s->H), d, rms_lowrank, eps,
                                                      static_cast<T*>(y_lr), o_lr);
  }
  return launch_status();
}

namespace ropeslr {
// K4 with the output in `out_dtype` (the shape's dtype, or float32).
int fuse_output(const ropeslr_shape* s, const float* o_sparse, const void* y_lr, const float* g_logit, float b_g,
                const float* rms_sparse, float eps, void* out, int out_dtype, cudaStream_t stream_) {
  int st = check_shape(s);
  if (st) return st;
  if (!o_sparse || !y_lr || !g_logit || !rms_sparse || !out) return ROPESLR_ERR_NULL;
  if (s->d < 32 || s->d > 256 || s->d % 32) return ROPESLR_ERR_SHAPE;
  if (!(eps > 0.f)) return ROPESLR_ERR_VALUE;
  if (out_dtype != s->dtype && out_dtype != ROPESLR_F32) return ROPESLR_ERR_DTYPE;
  const int64_t rows = s->B * s->L * s->H;
  dim3 grid(static_cast<unsigned>(ceil_div(rows, 8)));
  const int H = static_cast<int>(s->H), d = static_cast<int>(s->d);
  if (s->dtype == ROPESLR_BF16 && out_dtype == ROPESLR_BF16)
    fuse_output_kernel<__nv_bfloat16><<<grid, 256, 0, stream_>>>(
        o_sparse, static_cast<const __nv_bfloat16*>(y_lr), g_logit, b_g, rms_sparse, eps, s->B, s->L, H, d,
        static_cast<__nv_bfloat16*>(out));
  else if (s->dtype == ROPESLR_BF16)
    fuse_output_kernel<__nv_bfloat16, float><<<grid, 256, 0, stream_>>>(
        o_sparse, static_cast<const __nv_bfloat16*>(y_lr), g_logit, b_g, rms_sparse, eps, s->B, s->L, H, d,
        static_cast<float*>(out));
  else
    fuse_output_kernel<float><<<grid, 256, 0, stream_>>>(o_sparse, static_cast<const float*>(y_lr), g_logit, b_g,
                                                         rms_sparse, eps, s->B, s->L, H, d, static_cast<float*>(out));
  return launch_status();
}
}  // namespace ropeslr

extern "C" int ropeslr_fuse_output(const ropeslr_shape* s, const float* o_sparse, const void* y_lr,
                                   const float* g_logit, float b_g, const float* rms_sparse, float eps, void* out,
                                   void* stream) {
  if (!s) return ROPESLR_ERR_NULL;
  return ropeslr::fuse_output(s, o_sparse, y_lr, g_logit, b_g, rms_sparse, eps, out, s->dtype,
                              static_cast<cudaStream_t>(stream));
}
