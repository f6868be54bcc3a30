// K3 `linear` mode on the tensor cores (bf16, d = 128): the linear
// compensator of mechanism.py:33-36, 347-362,
//
//   S_h = phi(K_h)^T V_h,  z_h = sum_tokens phi(K_h),
//   o   = phi(Q_h) S_h / max(phi(Q_h) . z_h, 1e-8),  y = RMSNorm(o) * rms_lowrank,
//
// phi = elu + 1, as two GEMM-shaped passes with mma.sync (m16n8k16, bf16 in,
// fp32 accumulate) instead of the CUDA-core loops of compensator.cu:
//
//   linear_state_mma_kernel  one CTA per (1024-token chunk, head): the chunk's
//                            partial S (128 x 128) and z into the workspace,
//                            reduced over chunks in fixed order afterwards
//                            (linear_reduce_kernel, deterministic);
//   linear_apply_mma_kernel  one CTA per (128-token tile, head): phi(Q) S with
//                            S split into bf16 hi + lo parts (~16 mantissa
//                            bits), the denominator, RMSNorm, bf16 store.
//
// Operands are staged token-major in padded shared memory and read with
// ldmatrix (.trans where the reduction runs over tokens).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace ropeslr {
namespace lin {

constexpr int D = 128;
constexpr int STR = D + 8;       // padded row (bf16 elements): conflict-free ldmatrix
constexpr int kChunk = 1024;     // tokens per partial state (matches compensator.cu)
constexpr int kTT = 64;          // tokens per staged tile of the state kernel
constexpr int kAT = 128;         // tokens per CTA of the apply kernel
constexpr float kFloor = 1e-8f;  // mechanism.py:36

__device__ __forceinline__ float elu1(float v) { return v > 0.f ? v + 1.f : __expf(v); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// The warp's 32 x 64 block of a 128 x 128 product over one k16 step.
// A(m, k) from `a_base` (element (m, k) at a_base[m*STR + k] when !A_T, at
// a_base[k*STR + m] when A_T), B(k, n) = b_base[k*STR + n].
template <bool A_T>
__device__ __forceinline__ void warp_k16(float (&acc)[2][8][4], const __nv_bfloat16* a_base,
                                         const __nv_bfloat16* b_base, int m0, int n0, int k0, int lane) {
  const int j = lane >> 3, r = lane & 7;
  uint32_t a[2][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const int m = m0 + 16 * mi;
    if (A_T) {
      // matrices (m 0-7 | 8-15) x (k 0-7 | 8-15) in a0..a3 order, stored k-major
      ldsm_x4_t(a[mi], a_base + (k0 + (j >> 1) * 8 + r) * STR + m + (j & 1) * 8);
    } else {
      ldsm_x4(a[mi], a_base + (m + (j & 1) * 8 + r) * STR + k0 + (j >> 1) * 8);
    }
  }
#pragma unroll
  for (int np = 0; np < 4; ++np) {
    uint32_t b[4];  // n8 tiles 2np, 2np+1: (k 0-7, k 8-15) each
    ldsm_x4_t(b, b_base + (k0 + (j & 1) * 8 + r) * STR + n0 + 16 * np + (j >> 1) * 8);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      mma16816(acc[mi][2 * np], a[mi], b[0], b[1]);
      mma16816(acc[mi][2 * np + 1], a[mi], b[2], b[3]);
    }
  }
}

// grid (nchunks, B*H), 256 threads; partial[bh][chunk] = {S (128*128), z (128)}.
__global__ void __launch_bounds__(256) linear_state_mma_kernel(const __nv_bfloat16* __restrict__ k,
                                                               const __nv_bfloat16* __restrict__ v, int64_t L,
                                                               int nchunks, float* __restrict__ partial) {
  __shared__ __align__(16) __nv_bfloat16 sK[kTT * STR];
  __shared__ __align__(16) __nv_bfloat16 sV[kTT * STR];
  __shared__ float zred[16][D + 4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bh = blockIdx.y;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kChunk;
  const int64_t c1 = c0 + kChunk < L ? c0 + kChunk : L;
  const __nv_bfloat16* kb = k + bh * L * D;
  const __nv_bfloat16* vb = v + bh * L * D;
  const int m0 = 32 * (warp >> 1), n0 = 64 * (warp & 1);
  float acc[2][8][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.f;
  const int ch = tid & 15, rr = tid >> 4;  // staging: 8 columns, rows rr + 16 i
  float zacc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int64_t l0 = c0; l0 < c1; l0 += kTT) {
#pragma unroll
    for (int i = 0; i < kTT / 16; ++i) {
      const int row = rr + 16 * i;
      const int64_t l = l0 + row;
      uint4 ku = make_uint4(0, 0, 0, 0), vu = make_uint4(0, 0, 0, 0);
      if (l < c1) {
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(kb + l * D + ch * 8));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          const float p0 = elu1(f.x), p1 = elu1(f.y);
          pk[e] = pack_bf16(p0, p1);
          const float2 r2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[e]));
          zacc[2 * e] += r2.x;  // z sums the phi values the MMA sees
          zacc[2 * e + 1] += r2.y;
        }
        ku = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        vu = __ldg(reinterpret_cast<const uint4*>(vb + l * D + ch * 8));
      }
      *reinterpret_cast<uint4*>(sK + row * STR + ch * 8) = ku;
      *reinterpret_cast<uint4*>(sV + row * STR + ch * 8) = vu;
    }
    __syncthreads();
#pragma unroll
    for (int k0 = 0; k0 < kTT; k0 += 16) warp_k16<true>(acc, sK, sV, m0, n0, k0, lane);
    __syncthreads();
  }
  float* out = partial + (bh * nchunks + blockIdx.x) * static_cast<int64_t>(D * D + D);
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int m = m0 + 16 * mi + g, n = n0 + 8 * nt + 2 * t;
      *reinterpret_cast<float2*>(out + m * D + n) = make_float2(acc[mi][nt][0], acc[mi][nt][1]);
      *reinterpret_cast<float2*>(out + (m + 8) * D + n) = make_float2(acc[mi][nt][2], acc[mi][nt][3]);
    }
#pragma unroll
  for (int e = 0; e < 8; ++e) zred[rr][ch * 8 + e] = zacc[e];
  __syncthreads();
  if (tid < D) {
    float z = 0.f;
    for (int i = 0; i < 16; ++i) z += zred[i][tid];
    out[D * D + tid] = z;
  }
}

// grid (ceil(L / 128), B*H), 256 threads.
__global__ void __launch_bounds__(256) linear_apply_mma_kernel(const __nv_bfloat16* __restrict__ q,
                                                               const float* __restrict__ state, int64_t L, int H,
                                                               const float* __restrict__ rms_lr, float eps,
                                                               __nv_bfloat16* __restrict__ y_lr,
                                                               float* __restrict__ o_lr) {
  extern __shared__ __align__(16) uint8_t smem[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem);  // [kAT][STR]; later the bf16 output tile
  __nv_bfloat16* sHi = sQ + kAT * STR;                          // [D][STR] S hi
  __nv_bfloat16* sLo = sHi + D * STR;                           // [D][STR] S lo
  float* sz = reinterpret_cast<float*>(sLo + D * STR);          // [D]
  float* sden = sz + D;                                         // [kAT]
  float* sss = sden + kAT;                                      // [kAT][2] partial sums of squares
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / H, h = bh % H;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kAT;
  const float* st = state + bh * static_cast<int64_t>(D * D + D);
  // S -> bf16 hi + lo (row m, col n), z
  for (int e = tid; e < D * D / 2; e += 256) {
    const int m = (2 * e) / D, n = (2 * e) % D;
    const float2 sv = *reinterpret_cast<const float2*>(st + m * D + n);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(sv.x, sv.y);
    const float2 hf = __bfloat1622float2(hi);
    *reinterpret_cast<__nv_bfloat162*>(sHi + m * STR + n) = hi;
    *reinterpret_cast<__nv_bfloat162*>(sLo + m * STR + n) = __floats2bfloat162_rn(sv.x - hf.x, sv.y - hf.y);
  }
  if (tid < D) sz[tid] = st[D * D + tid];
  __syncthreads();
  // phi(Q) tile and the denominators (16 threads per token)
  const int ch = tid & 15, rr = tid >> 4;
#pragma unroll
  for (int i = 0; i < kAT / 16; ++i) {
    const int row = rr + 16 * i;
    const int64_t tok = t0 + row;
    uint4 qu = make_uint4(0, 0, 0, 0);
    float dp = 0.f;
    if (tok < L) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(q + (bh * L + tok) * D + ch * 8));
      const __nv_bfloat162* hq = reinterpret_cast<const __nv_bfloat162*>(&raw);
      uint32_t pk[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(hq[e]);
        pk[e] = pack_bf16(elu1(f.x), elu1(f.y));
        const float2 r2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[e]));
        dp = fmaf(r2.x, sz[ch * 8 + 2 * e], fmaf(r2.y, sz[ch * 8 + 2 * e + 1], dp));
      }
      qu = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) dp += __shfl_xor_sync(0xffffffffu, dp, o);
    if (ch == 0) sden[row] = fmaxf(dp, kFloor);
    *reinterpret_cast<uint4*>(sQ + row * STR + ch * 8) = qu;
  }
  __syncthreads();
  const int m0 = 32 * (warp >> 1), n0 = 64 * (warp & 1);  // token rows, output columns
  float acc[2][8][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][c][e] = 0.f;
#pragma unroll
  for (int k0 = 0; k0 < D; k0 += 16) {
    warp_k16<false>(acc, sQ, sHi, m0, n0, k0, lane);
    warp_k16<false>(acc, sQ, sLo, m0, n0, k0, lane);
  }
  // o = acc / den; RMSNorm over the 128 columns of each token row (this
  // warp holds 64 of them, its partner warp the other 64)
  const int g = lane >> 2, t = lane & 3;
  float ss[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const float i0 = 1.f / sden[m0 + 16 * mi + g], i1 = 1.f / sden[m0 + 16 * mi + g + 8];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      acc[mi][nt][0] *= i0;
      acc[mi][nt][1] *= i0;
      acc[mi][nt][2] *= i1;
      acc[mi][nt][3] *= i1;
      ss[mi][0] = fmaf(acc[mi][nt][0], acc[mi][nt][0], fmaf(acc[mi][nt][1], acc[mi][nt][1], ss[mi][0]));
      ss[mi][1] = fmaf(acc[mi][nt][2], acc[mi][nt][2], fmaf(acc[mi][nt][3], acc[mi][nt][3], ss[mi][1]));
    }
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float x = ss[mi][hh];
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      x += __shfl_xor_sync(0xffffffffu, x, 2);
      if (t == 0) sss[(m0 + 16 * mi + g + 8 * hh) * 2 + (warp & 1)] = x;
    }
  __syncthreads();  // sums of squares posted; every warp is past its MMAs (sQ is free)
  __nv_bfloat16* sOut = sQ;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int row = m0 + 16 * mi + g + 8 * hh;
      const float inv = rsqrtf((sss[row * 2] + sss[row * 2 + 1]) * (1.f / D) + eps);
      const int64_t tok = t0 + row;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int n = n0 + 8 * nt + 2 * t;
        const float o0 = acc[mi][nt][2 * hh], o1 = acc[mi][nt][2 * hh + 1];
        *reinterpret_cast<__nv_bfloat162*>(sOut + row * STR + n) =
            __floats2bfloat162_rn(o0 * inv * rms_lr[n], o1 * inv * rms_lr[n + 1]);
        if (o_lr != nullptr && tok < L) *reinterpret_cast<float2*>(o_lr + (bh * L + tok) * D + n) = make_float2(o0, o1);
      }
    }
  __syncthreads();
  // coalesced row stores of y_lr [B, L, H, d]
#pragma unroll
  for (int i = 0; i < kAT / 16; ++i) {
    const int row = rr + 16 * i;
    const int64_t tok = t0 + row;
    if (tok < L)
      *reinterpret_cast<uint4*>(y_lr + ((b * L + tok) * H + h) * D + ch * 8) =
          *reinterpret_cast<const uint4*>(sOut + row * STR + ch * 8);
  }
}

}  // namespace lin

// Entry from ropeslr_linear_branch (compensator.cu) for bf16, d = 128.
int linear_branch_tc(const ropeslr_shape* s, const void* q_lin, const void* k_lin, const void* v_lin,
                     const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* partial, float* state,
                     int nchunks, cudaStream_t st) {
  using namespace lin;
  const int64_t BH = s->B * s->H;
  const int n = D * D + D;
  lin::linear_state_mma_kernel<<<dim3(nchunks, static_cast<unsigned>(BH)), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(k_lin), static_cast<const __nv_bfloat16*>(v_lin), s->L, nchunks, partial);
  if (cudaGetLastError() != cudaSuccess) return ROPESLR_ERR_LAUNCH;
  int linear_reduce(const float* partial, int nchunks, int n, float* state, int64_t BH, cudaStream_t st);
  if (int e = linear_reduce(partial, nchunks, n, state, BH, st)) return e;
  const size_t smem = (static_cast<size_t>(kAT) * STR + 2 * static_cast<size_t>(D) * STR) * sizeof(__nv_bfloat16) +
                      (D + kAT + 2 * kAT) * sizeof(float);
  if (cudaFuncSetAttribute(lin::linear_apply_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  lin::linear_apply_mma_kernel<<<dim3(static_cast<unsigned>(ceil_div(s->L, kAT)), static_cast<unsigned>(BH)), 256,
                                 smem, st>>>(static_cast<const __nv_bfloat16*>(q_lin), state, s->L,
                                             static_cast<int>(s->H), rms_lowrank, eps,
                                             static_cast<__nv_bfloat16*>(y_lr), o_lr);
  return launch_status();
}

}  // namespace ropeslr
