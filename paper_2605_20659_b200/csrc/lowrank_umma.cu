// K3 on the 5th-generation tensor cores: the low-rank compensator, its
// RMSNorm and the partial gate logits (mechanism.py:225-235, 238-255,
// 429-447) for bf16 X with d = 128 and rank r <= 112 (r % 16 == 0).
//
// Algebra (exact in real arithmetic): x_hat_h W_A = X_h W_A + sum_axis
// Z_axis[coord] with Z_axis = (alpha * P_axis)_h W_A (lowrank_fold_kernel),
// and x_hat . w_g = X . w_g + sum_axis G_axis[coord].  X is read once by TMA
// and x_hat is never materialised.  The gate dot rides GEMM1 as two extra
// columns (w_g split into bf16 hi + lo, ~16 mantissa bits).
//
// One CTA per SM-slot works on a single (batch, head): its W_A / W_B images
// and Z / G tables are staged in shared memory once, then it walks 128-token
// tiles t = blockIdx.x, + gridDim.x, ...  Warp roles:
//
//   warp 0        TMA producer: X tile [128 tokens x 128 cols] (two 64-col
//                 boxes, 128-byte swizzle) into a 3-stage ring
//   warp 1        MMA issuer:  D1_w = X W_A^T   (M 128, N r+16, K 128)
//                              D2_w = H1_w W_B^T (M 128, N 128, K 64)
//                 in the order MMA1(i), MMA2(i-1), ...
//   warp 2        TMEM allocation (512 columns)
//   warps 4-11    two epilogue warpgroups, WG w owns tiles i = w (mod 2) and
//                 the TMEM buffers D1_w, D2_w and the smem operand H1_w.
//                 Thread = token row: D1 row + Z gathers -> sigmoid -> bf16
//                 into the swizzled H1 tile (GEMM2's A operand); gate partial;
//                 D2 row -> sigmoid (written back to TMEM) -> RMSNorm *
//                 rms_lowrank -> bf16 y_lr row.
//
// TMEM columns: D1_0 [0, 128), D1_1 [128, 256), D2_0 [256, 384), D2_1 [384, 512).
// HBM traffic per (token, head): 256 B of X in, 256 B of y_lr out.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace ropeslr {
namespace lu {

using namespace sm100;

constexpr int D = 128;        // head dim
constexpr int M = 128;        // tokens per tile (MMA rows)
constexpr int KR = 64;        // GEMM2 K: rank padded to one 128-byte swizzle atom
constexpr int XSTAGES = 3;
constexpr int kThreads = 384;

template <int R>
struct Lay {
  static constexpr int N1 = R + 16;              // GEMM1 N: rank + gate hi / lo (+ zero pad)
  static constexpr int X_BYTES = M * D * 2;      // 32 KiB
  static constexpr int WA_BYTES = N1 * D * 2;    // two 64-col atoms of N1 rows
  static constexpr int WB_BYTES = D * KR * 2;    // 16 KiB
  static constexpr int H1_BYTES = M * KR * 2;    // 16 KiB
  static constexpr int OFF_X = 0;
  static constexpr int OFF_WA = OFF_X + XSTAGES * X_BYTES;
  static constexpr int OFF_WB = OFF_WA + (WA_BYTES + 1023) / 1024 * 1024;
  static constexpr int OFF_H1 = OFF_WB + WB_BYTES;
  static constexpr int OFF_BAR = OFF_H1 + 2 * H1_BYTES;
  static constexpr int NBAR = 2 * XSTAGES + 12;   // X ring full/empty + 6 per-warpgroup pairs
  static constexpr int OFF_TAB = OFF_BAR + 256;  // Z [nrows][R + 4] f32, then G [nrows] f32
  static_assert(NBAR * 8 + 4 <= 256, "barrier block overflows");
  static constexpr int ZP = R + 4;               // Z row pitch (floats): float4 rows spread over the banks
  static int bytes(int nrows) { return OFF_TAB + nrows * (ZP + 1) * 4; }
};

enum Bar { XF = 0, XE = XSTAGES, D1F = 2 * XSTAGES, D1E = D1F + 2, H1F = D1E + 2, H1E = H1F + 2, D2F = H1E + 2,
           D2E = D2F + 2, BAR_END = D2E + 2 };
static_assert(BAR_END == 2 * XSTAGES + 12, "barrier enum and Lay::NBAR disagree");

struct FoldArgs {
  const float* w_a;   // [H, d, r]
  const float* w_b;   // [H, r, d]
  const float* alpha; // [D_total]
  const float* w_g;   // [D_total]
  const float *pe_t, *pe_x, *pe_y;  // [n, D_total]
  int64_t d_model, head_offset;
  int H, r, T, Hg, Wg, use_pe;
  uint8_t* wa_img;    // [H][Lay::WA_BYTES] swizzled smem images
  uint8_t* wb_img;    // [H][Lay::WB_BYTES]
  float* Z;           // [H][nrows][r]
  float* G;           // [H][nrows]
};

__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
  return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

// grid (nrows + 2, H), 128 threads.  Blocks [0, nrows): Z / G rows of the
// per-axis PE tables; block nrows: W_A^T image (+ w_g hi/lo rows); block
// nrows + 1: W_B^T image (rank zero-padded to 64).
template <int R>
__global__ void __launch_bounds__(128) lowrank_fold_umma_kernel(FoldArgs a) {
  const int h = blockIdx.y;
  const int nrows = a.T + a.Hg + a.Wg;
  const int64_t gc0 = (a.head_offset + h) * D;
  const int tid = threadIdx.x;
  if (blockIdx.x == nrows) {
    constexpr int N1 = Lay<R>::N1;
    const float* wa = a.w_a + static_cast<int64_t>(h) * D * R;
    uint8_t* img = a.wa_img + static_cast<int64_t>(h) * Lay<R>::WA_BYTES;
    for (int e = tid; e < N1 * (D / 8); e += blockDim.x) {
      const int n = e / (D / 8), c16 = e % (D / 8);  // 16-byte chunk of 8 k-values
      uint32_t pk[4];
      for (int q = 0; q < 4; ++q) {
        float v2[2];
        for (int u = 0; u < 2; ++u) {
          const int k = c16 * 8 + q * 2 + u;
          float v = 0.f;
          if (n < R) {
            v = wa[k * R + n];
          } else if (n == R || n == R + 1) {
            const float wg = a.w_g[gc0 + k];
            const float hi = __bfloat162float(__float2bfloat16_rn(wg));
            v = n == R ? hi : wg - hi;
          }
          v2[u] = v;
        }
        __nv_bfloat162 hb = __floats2bfloat162_rn(v2[0], v2[1]);
        pk[q] = *reinterpret_cast<uint32_t*>(&hb);
      }
      const int atom = c16 >> 3, chunk = c16 & 7;
      *reinterpret_cast<uint4*>(img + atom * N1 * 128 + sw128(n, chunk)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    return;
  }
  if (blockIdx.x == nrows + 1) {
    const float* wb = a.w_b + static_cast<int64_t>(h) * R * D;
    uint8_t* img = a.wb_img + static_cast<int64_t>(h) * Lay<R>::WB_BYTES;
    for (int e = tid; e < D * (KR / 8); e += blockDim.x) {
      const int n = e / (KR / 8), chunk = e % (KR / 8);
      uint32_t pk[4];
      for (int q = 0; q < 4; ++q) {
        const int k0 = chunk * 8 + q * 2;
        const float v0 = k0 < R ? wb[k0 * D + n] : 0.f;
        const float v1 = k0 + 1 < R ? wb[(k0 + 1) * D + n] : 0.f;
        __nv_bfloat162 hb = __floats2bfloat162_rn(v0, v1);
        pk[q] = *reinterpret_cast<uint32_t*>(&hb);
      }
      *reinterpret_cast<uint4*>(img + sw128(n, chunk)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    return;
  }
  const int i = blockIdx.x;
  float* zrow = a.Z + (static_cast<int64_t>(h) * nrows + i) * R;
  if (!a.use_pe) {
    for (int j = tid; j < R; j += blockDim.x) zrow[j] = 0.f;
    if (tid == 0) a.G[static_cast<int64_t>(h) * nrows + i] = 0.f;
    return;
  }
  __shared__ float v[D];
  __shared__ float red[4];
  const float* tab = i < a.T ? a.pe_t + static_cast<int64_t>(i) * a.d_model
                             : (i < a.T + a.Hg ? a.pe_x + static_cast<int64_t>(i - a.T) * a.d_model
                                               : a.pe_y + static_cast<int64_t>(i - a.T - a.Hg) * a.d_model);
  const float pv = a.alpha[gc0 + tid] * tab[gc0 + tid];  // blockDim == D
  v[tid] = pv;
  float gp = warp_sum(pv * a.w_g[gc0 + tid]);
  if ((tid & 31) == 0) red[tid >> 5] = gp;
  __syncthreads();
  if (tid < R) {
    const float* wa = a.w_a + static_cast<int64_t>(h) * D * R;
    float z = 0.f;
    for (int k = 0; k < D; ++k) z = fmaf(v[k], wa[k * R + tid], z);
    zrow[tid] = z;
  }
  if (tid == 0) a.G[static_cast<int64_t>(h) * nrows + i] = (red[0] + red[1]) + (red[2] + red[3]);
}

struct MainArgs {
  const uint8_t* wa_img;
  const uint8_t* wb_img;
  const float* Z;
  const float* G;
  const float* rms_lr;
  float eps;
  int64_t L;
  int H, T, Hg, Wg, use_pe, ntiles;
  __nv_bfloat16* y_lr;  // [B, L, H, d]
  float* o_lr;          // [B, H, L, d] or null
  float* g_part;        // [B, H, L]
};

template <int R>
__global__ void __launch_bounds__(kThreads, 1) lowrank_umma_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                   const MainArgs a) {
  using Lay_ = Lay<R>;
  constexpr int N1 = Lay_::N1;
  constexpr int ZP = Lay_::ZP;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  uint8_t* sX = smem + Lay_::OFF_X;
  uint8_t* sWA = smem + Lay_::OFF_WA;
  uint8_t* sWB = smem + Lay_::OFF_WB;
  uint8_t* sH1 = smem + Lay_::OFF_H1;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay_::OFF_BAR);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Lay_::OFF_BAR + Lay_::NBAR * 8);
  const int nrows = a.T + a.Hg + a.Wg;
  float* sZ = reinterpret_cast<float*>(smem + Lay_::OFF_TAB);
  float* sG = sZ + nrows * ZP;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y;
  const int b = bh / a.H, h = bh % a.H;

  // ---- stage the per-head operands (generic proxy), then publish to the async proxy
  {
    const uint4* wa = reinterpret_cast<const uint4*>(a.wa_img + static_cast<int64_t>(h) * Lay_::WA_BYTES);
    for (int e = threadIdx.x; e < Lay_::WA_BYTES / 16; e += kThreads) reinterpret_cast<uint4*>(sWA)[e] = wa[e];
    const uint4* wb = reinterpret_cast<const uint4*>(a.wb_img + static_cast<int64_t>(h) * Lay_::WB_BYTES);
    for (int e = threadIdx.x; e < Lay_::WB_BYTES / 16; e += kThreads) reinterpret_cast<uint4*>(sWB)[e] = wb[e];
    const float* z = a.Z + static_cast<int64_t>(h) * nrows * R;
    for (int e = threadIdx.x; e < nrows * R / 4; e += kThreads) {
      const int row = e / (R / 4), c4 = e % (R / 4);
      *reinterpret_cast<float4*>(sZ + row * ZP + c4 * 4) = reinterpret_cast<const float4*>(z)[e];
    }
    for (int e = threadIdx.x; e < nrows; e += kThreads) sG[e] = a.G[static_cast<int64_t>(h) * nrows + e];
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < Lay_::NBAR; ++i) {
      const bool per_thread = (i >= D1E && i < D1E + 2) || (i >= H1F && i < H1F + 2) || (i >= D2E && i < D2E + 2);
      mbar_init(&bars[i], per_thread ? 128 : 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int first = blockIdx.x, stride = gridDim.x;
  const int n_my = first < a.ntiles ? (a.ntiles - first + stride - 1) / stride : 0;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < n_my; ++i) {
        const int t = first + i * stride;
        const int s = i % XSTAGES;
        mbar_wait(&bars[XE + s], ((i / XSTAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars[XF + s], Lay_::X_BYTES);
        const int row = static_cast<int>(static_cast<int64_t>(b) * a.L + static_cast<int64_t>(t) * M);
        uint8_t* dst = sX + s * Lay_::X_BYTES;
        tma_load_2d_hint(dst, &tmX, &bars[XF + s], h * D, row, pol);
        tma_load_2d_hint(dst + M * 128, &tmX, &bars[XF + s], h * D + 64, row, pol);
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc1 = idesc_bf16_f32(M, N1, false, false);
    constexpr uint32_t idesc2 = idesc_bf16_f32(M, D, false, false);
    const uint64_t dX0 = desc_sw128(smem_u32(sX), 16, 1024);
    const uint64_t dWA = desc_sw128(smem_u32(sWA), 16, 1024);
    const uint64_t dH10 = desc_sw128(smem_u32(sH1), 16, 1024);
    const uint64_t dWB = desc_sw128(smem_u32(sWB), 16, 1024);
    const bool leader = elect_one();
    for (int i = 0; i <= n_my; ++i) {
      if (i < n_my) {
        const int s = i % XSTAGES, w = i & 1;
        mbar_wait(&bars[XF + s], (i / XSTAGES) & 1);
        mbar_wait(&bars[D1E + w], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        if (leader) {
          const uint64_t dX = dX0 + static_cast<uint64_t>((s * Lay_::X_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t da = dX + static_cast<uint64_t>(((kk >> 2) * (M * 128) + (kk & 3) * 32) >> 4);
            const uint64_t db = dWA + static_cast<uint64_t>(((kk >> 2) * (N1 * 128) + (kk & 3) * 32) >> 4);
            mma_bf16_ss(tmem + w * 128, da, db, idesc1, kk > 0 ? 1u : 0u);
          }
          mma_commit(&bars[XE + s]);
          mma_commit(&bars[D1F + w]);
        }
        __syncwarp();
      }
      if (i >= 1) {
        const int j = i - 1, w = j & 1;
        mbar_wait(&bars[H1F + w], (j >> 1) & 1);
        mbar_wait(&bars[D2E + w], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        if (leader) {
          const uint64_t dA = dH10 + static_cast<uint64_t>((w * Lay_::H1_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < KR / 16; ++kk) {
            const uint64_t off = static_cast<uint64_t>((kk * 32) >> 4);
            mma_bf16_ss(tmem + 256 + w * 128, dA + off, dWB + off, idesc2, kk > 0 ? 1u : 0u);
          }
          mma_commit(&bars[H1E + w]);
          mma_commit(&bars[D2F + w]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue warpgroups
    const int w = (warp - 4) >> 2;
    const int row = (threadIdx.x - 128) & 127;
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t tD1 = lane_addr + w * 128;
    const uint32_t tD2 = lane_addr + 256 + w * 128;
    uint8_t* h1row = sH1 + w * Lay_::H1_BYTES;
    const int64_t hw = static_cast<int64_t>(a.Hg) * a.Wg;
    for (int i = w; i < n_my; i += 2) {
      const int n = i >> 1;  // use count of this warpgroup's buffers
      const int64_t tok = static_cast<int64_t>(first + i * stride) * M + row;
      const bool live = tok < a.L;
      const int64_t tt = live ? tok : a.L - 1;
      const int ct = static_cast<int>(tt / hw);
      const int cx = a.T + static_cast<int>((tt % hw) / a.Wg);
      const int cy = a.T + a.Hg + static_cast<int>(tt % a.Wg);

      // ---- GEMM1 row -> + Z -> sigmoid -> bf16 H1 row; gate partial
      mbar_wait(&bars[D1F + w], n & 1);
      tc_fence_after();
      uint32_t d1[96];
      tmem_ld32(tD1, d1);
      tmem_ld32(tD1 + 32, d1 + 32);
      if (N1 > 64) tmem_ld32(tD1 + 64, d1 + 64);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars[D1E + w]);
      float gpart = __uint_as_float(d1[R]) + __uint_as_float(d1[R + 1]);
      if (a.use_pe) gpart += (sG[ct] + sG[cx]) + sG[cy];
      uint32_t hp[KR / 2];
      const float* zt = sZ + ct * ZP;
      const float* zx = sZ + cx * ZP;
      const float* zy = sZ + cy * ZP;
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) {
        const float4 a4 = *reinterpret_cast<const float4*>(zt + c4 * 4);
        const float4 b4 = *reinterpret_cast<const float4*>(zx + c4 * 4);
        const float4 e4 = *reinterpret_cast<const float4*>(zy + c4 * 4);
        const float v0 = __uint_as_float(d1[c4 * 4 + 0]) + ((a4.x + b4.x) + e4.x);
        const float v1 = __uint_as_float(d1[c4 * 4 + 1]) + ((a4.y + b4.y) + e4.y);
        const float v2 = __uint_as_float(d1[c4 * 4 + 2]) + ((a4.z + b4.z) + e4.z);
        const float v3 = __uint_as_float(d1[c4 * 4 + 3]) + ((a4.w + b4.w) + e4.w);
        __nv_bfloat162 p0 = __floats2bfloat162_rn(sigmoid_fast(v0), sigmoid_fast(v1));
        __nv_bfloat162 p1 = __floats2bfloat162_rn(sigmoid_fast(v2), sigmoid_fast(v3));
        hp[c4 * 2] = *reinterpret_cast<uint32_t*>(&p0);
        hp[c4 * 2 + 1] = *reinterpret_cast<uint32_t*>(&p1);
      }
#pragma unroll
      for (int c = R / 2; c < KR / 2; ++c) hp[c] = 0u;
      mbar_wait(&bars[H1E + w], (n & 1) ^ 1);
#pragma unroll
      for (int c = 0; c < KR / 8; ++c)
        *reinterpret_cast<uint4*>(h1row + sw128(row, c)) = make_uint4(hp[4 * c], hp[4 * c + 1], hp[4 * c + 2], hp[4 * c + 3]);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars[H1F + w]);
      if (live) a.g_part[(static_cast<int64_t>(b) * a.H + h) * a.L + tok] = gpart;

      // ---- GEMM2 row -> sigmoid (kept in TMEM) -> RMSNorm -> bf16 y_lr row
      mbar_wait(&bars[D2F + w], n & 1);
      tc_fence_after();
      float ss = 0.f;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tD2 + c * 32, o);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float s = sigmoid_fast(__uint_as_float(o[e]));
          ss = fmaf(s, s, ss);
          o[e] = __float_as_uint(s);
        }
        tmem_st32(tD2 + c * 32, o);
      }
      tmem_wait_st();
      const float inv = rsqrtf(ss * (1.f / D) + a.eps);
      const int64_t yrow = ((static_cast<int64_t>(b) * a.L + tt) * a.H + h) * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tD2 + c * 32, o);
        tmem_wait_ld();
        if (c == D / 32 - 1) {
          tc_fence_before();
          mbar_arrive(&bars[D2E + w]);
        }
        if (!live) continue;
        if (a.o_lr) {
          float* dst = a.o_lr + ((static_cast<int64_t>(b) * a.H + h) * a.L + tok) * D + c * 32;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(dst + e) = make_float4(__uint_as_float(o[e]), __uint_as_float(o[e + 1]),
                                                              __uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
        }
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 wv = *reinterpret_cast<const float2*>(a.rms_lr + c * 32 + 2 * e);
          __nv_bfloat162 hb = __floats2bfloat162_rn(__uint_as_float(o[2 * e]) * inv * wv.x,
                                                    __uint_as_float(o[2 * e + 1]) * inv * wv.y);
          pk[e] = *reinterpret_cast<uint32_t*>(&hb);
        }
        uint4* dst = reinterpret_cast<uint4*>(a.y_lr + yrow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e) __stcs(dst + e, make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// g_logit[b, l] = sum_h g_part[b, h, l] in fixed head order (deterministic).
__global__ void gate_sum_kernel(const float* __restrict__ g_part, int H, int64_t L, int64_t BL,
                                float* __restrict__ g_logit) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= BL) return;
  const int64_t b = e / L, l = e % L;
  const float* src = g_part + b * H * L + l;
  float s = 0.f;
  for (int h = 0; h < H; ++h) s += src[static_cast<int64_t>(h) * L];
  g_logit[e] = s;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

size_t up(size_t x) { return (x + 255) / 256 * 256; }

template <int R>
size_t ws_bytes(int64_t B, int64_t H, int64_t L, int nrows) {
  return up(static_cast<size_t>(H) * Lay<R>::WA_BYTES) + up(static_cast<size_t>(H) * Lay<R>::WB_BYTES) +
         up(static_cast<size_t>(H) * nrows * R * 4) + up(static_cast<size_t>(H) * nrows * 4) +
         up(static_cast<size_t>(B * H * L) * 4);
}

template <int R>
int launch(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b,
           const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* g_logit, void* ws, cudaStream_t st) {
  const int H = static_cast<int>(s->H);
  const int nrows = t->grid_t + t->grid_h + t->grid_w;
  uint8_t* p = static_cast<uint8_t*>(ws);
  FoldArgs f;
  f.w_a = w_a;
  f.w_b = w_b;
  f.alpha = t->alpha;
  f.w_g = t->w_g;
  f.pe_t = t->pe_t;
  f.pe_x = t->pe_x;
  f.pe_y = t->pe_y;
  f.d_model = t->d_model;
  f.head_offset = t->head_offset;
  f.H = H;
  f.r = R;
  f.T = t->grid_t;
  f.Hg = t->grid_h;
  f.Wg = t->grid_w;
  f.use_pe = t->use_pe;
  f.wa_img = p;
  p += up(static_cast<size_t>(H) * Lay<R>::WA_BYTES);
  f.wb_img = p;
  p += up(static_cast<size_t>(H) * Lay<R>::WB_BYTES);
  f.Z = reinterpret_cast<float*>(p);
  p += up(static_cast<size_t>(H) * nrows * R * 4);
  f.G = reinterpret_cast<float*>(p);
  p += up(static_cast<size_t>(H) * nrows * 4);
  float* g_part = reinterpret_cast<float*>(p);
  lowrank_fold_umma_kernel<R><<<dim3(nrows + 2, H), 128, 0, st>>>(f);
  if (launch_status()) return ROPESLR_ERR_LAUNCH;

  auto enc = encode_fn();
  if (enc == nullptr) return ROPESLR_ERR_LAUNCH;
  CUtensorMap mx;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(H * D), static_cast<cuuint64_t>(s->B * s->L)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(t->x_row_stride) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(M)};
  cuuint32_t es[2] = {1, 1};
  if (enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(t->x), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return ROPESLR_ERR_LAUNCH;

  MainArgs m;
  m.wa_img = f.wa_img;
  m.wb_img = f.wb_img;
  m.Z = f.Z;
  m.G = f.G;
  m.rms_lr = rms_lowrank;
  m.eps = eps;
  m.L = s->L;
  m.H = H;
  m.T = t->grid_t;
  m.Hg = t->grid_h;
  m.Wg = t->grid_w;
  m.use_pe = t->use_pe;
  m.ntiles = static_cast<int>(ceil_div(s->L, M));
  m.y_lr = static_cast<__nv_bfloat16*>(y_lr);
  m.o_lr = o_lr;
  m.g_part = g_part;
  const int64_t BH = s->B * H;
  int64_t per = num_sms() / BH;
  if (per < 1) per = 1;
  if (per > m.ntiles) per = m.ntiles;
  const int smem = Lay<R>::bytes(nrows);
  auto kfn = lowrank_umma_kernel<R>;
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  kfn<<<dim3(static_cast<unsigned>(per), static_cast<unsigned>(BH)), kThreads, smem, st>>>(mx, m);
  if (launch_status()) return ROPESLR_ERR_LAUNCH;
  if (g_logit != nullptr) {
    const int64_t BL = s->B * s->L;
    gate_sum_kernel<<<static_cast<unsigned>(ceil_div(BL, 256)), 256, 0, st>>>(g_part, H, s->L, BL, g_logit);
  }
  return launch_status();
}

}  // namespace lu

// r % 16 == 0, r <= 112 keeps GEMM1's N (r + 16) within one 128-column TMEM
// buffer; the per-axis tables must fit in shared memory.
bool lowrank_umma_eligible(const ropeslr_shape* s, const ropeslr_token_args* t, int r) {
  if (s->dtype != ROPESLR_BF16 || s->d != lu::D) return false;
  if (r != 16 && r != 32 && r != 48 && r != 64) return false;
  if (s->B * s->L > 0x7fffffffLL) return false;
  const int nrows = t->grid_t + t->grid_h + t->grid_w;
  const int bytes = r <= 16 ? lu::Lay<16>::bytes(nrows) : r <= 32 ? lu::Lay<32>::bytes(nrows)
                  : r <= 48 ? lu::Lay<48>::bytes(nrows) : lu::Lay<64>::bytes(nrows);
  return bytes <= 227 * 1024;
}

size_t lowrank_umma_workspace_bytes(const ropeslr_shape* s, const ropeslr_token_args* t, int r) {
  const int nrows = t->grid_t + t->grid_h + t->grid_w;
  switch (r) {
    case 16: return lu::ws_bytes<16>(s->B, s->H, s->L, nrows);
    case 32: return lu::ws_bytes<32>(s->B, s->H, s->L, nrows);
    case 48: return lu::ws_bytes<48>(s->B, s->H, s->L, nrows);
    default: return lu::ws_bytes<64>(s->B, s->H, s->L, nrows);
  }
}

int launch_lowrank_umma(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b,
                        int r, const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* g_logit,
                        void* ws, cudaStream_t st) {
  switch (r) {
    case 16: return lu::launch<16>(s, t, w_a, w_b, rms_lowrank, eps, y_lr, o_lr, g_logit, ws, st);
    case 32: return lu::launch<32>(s, t, w_a, w_b, rms_lowrank, eps, y_lr, o_lr, g_logit, ws, st);
    case 48: return lu::launch<48>(s, t, w_a, w_b, rms_lowrank, eps, y_lr, o_lr, g_logit, ws, st);
    case 64: return lu::launch<64>(s, t, w_a, w_b, rms_lowrank, eps, y_lr, o_lr, g_logit, ws, st);
    default: return ROPESLR_ERR_SHAPE;
  }
}

}  // namespace ropeslr
