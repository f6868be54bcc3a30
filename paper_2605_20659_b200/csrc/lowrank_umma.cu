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
//                 boxes, 128-byte swizzle) into a 4-stage ring
//   warp 1        MMA issuer:  D1_w = X W_A^T    (M 128, N r+16, K 128, A/B smem)
//                              D2_w = H1_w W_B^T (M 128, N 128, K 64, A in TMEM)
//                 as soon as their inputs are ready (GEMM2 first)
//   warp 2        TMEM allocation (512 columns)
//   warps 4-15    three epilogue warpgroups, WG w owns tiles i = w (mod 3),
//                 the TMEM columns [128w, 128w + 128) (D1, then D2) and
//                 [384 + 32w, +32) (H1_w).  Thread = token row: D1 row + Z
//                 gathers -> sigmoid -> bf16 pairs stored to H1_w in TMEM
//                 (GEMM2's A operand); gate partial; D2 row -> sigmoid ->
//                 RMSNorm * rms_lowrank -> bf16 y_lr row.
// Shared memory holds the 4-stage X ring (128 KiB, enough bytes in flight to
// cover HBM latency), the W_A / W_B images and the Z / G tables; the last
// three are one contiguous per-head blob in the tables buffer, staged by a
// single bulk copy that overlaps the CTA's set-up and first X loads (the
// per-thread staging it replaced was ~10% of a 21-tile CTA at the Wan shape).
// HBM traffic per (token, head): 256 B of X in, 256 B of y_lr out.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
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
constexpr int XSTAGES = 4;
constexpr int NWG = 3;                 // epilogue warpgroups
constexpr int kThreads = 128 + NWG * 128;
constexpr uint32_t H1_COL = 384;       // TMEM columns [384 + 32w, 384 + 32w + 32): H1_w, bf16 pairs

// One head's parameter-only operands ("blob"), laid out identically in the
// tables buffer (per head, contiguous) and in shared memory, so the kernel
// stages them with one bulk copy: W_A^T image | W_B^T image | Z [nrows][ZP]
// f32 | G [nrows] f32 (padded to 16 bytes).
template <int R>
struct Lay {
  static constexpr int N1 = R + 16;              // GEMM1 N: rank + gate hi / lo (+ zero pad)
  static constexpr int X_BYTES = M * D * 2;      // 32 KiB
  static constexpr int WA_BYTES = N1 * D * 2;    // two 64-col atoms of N1 rows
  static constexpr int WB_BYTES = D * KR * 2;    // 16 KiB
  static_assert(WA_BYTES % 1024 == 0, "W_B^T image must stay 1024-byte aligned");
  static constexpr int ZP = R + 4;               // Z row pitch (floats): float4 rows spread over the banks
  static constexpr int OFF_X = 0;
  static constexpr int OFF_BAR = OFF_X + XSTAGES * X_BYTES;
  static constexpr int NBAR = 2 * XSTAGES + 4 * NWG + 1;  // X ring full/empty + 4 per warpgroup + blob
  static constexpr int OFF_RMS = OFF_BAR + 256;           // rms_lowrank [128] f32
  static constexpr int OFF_WA = OFF_RMS + 1024 - 256;     // the blob, 1024-byte aligned
  static constexpr int OFF_WB = OFF_WA + WA_BYTES;
  static constexpr int OFF_TAB = OFF_WB + WB_BYTES;       // Z, then G
  static_assert(NBAR * 8 + 4 <= 256, "barrier block overflows");
  static_assert(OFF_RMS + D * 4 <= OFF_WA && OFF_WA % 1024 == 0, "smem layout");
  __host__ __device__ static int tab_bytes(int nrows) { return (nrows * (ZP + 1) * 4 + 15) / 16 * 16; }
  __host__ __device__ static int blob_bytes(int nrows) { return WA_BYTES + WB_BYTES + tab_bytes(nrows); }
  __host__ __device__ static int bytes(int nrows) { return OFF_WA + blob_bytes(nrows); }
};

// Per warpgroup w: D1F (GEMM1 done), H1F (H1 written to TMEM), D2F (GEMM2
// done), RE (its TMEM region read out: the next GEMM1 may overwrite it).
enum Bar { XF = 0, XE = XSTAGES, D1F = 2 * XSTAGES, H1F = D1F + NWG, D2F = H1F + NWG, RE = D2F + NWG,
           BLOB = RE + NWG, BAR_END = BLOB + 1 };
static_assert(BAR_END == 2 * XSTAGES + 4 * NWG + 1, "barrier enum and Lay::NBAR disagree");

struct FoldArgs {
  const float* w_a;   // [H, d, r]
  const float* w_b;   // [H, r, d]
  const float* alpha; // [D_total]
  const float* w_g;   // [D_total]
  const float *pe_t, *pe_x, *pe_y;  // [n, D_total]
  int64_t d_model, head_offset;
  int H, r, T, Hg, Wg, use_pe;
  uint8_t* blob;      // [H][Lay::blob_bytes(nrows)]: swizzled W_A^T / W_B^T images, Z, G
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
    uint8_t* img = a.blob + static_cast<int64_t>(h) * Lay<R>::blob_bytes(nrows);
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
    uint8_t* img = a.blob + static_cast<int64_t>(h) * Lay<R>::blob_bytes(nrows) + Lay<R>::WA_BYTES;
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
  float* ztab = reinterpret_cast<float*>(a.blob + static_cast<int64_t>(h) * Lay<R>::blob_bytes(nrows) +
                                         Lay<R>::WA_BYTES + Lay<R>::WB_BYTES);
  float* zrow = ztab + i * Lay<R>::ZP;
  float* grow = ztab + nrows * Lay<R>::ZP + i;
  if (!a.use_pe) {
    for (int j = tid; j < Lay<R>::ZP; j += blockDim.x) zrow[j] = 0.f;
    if (tid == 0) *grow = 0.f;
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
  } else if (tid < Lay<R>::ZP) {
    zrow[tid] = 0.f;  // pitch padding
  }
  if (tid == 0) *grow = (red[0] + red[1]) + (red[2] + red[3]);
}

struct MainArgs {
  const uint8_t* blob;  // [H][Lay::blob_bytes(nrows)]
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
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay_::OFF_BAR);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Lay_::OFF_BAR + Lay_::NBAR * 8);
  float* sRms = reinterpret_cast<float*>(smem + Lay_::OFF_RMS);
  const int nrows = a.T + a.Hg + a.Wg;
  float* sZ = reinterpret_cast<float*>(smem + Lay_::OFF_TAB);
  float* sG = sZ + nrows * ZP;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y;
  const int b = bh / a.H, h = bh % a.H;

  // The head's blob (W_A^T / W_B^T images, Z, G) arrives by one bulk copy,
  // issued right after the barriers are initialised, behind nothing; the MMA
  // warp and the epilogue wait on its barrier before their first use.
  for (int e = threadIdx.x; e < D; e += kThreads) sRms[e] = a.rms_lr[e];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < Lay_::NBAR; ++i) {
      const bool per_thread = (i >= H1F && i < H1F + NWG) || (i >= RE && i < RE + NWG);
      mbar_init(&bars[i], per_thread ? 128 : 1);
    }
    fence_mbar_init();
    const uint32_t blob_bytes = static_cast<uint32_t>(Lay_::blob_bytes(nrows));
    mbar_arrive_expect_tx(&bars[BLOB], blob_bytes);
    bulk_load_1d(sWA, a.blob + static_cast<int64_t>(h) * blob_bytes, blob_bytes, &bars[BLOB], policy_evict_last());
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
    // Tile i belongs to warpgroup w = i % NWG and its 128-column TMEM region
    // (GEMM1 writes columns [0, N1), GEMM2 then all 128).  The warp polls
    // instead of issuing in a fixed order: GEMM2 of the oldest tile whose H1
    // is ready goes first, else GEMM1 of the next tile once its X stage has
    // landed and its region has been drained -- so no warpgroup waits behind
    // another one's epilogue.
    constexpr uint32_t idesc1 = idesc_bf16_f32(M, N1, false, false);
    constexpr uint32_t idesc2 = idesc_bf16_f32(M, D, false, false);
    const uint64_t dX0 = desc_sw128(smem_u32(sX), 16, 1024);
    const uint64_t dWA = desc_sw128(smem_u32(sWA), 16, 1024);
    const uint64_t dWB = desc_sw128(smem_u32(sWB), 16, 1024);
    const bool leader = elect_one();
    mbar_wait(&bars[BLOB], 0);
    int n1 = 0, n2 = 0;
    while (n2 < n_my) {
      bool issued = false;
      if (n2 < n1) {
        const int w = n2 % NWG;
        if (__all_sync(0xffffffffu, mbar_try_wait(&bars[H1F + w], (n2 / NWG) & 1))) {
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < KR / 16; ++kk) {
              const uint64_t off = static_cast<uint64_t>((kk * 32) >> 4);
              mma_bf16_ts(tmem + w * 128, tmem + H1_COL + w * 32 + kk * 8, dWB + off, idesc2, kk > 0 ? 1u : 0u);
            }
            mma_commit(&bars[D2F + w]);
          }
          __syncwarp();
          ++n2;
          issued = true;
        }
      }
      if (!issued && n1 < n_my) {
        const int s = n1 % XSTAGES, w = n1 % NWG;
        if (__all_sync(0xffffffffu, mbar_try_wait(&bars[XF + s], (n1 / XSTAGES) & 1) &&
                                        mbar_try_wait(&bars[RE + w], ((n1 / NWG) & 1) ^ 1))) {
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
          ++n1;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue warpgroups
    const int w = (warp - 4) >> 2;
    const int row = (threadIdx.x - 128) & 127;
    const uint32_t tlane = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t treg = tlane + w * 128;
    const uint32_t th1 = tlane + H1_COL + w * 32;
    const int hw = a.Hg * a.Wg;
    if (w < n_my) mbar_wait(&bars[BLOB], 0);
    for (int i = w; i < n_my; i += NWG) {
      const uint32_t ph = (i / NWG) & 1;
      const int t = first + i * stride;
      const int64_t tok = static_cast<int64_t>(t) * M + row;
      const bool live = tok < a.L;
      const int tt = static_cast<int>(live ? tok : a.L - 1);
      const int ct = tt / hw;
      const int rem = tt - ct * hw;
      const int cxr = rem / a.Wg;
      const int cx = a.T + cxr;
      const int cy = a.T + a.Hg + (rem - cxr * a.Wg);

      // ---- GEMM1 row (+ Z gathers) -> sigmoid -> bf16 H1 row; gate partial
      mbar_wait(&bars[D1F + w], ph);
      tc_fence_after();
      // one round trip: all of the row's GEMM1 columns (+ the gate pair) at once
      uint32_t d1[R];
      uint32_t gg[2];
#pragma unroll
      for (int c = 0; c < R / 16; ++c) tmem_ld16(treg + c * 16, d1 + c * 16);
      tmem_ld2(treg + R, gg);
      tmem_wait_ld();
      float gpart = __uint_as_float(gg[0]) + __uint_as_float(gg[1]);
      if (a.use_pe) gpart += (sG[ct] + sG[cx]) + sG[cy];
      const float* zt = sZ + ct * ZP;
      const float* zx = sZ + cx * ZP;
      const float* zy = sZ + cy * ZP;
#pragma unroll
      for (int c = 0; c < R / 16; ++c) {
        uint32_t hp[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int col = c * 16 + q * 4;
          const float4 a4 = *reinterpret_cast<const float4*>(zt + col);
          const float4 b4 = *reinterpret_cast<const float4*>(zx + col);
          const float4 e4 = *reinterpret_cast<const float4*>(zy + col);
          const float v0 = __uint_as_float(d1[col + 0]) + ((a4.x + b4.x) + e4.x);
          const float v1 = __uint_as_float(d1[col + 1]) + ((a4.y + b4.y) + e4.y);
          const float v2 = __uint_as_float(d1[col + 2]) + ((a4.z + b4.z) + e4.z);
          const float v3 = __uint_as_float(d1[col + 3]) + ((a4.w + b4.w) + e4.w);
          __nv_bfloat162 p0 = __floats2bfloat162_rn(sigmoid_fast(v0), sigmoid_fast(v1));
          __nv_bfloat162 p1 = __floats2bfloat162_rn(sigmoid_fast(v2), sigmoid_fast(v3));
          hp[q * 2] = *reinterpret_cast<uint32_t*>(&p0);
          hp[q * 2 + 1] = *reinterpret_cast<uint32_t*>(&p1);
        }
        tmem_st8(th1 + c * 8, hp);
      }
      if (R < KR) {
        const uint32_t zero[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
        for (int c = R / 16; c < KR / 16; ++c) tmem_st8(th1 + c * 8, zero);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars[H1F + w]);
      if (live) a.g_part[(static_cast<int64_t>(b) * a.H + h) * a.L + tok] = gpart;

      // ---- GEMM2 row -> sigmoid -> RMSNorm -> bf16 y_lr row.  Pass 1 reads
      // the row in two 64-column halves (one TMEM round trip each), applies
      // the sigmoid, accumulates the fp32 sum of squares and writes the
      // values back as fp16 pairs (2^-11 relative rounding, an eighth of the
      // final bf16 ulp) into columns [0, 64) of the region; pass 2 reads those
      // 64 packed columns in one round trip.
      mbar_wait(&bars[D2F + w], ph);
      tc_fence_after();
      float ss = 0.f;
#pragma unroll
      for (int p2 = 0; p2 < 2; ++p2) {
        uint32_t o[64];
        tmem_ld32(treg + p2 * 64, o);
        tmem_ld32(treg + p2 * 64 + 32, o + 32);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          const float s0 = sigmoid_fast(__uint_as_float(o[e]));
          const float s1 = sigmoid_fast(__uint_as_float(o[e + 1]));
          ss = fmaf(s0, s0, ss);
          ss = fmaf(s1, s1, ss);
          __half2 hh = __floats2half2_rn(s0, s1);
          o[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
        }
        tmem_st32(treg + p2 * 32, o);
      }
      tmem_wait_st();
      uint32_t sv[D / 2];
      tmem_ld32(treg, sv);
      tmem_ld32(treg + 32, sv + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars[RE + w]);
      if (!live) continue;
      const float inv = rsqrtf(ss * (1.f / D) + a.eps);
      const int64_t yrow = ((static_cast<int64_t>(b) * a.L + tt) * a.H + h) * D;
      uint4* dst = reinterpret_cast<uint4*>(a.y_lr + yrow);
      uint32_t packed[8];  // 16 columns: one 256-bit store (a full 32-byte sector per thread)
#pragma unroll
      for (int e = 0; e < D / 8; ++e) {
        const float4 w0 = *reinterpret_cast<const float4*>(sRms + 8 * e);
        const float4 w1 = *reinterpret_cast<const float4*>(sRms + 8 * e + 4);
        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&sv[4 * e]));
        const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&sv[4 * e + 1]));
        const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&sv[4 * e + 2]));
        const float2 f3 = __half22float2(*reinterpret_cast<const __half2*>(&sv[4 * e + 3]));
        __nv_bfloat162 p0 = __floats2bfloat162_rn(f0.x * inv * w0.x, f0.y * inv * w0.y);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(f1.x * inv * w0.z, f1.y * inv * w0.w);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(f2.x * inv * w1.x, f2.y * inv * w1.y);
        __nv_bfloat162 p3 = __floats2bfloat162_rn(f3.x * inv * w1.z, f3.y * inv * w1.w);
        const int o4 = (e & 1) * 4;
        packed[o4 + 0] = *reinterpret_cast<uint32_t*>(&p0);
        packed[o4 + 1] = *reinterpret_cast<uint32_t*>(&p1);
        packed[o4 + 2] = *reinterpret_cast<uint32_t*>(&p2);
        packed[o4 + 3] = *reinterpret_cast<uint32_t*>(&p3);
        if (e & 1)
          asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + e - 1),
                       "r"(packed[0]), "r"(packed[1]), "r"(packed[2]), "r"(packed[3]), "r"(packed[4]),
                       "r"(packed[5]), "r"(packed[6]), "r"(packed[7])
                       : "memory");
        if (a.o_lr) {
          float* od = a.o_lr + ((static_cast<int64_t>(b) * a.H + h) * a.L + tok) * D + 8 * e;
          *reinterpret_cast<float4*>(od) = make_float4(f0.x, f0.y, f1.x, f1.y);
          *reinterpret_cast<float4*>(od + 4) = make_float4(f2.x, f2.y, f3.x, f3.y);
        }
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

// The parameter-only part of the workspace (W_A^T / W_B^T images, Z, G),
// then the gate partials.
template <int R>
size_t tables_bytes(int64_t H, int nrows) {
  return up(static_cast<size_t>(H) * Lay<R>::blob_bytes(nrows));
}

template <int R>
size_t ws_bytes(int64_t B, int64_t H, int64_t L, int nrows) {
  return tables_bytes<R>(H, nrows) + up(static_cast<size_t>(B * H * L) * 4);
}

// The fold kernel's outputs inside a tables buffer.
template <int R>
FoldArgs fold_args(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b,
                   void* tables) {
  const int H = static_cast<int>(s->H);
  uint8_t* p = static_cast<uint8_t*>(tables);
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
  f.blob = p;
  return f;
}

template <int R>
int fold(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b, void* tables,
         cudaStream_t st) {
  const FoldArgs f = fold_args<R>(s, t, w_a, w_b, tables);
  const int nrows = t->grid_t + t->grid_h + t->grid_w;
  lowrank_fold_umma_kernel<R><<<dim3(nrows + 2, f.H), 128, 0, st>>>(f);
  return launch_status();
}

// The main kernel (+ the gate sum) from folded tables; g_part: B*H*L floats.
template <int R>
int run_main(const ropeslr_shape* s, const ropeslr_token_args* t, const void* tables, const float* rms_lowrank,
             float eps, void* y_lr, float* o_lr, float* g_logit, float* g_part, cudaStream_t st) {
  const int H = static_cast<int>(s->H);
  const int nrows = t->grid_t + t->grid_h + t->grid_w;
  const FoldArgs f = fold_args<R>(s, t, nullptr, nullptr, const_cast<void*>(tables));
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
  m.blob = f.blob;
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

template <int R>
int launch(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b,
           const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* g_logit, void* ws, cudaStream_t st) {
  const int nrows = t->grid_t + t->grid_h + t->grid_w;
  if (int e = fold<R>(s, t, w_a, w_b, ws, st)) return e;
  float* g_part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + tables_bytes<R>(s->H, nrows));
  return run_main<R>(s, t, ws, rms_lowrank, eps, y_lr, o_lr, g_logit, g_part, st);
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

size_t lowrank_umma_tables_bytes(const ropeslr_shape* s, const ropeslr_token_args* t, int r) {
  const int nrows = t->grid_t + t->grid_h + t->grid_w;
  switch (r) {
    case 16: return lu::tables_bytes<16>(s->H, nrows);
    case 32: return lu::tables_bytes<32>(s->H, nrows);
    case 48: return lu::tables_bytes<48>(s->H, nrows);
    default: return lu::tables_bytes<64>(s->H, nrows);
  }
}

int lowrank_umma_fold(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b, int r,
                      void* tables, cudaStream_t st) {
  switch (r) {
    case 16: return lu::fold<16>(s, t, w_a, w_b, tables, st);
    case 32: return lu::fold<32>(s, t, w_a, w_b, tables, st);
    case 48: return lu::fold<48>(s, t, w_a, w_b, tables, st);
    case 64: return lu::fold<64>(s, t, w_a, w_b, tables, st);
    default: return ROPESLR_ERR_SHAPE;
  }
}

int lowrank_umma_folded(const ropeslr_shape* s, const ropeslr_token_args* t, int r, const void* tables,
                        const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* g_logit, float* g_part,
                        cudaStream_t st) {
  switch (r) {
    case 16: return lu::run_main<16>(s, t, tables, rms_lowrank, eps, y_lr, o_lr, g_logit, g_part, st);
    case 32: return lu::run_main<32>(s, t, tables, rms_lowrank, eps, y_lr, o_lr, g_logit, g_part, st);
    case 48: return lu::run_main<48>(s, t, tables, rms_lowrank, eps, y_lr, o_lr, g_logit, g_part, st);
    case 64: return lu::run_main<64>(s, t, tables, rms_lowrank, eps, y_lr, o_lr, g_logit, g_part, st);
    default: return ROPESLR_ERR_SHAPE;
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
