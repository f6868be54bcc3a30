// K2 + K4: block-sparse softmax attention on the 5th-generation tensor cores
// with the fused RoPeSLR epilogue (mechanism.py:321-326 and 437-451).
//
// One persistent CTA per SM walks work units (bh, query block) in head-major
// order, so the ~150 CTAs in flight read the K/V blocks of one or two heads
// and those stay resident in the 126 MB L2.  Per unit:
//
//   warp 0  TMA producer   Q tile once per unit, then K_j for every selected
//                          key block j (contiguous [block, 128] boxes of the
//                          [B*H, L, d] tensors, 128-byte swizzle), 2-stage ring.
//   warp 3  TMA producer   V_j, its own 2-stage ring (a V slot frees only after
//                          its PV, so it must not hold back the K prefetch).
//   warp 1  MMA issuer     S_w = Q K_j^T into TMEM for w = j & 1, then
//                          O_w += P_w V_j; tcgen05.commit releases smem
//                          stages and signals the softmax warpgroups.
//   warp 2  TMEM owner     alloc / dealloc of the 512 columns.
//   warps 4-7, 8-11        two softmax warpgroups; WG w owns the key blocks
//                          j = w, w+2, ... of the unit with its own online
//                          softmax state and its own TMEM accumulator O_w
//                          (split-K over the key list).  One query row per
//                          thread: tcgen05.ld of the S row, exp2-domain
//                          softmax with the lazy (threshold 8) rescale of
//                          O_w, bf16 P into swizzled smem for the PV MMA.
//                          Two warps per SMSP hide each other's latency.
//                          Epilogue: O = sum_w O_w 2^(m_w-m) / l, RMSNorm *
//                          rms_sparse, + sigmoid(g_logit + b_g) * y_lr, bf16
//                          store; WG w finalises columns [64w, 64w+64).
//
// TMEM columns: S0 [0,128), S1 [128,256), O0 [256,384), O1 [384,512).
// Shared memory (block 128): Q 32K, K 2x32K, V 2x32K, P 2x32K = 224 KiB.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace ropeslr {

int launch_sparse_attention_simt(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                                 const int32_t* idx, int kmax, const int32_t* cnt, const int32_t* perm,
                                 float* o_sparse, cudaStream_t st);

namespace tc {

using namespace sm100;

constexpr int D = 128;   // head dim handled by this kernel
constexpr int M = 128;   // MMA rows (query rows per tile)
constexpr int kThreads = 384;  // 4 control warps + 2 softmax warpgroups

template <int BLK>
struct Layout {
  static constexpr int Q_BYTES = M * D * 2;
  static constexpr int KV_BYTES = BLK * D * 2;
  static constexpr int P_BYTES = M * BLK * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;
  static constexpr int OFF_P = OFF_V + 2 * KV_BYTES;
  static constexpr int OFF_XCH = OFF_P + 2 * P_BYTES;      // epilogue exchange, 2 KiB
  static constexpr int OFF_BAR = OFF_XCH + 2048;
  static constexpr int NBAR = 22;
  static constexpr int BYTES = OFF_BAR + NBAR * 8 + 16;
  // dynamic smem starts 1024-aligned (after the driver's 1 KiB reservation);
  // the kernel traps if that ever changes
  static constexpr int ALLOC = BYTES;
};

enum Bar {
  Q_FULL = 0,
  Q_EMPTY = 1,
  K_FULL = 2,   // +stage
  K_EMPTY = 4,  // +stage
  V_FULL = 6,
  V_EMPTY = 8,
  S_FULL = 10,
  S_EMPTY = 12,
  P_FULL = 14,
  P_EMPTY = 16,
  PV_DONE = 18,
  O_FULL = 20,
  O_EMPTY = 21
};

struct Params {
  const int32_t* idx;
  const int32_t* cnt;
  int kmax;
  int nb;
  int H;
  int64_t L;
  int64_t num_units;
  const int32_t* perm;
  float scale_log2;
  const __nv_bfloat16* y_lr;
  const float* g_logit;
  float b_g;
  const float* rms_sp;
  float eps;
  __nv_bfloat16* out;
  float* o_sparse;
  int out_H;   // heads per token row of out / y_lr (>= H when a head chunk writes into a wider row)
  int out_h0;  // first head of this call inside that row
  int kv_evict_last;
  int debug_mode;  // 0 normal; 1 no softmax math; 2 every K/V load hits block 0; 3 no K/V TMA
};

__device__ __forceinline__ bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe for a pair: x = n + f (n = rint(x), |f| <= 1/2),
// 2^f by a degree-3 minimax polynomial (max rel. error 7.5e-5, far below the
// bf16 rounding of P), 2^n added to the exponent field.  x is clamped at -126.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 q = __ffma2_rn(make_float2(0.05517125502228737f, 0.05517125502228737f), f,
                        make_float2(0.2426103800535202f, 0.2426103800535202f));
  q = __ffma2_rn(q, f, make_float2(0.6932609677314758f, 0.6932609677314758f));
  q = __ffma2_rn(q, f, make_float2(0.9999281167984009f, 0.9999281167984009f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

template <int BLK>
__global__ void __launch_bounds__(kThreads, 1)
    sparse_attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const Params p) {
  using Lay = Layout<BLK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint8_t* sP = smem + Lay::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Lay::OFF_BAR + Lay::NBAR * 8);
  float2* xch_ml = reinterpret_cast<float2*>(smem + Lay::OFF_XCH);  // [2][128] (m, l), then (ss, -)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < Lay::NBAR; ++i) {
      uint32_t count = 1;
      if (i == S_EMPTY || i == S_EMPTY + 1 || i == P_FULL || i == P_FULL + 1) count = 128;
      if (i == O_EMPTY) count = 256;
      mbar_init(&bars[i], count);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  if (BLK < M && warp >= 4 && warp < 8) {
    // query rows [BLK, 128) of the MMA tile are never loaded: keep them zero
    const int t = threadIdx.x - 128;
    for (int half = 0; half < 2; ++half) {
      uint4* z = reinterpret_cast<uint4*>(sQ + half * (M * 128) + BLK * 128);
      for (int i = t; i < (M - BLK) * 128 / 16; i += 128) z[i] = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0 || warp == 3) {
    if (elect_one_sync()) {
      // ------------------------------------------- TMA producers
      // warp 0: Q and K (K runs ahead: a K slot frees as soon as its QK^T
      // completes); warp 3: V (a V slot frees only after its PV).
      const bool is_k = (warp == 0);
      const uint64_t pol_kv = p.kv_evict_last ? policy_evict_last() : policy_evict_normal();
      const uint64_t pol_q = policy_evict_first();
      const CUtensorMap* map = is_k ? &tmK : &tmV;
      uint8_t* ring = is_k ? sK : sV;
      const int full = is_k ? K_FULL : V_FULL;
      const int empty = is_k ? K_EMPTY : V_EMPTY;
      uint32_t g = 0, uc = 0;
      for (int64_t u = blockIdx.x; u < p.num_units; u += gridDim.x, ++uc) {
        const int bh = static_cast<int>(u / p.nb);
        const int n = p.cnt[u];
        const int32_t* irow = p.idx + u * p.kmax;
        if (is_k) {
          const int qb = static_cast<int>(u % p.nb);
          mbar_wait(&bars[Q_EMPTY], (uc & 1) ^ 1);
          mbar_arrive_expect_tx(&bars[Q_FULL], 2 * BLK * 128);
          tma_load_3d_hint(sQ, &tmQ, &bars[Q_FULL], 0, qb * BLK, bh, pol_q);
          tma_load_3d_hint(sQ + M * 128, &tmQ, &bars[Q_FULL], 64, qb * BLK, bh, pol_q);
        }
        for (int j = 0; j < n; ++j, ++g) {
          const int kb = p.debug_mode == 2 ? 0 : irow[j];
          const int s = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          uint8_t* dst = ring + s * Lay::KV_BYTES;
          mbar_wait(&bars[empty + s], ph ^ 1);
          if (p.debug_mode == 3) {
            mbar_arrive(&bars[full + s]);
            continue;
          }
          mbar_arrive_expect_tx(&bars[full + s], Lay::KV_BYTES);
          tma_load_3d_hint(dst, map, &bars[full + s], 0, kb * BLK, bh, pol_kv);
          tma_load_3d_hint(dst + BLK * 128, map, &bars[full + s], 64, kb * BLK, bh, pol_kv);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // The whole warp runs the (uniform) control flow and waits; one elected
    // lane issues tcgen05.mma / commit, so descriptors live in uniform
    // registers.  Key block j is owned by softmax warpgroup w = j & 1:
    // S_w = Q K_j^T, P_w from that WG, O_w += P_w V_j.  Issue order per unit:
    // QK(0), QK(1), [QK(j), PV(j-2)] for j >= 2, then PV(n-2), PV(n-1).
    constexpr uint32_t idesc_qk = idesc_bf16_f32(M, BLK, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(M, D, false, true);
    // descriptor bases; the K-step offsets below are added to the low word
    // (start address field, 16-byte units, no carry: smem < 256 KiB)
    const uint64_t dQ = desc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t dK0 = desc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t dV0 = desc_sw128(smem_u32(sV), BLK * 128, 1024);
    const uint64_t dP0 = desc_sw128(smem_u32(sP), 16, 1024);
    const bool leader = elect_one_sync();
    uint32_t g = 0, uc = 0;
    uint32_t qk0 = 0, qk1 = 0, pv0 = 0, pv1 = 0;
    for (int64_t u = blockIdx.x; u < p.num_units; u += gridDim.x, ++uc) {
      const int n = p.cnt[u];
      mbar_wait(&bars[Q_FULL], uc & 1);
      tc_fence_after();
      for (int j = 0; j < n + 2; ++j) {
        if (j < n) {
          const uint32_t gg = g + j;
          const int s = gg & 1;
          const int w = j & 1;
          const uint32_t cntw = w ? qk1 : qk0;
          mbar_wait(&bars[K_FULL + s], (gg >> 1) & 1);
          mbar_wait(&bars[S_EMPTY + w], (cntw & 1) ^ 1);
          tc_fence_after();
          if (leader) {
            const uint32_t tS = tmem + w * 128;
            const uint64_t dK = dK0 + static_cast<uint64_t>((s * Lay::KV_BYTES) >> 4);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint64_t da = dQ + static_cast<uint64_t>(((kk >> 2) * (M * 128) + (kk & 3) * 32) >> 4);
              const uint64_t db = dK + static_cast<uint64_t>(((kk >> 2) * (BLK * 128) + (kk & 3) * 32) >> 4);
              mma_bf16_ss(tS, da, db, idesc_qk, kk > 0 ? 1u : 0u);
            }
            mma_commit(&bars[K_EMPTY + s]);
            mma_commit(&bars[S_FULL + w]);
            if (j == n - 1) mma_commit(&bars[Q_EMPTY]);
          }
          __syncwarp();
          if (w) ++qk1; else ++qk0;
        }
        if (j >= 2) {
          const int jp = j - 2;
          const uint32_t gp = g + jp;
          const int s = gp & 1;
          const int w = jp & 1;
          const uint32_t cntw = w ? pv1 : pv0;
          mbar_wait(&bars[V_FULL + s], (gp >> 1) & 1);
          mbar_wait(&bars[P_FULL + w], cntw & 1);
          if (jp == 0) mbar_wait(&bars[O_EMPTY], (uc & 1) ^ 1);
          tc_fence_after();
          if (leader) {
            const uint32_t tO = tmem + 256 + w * 128;
            const uint64_t dP = dP0 + static_cast<uint64_t>((w * Lay::P_BYTES) >> 4);
            const uint64_t dV = dV0 + static_cast<uint64_t>((s * Lay::KV_BYTES) >> 4);
#pragma unroll
            for (int kk = 0; kk < BLK / 16; ++kk) {
              const uint64_t da = dP + static_cast<uint64_t>(((kk >> 2) * (M * 128) + (kk & 3) * 32) >> 4);
              const uint64_t db = dV + static_cast<uint64_t>((kk * 2048) >> 4);
              mma_bf16_ss(tO, da, db, idesc_pv, (jp >= 2 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&bars[V_EMPTY + s]);
            mma_commit(&bars[P_EMPTY + w]);
          }
          __syncwarp();
          if (w) ++pv1; else ++pv0;
        }
      }
      if (leader) mma_commit(&bars[O_FULL]);
      __syncwarp();
      g += n;
    }
  } else if (warp >= 4) {
    // ------------------------------------ softmax warpgroups + epilogue
    const int w = (warp - 4) >> 2;                 // 0: even key blocks, 1: odd
    const int row = (threadIdx.x - 128) & 127;     // query row == TMEM lane
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t tS = lane_addr + w * 128;
    const uint32_t tO = lane_addr + 256 + w * 128;
    uint8_t* prow_base = sP + w * Lay::P_BYTES + row * 128;
    uint32_t cnt = 0, uc = 0;
    for (int64_t u = blockIdx.x; u < p.num_units; u += gridDim.x, ++uc) {
      const int bh = static_cast<int>(u / p.nb);
      const int qb = static_cast<int>(u % p.nb);
      const int n = p.cnt[u];
      const int32_t* irow = p.idx + u * p.kmax;
      const int qrows = block_size(p.L, BLK, qb);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = w; j < n; j += 2, ++cnt) {
        const int kreal = block_size(p.L, BLK, irow[j]);
        mbar_wait(&bars[S_FULL + w], cnt & 1);
        tc_fence_after();
        if (p.debug_mode == 1) {
          tc_fence_before();
          mbar_arrive(&bars[S_EMPTY + w]);
          mbar_wait(&bars[P_EMPTY + w], (cnt & 1) ^ 1);
          m_run = 0.f;
          l_run = 1.f;
          fence_proxy_async_smem();
          tc_fence_before();
          mbar_arrive(&bars[P_FULL + w]);
          continue;
        }
        // pass 1: row max (TMEM is re-read in pass 2 instead of holding 128 registers)
        float mx = -INFINITY;
#pragma unroll
        for (int h2 = 0; h2 < BLK / 64; ++h2) {
          uint32_t sr[64];
          tmem_ld32(tS + h2 * 64, sr);
          tmem_ld32(tS + h2 * 64 + 32, sr + 32);
          tmem_wait_ld();
          if (kreal == BLK) {
#pragma unroll
            for (int c = 0; c < 64; ++c) mx = fmaxf(mx, __uint_as_float(sr[c]));
          } else {
#pragma unroll
            for (int c = 0; c < 64; ++c)
              if (h2 * 64 + c < kreal) mx = fmaxf(mx, __uint_as_float(sr[c]));
          }
        }
        mx *= p.scale_log2;
        // P_w free <=> this WG's previous PV into O_w has completed
        mbar_wait(&bars[P_EMPTY + w], (cnt & 1) ^ 1);
        if (j == w) {
          m_run = mx;
        } else if (mx > m_run + 8.f) {
          // lazy rescale: only when the running max grows by more than 2^8
          const float alpha = ex2_approx(m_run - mx);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tO + c * 32, o);
          }
          tmem_wait_st();
          l_run *= alpha;
          m_run = mx;
        }
        // pass 2: p = 2^(s * scale - m), bf16 P rows into the swizzled smem tile
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nm2 = make_float2(-m_run, -m_run);
        float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int h2 = 0; h2 < BLK / 64; ++h2) {
          uint32_t sr[64];
          tmem_ld32(tS + h2 * 64, sr);
          tmem_ld32(tS + h2 * 64 + 32, sr + 32);
          tmem_wait_ld();
          if (h2 == BLK / 64 - 1) {
            tc_fence_before();
            mbar_arrive(&bars[S_EMPTY + w]);
          }
          if (kreal < BLK) {
#pragma unroll
            for (int c = 0; c < 64; ++c)
              if (h2 * 64 + c >= kreal) sr[c] = __float_as_uint(-INFINITY);
          }
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            uint32_t pk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int i = cc * 4 + q;
              const float2 x2 =
                  __ffma2_rn(make_float2(__uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1])), sc2, nm2);
              float2 e2;
              if (q == 3) {
                e2 = ex2_poly2(x2);  // FMA-pipe exp2 for 1/4 of the scores: offloads the MUFU
              } else {
                e2.x = ex2_approx(x2.x);
                e2.y = ex2_approx(x2.y);
              }
              sum2 = __fadd2_rn(sum2, e2);
              __nv_bfloat162 hb = __floats2bfloat162_rn(e2.x, e2.y);
              pk[q] = *reinterpret_cast<uint32_t*>(&hb);
            }
            *reinterpret_cast<uint4*>(prow_base + h2 * (M * 128) + ((cc ^ (row & 7)) << 4)) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
        l_run += sum2.x + sum2.y;
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars[P_FULL + w]);
      }
      // ---------------------------------------------- fused epilogue
      // merge the two partial softmaxes: O = sum_w O_w 2^(m_w - m), l likewise
      mbar_wait(&bars[O_FULL], uc & 1);
      tc_fence_after();
      xch_ml[w * 128 + row] = make_float2(m_run, l_run);
      named_bar_sync(1, 256);
      const float2 other = xch_ml[(w ^ 1) * 128 + row];
      const float m0 = w == 0 ? m_run : other.x, l0 = w == 0 ? l_run : other.y;
      const float m1 = w == 0 ? other.x : m_run, l1 = w == 0 ? other.y : l_run;
      const bool has1 = n > 1;  // warpgroup 1 owned at least one key block
      const float mm = has1 ? fmaxf(m0, m1) : m0;
      const float f0 = ex2_approx(m0 - mm);
      const float f1 = has1 ? ex2_approx(m1 - mm) : 0.f;
      const float inv_l = 1.f / (l0 * f0 + l1 * f1);
      const float s0 = f0 * inv_l, s1 = f1 * inv_l;
      // this warpgroup finalises columns [64w, 64w + 64) of its rows, 32 at a
      // time: pass 1 accumulates the sum of squares, pass 2 re-reads TMEM and stores
      auto merged = [&](int c, uint32_t* ob) {
        uint32_t t1[32];
        tmem_ld32(lane_addr + 256 + w * 64 + c * 32, ob);
        if (has1) tmem_ld32(lane_addr + 384 + w * 64 + c * 32, t1);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float o1 = has1 ? __uint_as_float(t1[i]) * s1 : 0.f;
          ob[i] = __float_as_uint(fmaf(__uint_as_float(ob[i]), s0, o1));
        }
      };
      float ss = 0.f;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t ob[32];
        merged(c, ob);
#pragma unroll
        for (int i = 0; i < 32; ++i) ss = fmaf(__uint_as_float(ob[i]), __uint_as_float(ob[i]), ss);
      }
      named_bar_sync(1, 256);  // both warpgroups have read the (m, l) exchange
      xch_ml[w * 128 + row].x = ss;
      named_bar_sync(1, 256);
      ss += xch_ml[(w ^ 1) * 128 + row].x;
      const bool live = row < qrows;
      const int64_t flat = static_cast<int64_t>(qb) * BLK + row;
      const int64_t tok = live ? (p.perm ? p.perm[flat] : flat) : 0;
      const int b = bh / p.H, h = bh % p.H;
      const float inv = 1.f / sqrtf(ss / static_cast<float>(D) + p.eps);
      const float gate = (live && p.out) ? sigmoidf_stable(p.g_logit[static_cast<int64_t>(b) * p.L + tok] + p.b_g) : 0.f;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t ob[32];
        merged(c, ob);
        if (c == 1) {
          tc_fence_before();
          mbar_arrive(&bars[O_EMPTY]);
        }
        if (!live) continue;
        const int col0 = w * 64 + c * 32;
        if (p.o_sparse) {
          float* dst = p.o_sparse + (static_cast<int64_t>(bh) * p.L + tok) * D + col0;
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + i) = make_float4(__uint_as_float(ob[i]), __uint_as_float(ob[i + 1]),
                                                              __uint_as_float(ob[i + 2]), __uint_as_float(ob[i + 3]));
        }
        if (p.out) {
          const int64_t orow = ((static_cast<int64_t>(b) * p.L + tok) * p.out_H + p.out_h0 + h) * D + col0;
          const __nv_bfloat16* y = p.y_lr + orow;
          __nv_bfloat16* dst = p.out + orow;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            const uint4 uy = __ldcs(reinterpret_cast<const uint4*>(y + i));
            const __nv_bfloat162* hy = reinterpret_cast<const __nv_bfloat162*>(&uy);
            uint4 uo;
            __nv_bfloat162* ho = reinterpret_cast<__nv_bfloat162*>(&uo);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 yv = __bfloat1622float2(hy[e]);
              const float o0 = fmaf(gate, yv.x, __uint_as_float(ob[i + 2 * e]) * inv * p.rms_sp[col0 + i + 2 * e]);
              const float o1 = fmaf(gate, yv.y, __uint_as_float(ob[i + 2 * e + 1]) * inv * p.rms_sp[col0 + i + 2 * e + 1]);
              ho[e] = __floats2bfloat162_rn(o0, o1);
            }
            __stcs(reinterpret_cast<uint4*>(dst + i), uo);
          }
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

// ------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// [BH, L, 128] bf16 viewed as a 3-D tensor, box [64 cols, rows, 1], 128B swizzle.
static bool make_map(CUtensorMap* m, const void* base, int64_t BH, int64_t L, int rows) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(BH)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(L) * D * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(rows), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BLK>
static int launch_tc(const ropeslr_shape* s, const void* q, const void* k, const void* v, Params prm,
                     cudaStream_t st) {
  const int64_t BH = s->B * s->H;
  CUtensorMap mq, mk, mv;
  if (!make_map(&mq, q, BH, s->L, BLK) || !make_map(&mk, k, BH, s->L, BLK) || !make_map(&mv, v, BH, s->L, BLK))
    return ROPESLR_ERR_LAUNCH;
  auto kfn = sparse_attn_tc_kernel<BLK>;
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Layout<BLK>::ALLOC) != cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  const int64_t grid = prm.num_units < num_sms() ? prm.num_units : num_sms();
  kfn<<<static_cast<unsigned>(grid), kThreads, Layout<BLK>::ALLOC, st>>>(mq, mk, mv, prm);
  return launch_status();
}

static bool tc_eligible(const ropeslr_shape* s) {
  return s->dtype == ROPESLR_BF16 && s->d == D && (s->block == 64 || s->block == 128);
}

}  // namespace tc

static int device_is_sm100() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0;
}

static int check_attn_args(const ropeslr_shape* s, const void* q, const void* k, const void* v, const int32_t* idx,
                           int kmax, const int32_t* cnt) {
  if (!s) return ROPESLR_ERR_NULL;
  if (s->B < 1 || s->H < 1 || s->L < 1 || s->block < 1 || s->block > 128) return ROPESLR_ERR_SHAPE;
  if (s->dtype != ROPESLR_F32 && s->dtype != ROPESLR_BF16) return ROPESLR_ERR_DTYPE;
  if (!q || !k || !v || !idx || !cnt) return ROPESLR_ERR_NULL;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v)) return ROPESLR_ERR_ALIGN;
  if (kmax < 1) return ROPESLR_ERR_SHAPE;
  if (!device_is_sm100()) return ROPESLR_ERR_ARCH;
  return ROPESLR_OK;
}

static int resolve_impl(const ropeslr_shape* s, int impl) {
  if (impl == ROPESLR_IMPL_AUTO) return tc::tc_eligible(s) ? ROPESLR_IMPL_TCGEN05 : ROPESLR_IMPL_SIMT;
  if (impl == ROPESLR_IMPL_TCGEN05 && !tc::tc_eligible(s)) return -1;
  if (impl != ROPESLR_IMPL_SIMT && impl != ROPESLR_IMPL_TCGEN05) return -1;
  return impl;
}

static int launch_tc_dispatch(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                              const tc::Params& prm, cudaStream_t st) {
  return s->block == 128 ? tc::launch_tc<128>(s, q, k, v, prm, st) : tc::launch_tc<64>(s, q, k, v, prm, st);
}

static tc::Params base_params(const ropeslr_shape* s, const int32_t* idx, int kmax, const int32_t* cnt,
                              const int32_t* perm) {
  tc::Params prm{};
  prm.idx = idx;
  prm.cnt = cnt;
  prm.kmax = kmax;
  prm.nb = static_cast<int>(ceil_div(s->L, s->block));
  prm.H = static_cast<int>(s->H);
  prm.L = s->L;
  prm.num_units = s->B * s->H * prm.nb;
  prm.perm = perm;
  prm.out_H = static_cast<int>(s->H);
  prm.out_h0 = 0;
  prm.scale_log2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(s->d)));
  const char* pol = getenv("ROPESLR_KV_EVICT_LAST");
  prm.kv_evict_last = (pol != nullptr && pol[0] == '1') ? 1 : 0;
  const char* dbg = getenv("ROPESLR_DEBUG_MODE");
  prm.debug_mode = dbg ? atoi(dbg) : 0;
  return prm;
}

}  // namespace ropeslr

using namespace ropeslr;

extern "C" int ropeslr_sparse_attention(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                                        const int32_t* idx, int32_t kmax, const int32_t* cnt, const int32_t* row_perm,
                                        float* o_sparse, int32_t impl, void* stream) {
  int st = check_attn_args(s, q, k, v, idx, kmax, cnt);
  if (st) return st;
  if (!o_sparse) return ROPESLR_ERR_NULL;
  const int which = resolve_impl(s, impl);
  if (which < 0) return ROPESLR_ERR_VALUE;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  if (which == ROPESLR_IMPL_SIMT)
    return launch_sparse_attention_simt(s, q, k, v, idx, kmax, cnt, row_perm, o_sparse, cs);
  tc::Params prm = base_params(s, idx, kmax, cnt, row_perm);
  prm.o_sparse = o_sparse;
  return launch_tc_dispatch(s, q, k, v, prm, cs);
}

extern "C" size_t ropeslr_attend_workspace_bytes(const ropeslr_shape* s, int32_t impl) {
  if (!s) return 0;
  const int which = resolve_impl(s, impl);
  if (which == ROPESLR_IMPL_SIMT) return static_cast<size_t>(s->B * s->H * s->L * s->d) * sizeof(float);
  return 0;
}

namespace ropeslr {
// K2 + K4 (tcgen05 path only) writing heads [out_h0, out_h0 + H) of
// out / y_lr rows that hold out_H heads: a head chunk of a wider forward
// (forward_host.cu).
int attend_fused_tc_strided(const ropeslr_shape* s, const void* q, const void* k, const void* v, const int32_t* idx,
                            int32_t kmax, const int32_t* cnt, const void* y_lr, const float* g_logit, float b_g,
                            const float* rms_sparse, float eps, void* out, int out_H, int out_h0,
                            cudaStream_t stream) {
  int st = check_attn_args(s, q, k, v, idx, kmax, cnt);
  if (st) return st;
  if (!tc::tc_eligible(s)) return ROPESLR_ERR_VALUE;
  if (out_h0 < 0 || out_h0 + s->H > out_H) return ROPESLR_ERR_SHAPE;
  tc::Params prm = base_params(s, idx, kmax, cnt, nullptr);
  prm.y_lr = static_cast<const __nv_bfloat16*>(y_lr);
  prm.g_logit = g_logit;
  prm.b_g = b_g;
  prm.rms_sp = rms_sparse;
  prm.eps = eps;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.out_H = out_H;
  prm.out_h0 = out_h0;
  return launch_tc_dispatch(s, q, k, v, prm, stream);
}
bool attend_tc_eligible(const ropeslr_shape* s) { return tc::tc_eligible(s); }
}  // namespace ropeslr

extern "C" int ropeslr_attend_fused(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                                    const int32_t* idx, int32_t kmax, const int32_t* cnt, const int32_t* row_perm,
                                    const void* y_lr, const float* g_logit, float b_g, const float* rms_sparse,
                                    float eps, void* out, float* o_sparse, int32_t impl, void* ws, size_t ws_bytes,
                                    void* stream) {
  int st = check_attn_args(s, q, k, v, idx, kmax, cnt);
  if (st) return st;
  if (!y_lr || !g_logit || !rms_sparse || !out) return ROPESLR_ERR_NULL;
  if (!(eps > 0.f)) return ROPESLR_ERR_VALUE;
  const int which = resolve_impl(s, impl);
  if (which < 0) return ROPESLR_ERR_VALUE;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  if (which == ROPESLR_IMPL_SIMT) {
    float* osp = o_sparse;
    if (osp == nullptr) {
      if (!ws || ws_bytes < ropeslr_attend_workspace_bytes(s, impl)) return ROPESLR_ERR_WORKSPACE;
      osp = static_cast<float*>(ws);
    }
    st = launch_sparse_attention_simt(s, q, k, v, idx, kmax, cnt, row_perm, osp, cs);
    if (st) return st;
    return ropeslr_fuse_output(s, osp, y_lr, g_logit, b_g, rms_sparse, eps, out, stream);
  }
  tc::Params prm = base_params(s, idx, kmax, cnt, row_perm);
  prm.y_lr = static_cast<const __nv_bfloat16*>(y_lr);
  prm.g_logit = g_logit;
  prm.b_g = b_g;
  prm.rms_sp = rms_sparse;
  prm.eps = eps;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.o_sparse = o_sparse;
  return launch_tc_dispatch(s, q, k, v, prm, cs);
}
