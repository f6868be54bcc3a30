// K2 + K4: block-sparse softmax attention on the 5th-generation tensor cores
// with the fused RoPeSLR epilogue (mechanism.py:321-326 and 437-451).
//
// One persistent CTA per SM walks work units (bh, query block) in head-major
// order, so the ~150 CTAs in flight read the K/V blocks of one or two heads
// and those stay resident in the 126 MB L2.  Per unit:
//
//   warp 0  TMA producer   Q tile once, then K_j and V_j for every selected
//                          key block j (contiguous [block, 128] boxes of the
//                          [B*H, L, d] tensors, 128-byte swizzle), 2-stage rings.
//   warp 1  MMA issuer     S_j = Q K_j^T into TMEM (double buffered), then
//                          O += P_{j-1} V_{j-1} into a TMEM accumulator;
//                          tcgen05.commit releases smem stages / signals.
//   warp 2  TMEM owner     alloc / dealloc of the 512 columns.
//   warps 4-7 softmax      one query row per thread: tcgen05.ld of its S row,
//                          online softmax in the exp2 domain with the lazy
//                          (threshold 8) rescale of O, bf16 P into swizzled
//                          smem for the PV MMA; at the end of the unit the
//                          epilogue: O / l, RMSNorm * rms_sparse,
//                          + sigmoid(g_logit + b_g) * y_lr, bf16 store.
//
// TMEM columns: S0 [0,128), S1 [128,256), O [256,384).
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
constexpr int kThreads = 256;

template <int BLK>
struct Layout {
  static constexpr int Q_BYTES = M * D * 2;
  static constexpr int KV_BYTES = BLK * D * 2;
  static constexpr int P_BYTES = M * BLK * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;
  static constexpr int OFF_P = OFF_V + 2 * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int NBAR = 24;
  static constexpr int BYTES = OFF_BAR + NBAR * 8 + 16;
  static constexpr int ALLOC = BYTES + 1024;  // slack for 1024-byte alignment
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
  int kv_evict_last;
};

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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint8_t* sP = smem + Lay::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Lay::OFF_BAR + Lay::NBAR * 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < Lay::NBAR; ++i) {
      uint32_t count = 1;
      if (i == S_EMPTY || i == S_EMPTY + 1 || i == P_FULL || i == P_FULL + 1 || i == O_EMPTY) count = 128;
      mbar_init(&bars[i], count);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  if (BLK < M && warp >= 4) {
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

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      const uint64_t pol_kv = p.kv_evict_last ? policy_evict_last() : policy_evict_normal();
      const uint64_t pol_q = policy_evict_first();
      uint32_t g = 0, uc = 0;
      for (int64_t u = blockIdx.x; u < p.num_units; u += gridDim.x, ++uc) {
        const int bh = static_cast<int>(u / p.nb);
        const int qb = static_cast<int>(u % p.nb);
        const int n = p.cnt[u];
        const int32_t* irow = p.idx + u * p.kmax;
        mbar_wait(&bars[Q_EMPTY], (uc & 1) ^ 1);
        mbar_arrive_expect_tx(&bars[Q_FULL], 2 * BLK * 128);
        tma_load_3d_hint(sQ, &tmQ, &bars[Q_FULL], 0, qb * BLK, bh, pol_q);
        tma_load_3d_hint(sQ + M * 128, &tmQ, &bars[Q_FULL], 64, qb * BLK, bh, pol_q);
        for (int j = 0; j < n; ++j, ++g) {
          const int kb = irow[j];
          const int s = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          uint8_t* dk = sK + s * Lay::KV_BYTES;
          uint8_t* dv = sV + s * Lay::KV_BYTES;
          mbar_wait(&bars[K_EMPTY + s], ph ^ 1);
          mbar_arrive_expect_tx(&bars[K_FULL + s], Lay::KV_BYTES);
          tma_load_3d_hint(dk, &tmK, &bars[K_FULL + s], 0, kb * BLK, bh, pol_kv);
          tma_load_3d_hint(dk + BLK * 128, &tmK, &bars[K_FULL + s], 64, kb * BLK, bh, pol_kv);
          mbar_wait(&bars[V_EMPTY + s], ph ^ 1);
          mbar_arrive_expect_tx(&bars[V_FULL + s], Lay::KV_BYTES);
          tma_load_3d_hint(dv, &tmV, &bars[V_FULL + s], 0, kb * BLK, bh, pol_kv);
          tma_load_3d_hint(dv + BLK * 128, &tmV, &bars[V_FULL + s], 64, kb * BLK, bh, pol_kv);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_qk = idesc_bf16_f32(M, BLK, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(M, D, false, true);
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV), aP = smem_u32(sP);
      const uint32_t tO = tmem + 256;
      uint32_t g = 0, uc = 0;
      for (int64_t u = blockIdx.x; u < p.num_units; u += gridDim.x, ++uc) {
        const int n = p.cnt[u];
        mbar_wait(&bars[Q_FULL], uc & 1);
        tc_fence_after();
        for (int j = 0; j <= n; ++j) {
          if (j < n) {
            const uint32_t gg = g + j;
            const int s = gg & 1;
            const uint32_t ph = (gg >> 1) & 1;
            mbar_wait(&bars[K_FULL + s], ph);
            mbar_wait(&bars[S_EMPTY + s], ph ^ 1);
            tc_fence_after();
            const uint32_t tS = tmem + s * 128;
            const uint32_t kbase = aK + s * Lay::KV_BYTES;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint64_t da = desc_sw128(aQ + (kk >> 2) * (M * 128) + (kk & 3) * 32, 16, 1024);
              const uint64_t db = desc_sw128(kbase + (kk >> 2) * (BLK * 128) + (kk & 3) * 32, 16, 1024);
              mma_bf16_ss(tS, da, db, idesc_qk, kk > 0 ? 1u : 0u);
            }
            mma_commit(&bars[K_EMPTY + s]);
            mma_commit(&bars[S_FULL + s]);
            if (j == n - 1) mma_commit(&bars[Q_EMPTY]);
          }
          if (j >= 1) {
            const uint32_t gp = g + j - 1;
            const int s = gp & 1;
            const uint32_t ph = (gp >> 1) & 1;
            mbar_wait(&bars[V_FULL + s], ph);
            mbar_wait(&bars[P_FULL + s], ph);
            if (j == 1) mbar_wait(&bars[O_EMPTY], (uc & 1) ^ 1);
            tc_fence_after();
            const uint32_t pbase = aP + s * Lay::P_BYTES;
            const uint32_t vbase = aV + s * Lay::KV_BYTES;
#pragma unroll
            for (int kk = 0; kk < BLK / 16; ++kk) {
              const uint64_t da = desc_sw128(pbase + (kk >> 2) * (M * 128) + (kk & 3) * 32, 16, 1024);
              const uint64_t db = desc_sw128(vbase + kk * 2048, BLK * 128, 1024);
              mma_bf16_ss(tO, da, db, idesc_pv, (j > 1 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&bars[V_EMPTY + s]);
            mma_commit(&bars[P_EMPTY + s]);
            mma_commit(&bars[PV_DONE + s]);
          }
        }
        mma_commit(&bars[O_FULL]);
        g += n;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue
    const int row = threadIdx.x - 128;            // query row in the tile == TMEM lane
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>((warp - 4) * 32) << 16);
    uint32_t g = 0, uc = 0;
    for (int64_t u = blockIdx.x; u < p.num_units; u += gridDim.x, ++uc) {
      const int bh = static_cast<int>(u / p.nb);
      const int qb = static_cast<int>(u % p.nb);
      const int n = p.cnt[u];
      const int32_t* irow = p.idx + u * p.kmax;
      const int qrows = block_size(p.L, BLK, qb);
      float m_run = 0.f, l_run = 0.f;
      for (int j = 0; j < n; ++j) {
        const uint32_t gg = g + j;
        const int s = gg & 1;
        const uint32_t ph = (gg >> 1) & 1;
        const int kreal = block_size(p.L, BLK, irow[j]);
        mbar_wait(&bars[S_FULL + s], ph);
        tc_fence_after();
        uint32_t sr[BLK];
#pragma unroll
        for (int c = 0; c < BLK / 32; ++c) tmem_ld32(lane_addr + s * 128 + c * 32, sr + c * 32);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bars[S_EMPTY + s]);
        // raw scores; the softmax scale is folded into one FFMA2 below
        if (kreal < BLK) {
#pragma unroll
          for (int c = 0; c < BLK; ++c)
            if (c >= kreal) sr[c] = __float_as_uint(-INFINITY);
        }
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < BLK; ++c) mx = fmaxf(mx, __uint_as_float(sr[c]));
        mx *= p.scale_log2;
        if (j == 0) {
          m_run = mx;
        } else if (mx > m_run + 8.f) {
          // lazy rescale: only when the running max grows by more than 2^8
          const float alpha = ex2_approx(m_run - mx);
          const uint32_t gp = gg - 1;
          mbar_wait(&bars[PV_DONE + (gp & 1)], (gp >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(lane_addr + 256 + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(lane_addr + 256 + c * 32, o);
          }
          tmem_wait_st();
          l_run *= alpha;
          m_run = mx;
        }
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nm2 = make_float2(-m_run, -m_run);
        float2 sum2 = make_float2(0.f, 0.f);
        uint32_t pk[BLK / 2];
#pragma unroll
        for (int i = 0; i < BLK / 2; ++i) {
          const float2 x2 = __ffma2_rn(make_float2(__uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1])), sc2, nm2);
          float2 e2;
          if ((i & 3) == 3) {
            e2 = ex2_poly2(x2);  // FMA-pipe exp2 for 1/4 of the scores: offloads the MUFU
          } else {
            e2.x = ex2_approx(x2.x);
            e2.y = ex2_approx(x2.y);
          }
          sum2 = __fadd2_rn(sum2, e2);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(e2.x, e2.y);
          pk[i] = *reinterpret_cast<uint32_t*>(&h2);
        }
        const float rowsum = sum2.x + sum2.y;
        l_run += rowsum;
        mbar_wait(&bars[P_EMPTY + s], ph ^ 1);
        uint8_t* prow = sP + s * Lay::P_BYTES + row * 128;
#pragma unroll
        for (int cc = 0; cc < BLK / 8; ++cc) {
          const int half = cc >> 3, c8 = cc & 7;
          uint4 val = make_uint4(pk[cc * 4 + 0], pk[cc * 4 + 1], pk[cc * 4 + 2], pk[cc * 4 + 3]);
          *reinterpret_cast<uint4*>(prow + half * (M * 128) + ((c8 ^ (row & 7)) << 4)) = val;
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars[P_FULL + s]);
      }
      // ---------------------------------------------- fused epilogue
      mbar_wait(&bars[O_FULL], uc & 1);
      tc_fence_after();
      uint32_t ob[D];
#pragma unroll
      for (int c = 0; c < D / 32; ++c) tmem_ld32(lane_addr + 256 + c * 32, ob + c * 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars[O_EMPTY]);
      if (row < qrows) {
        const float inv_l = 1.f / l_run;
        const int64_t flat = static_cast<int64_t>(qb) * BLK + row;
        const int64_t tok = p.perm ? p.perm[flat] : flat;
        float ss = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const float o = __uint_as_float(ob[c]) * inv_l;
          ob[c] = __float_as_uint(o);
          ss = fmaf(o, o, ss);
        }
        if (p.o_sparse) {
          float* dst = p.o_sparse + (static_cast<int64_t>(bh) * p.L + tok) * D;
#pragma unroll
          for (int c = 0; c < D; c += 4)
            *reinterpret_cast<float4*>(dst + c) = make_float4(__uint_as_float(ob[c]), __uint_as_float(ob[c + 1]),
                                                              __uint_as_float(ob[c + 2]), __uint_as_float(ob[c + 3]));
        }
        if (p.out) {
          const int b = bh / p.H, h = bh % p.H;
          const float inv = 1.f / sqrtf(ss / static_cast<float>(D) + p.eps);
          const float gate = sigmoidf_stable(p.g_logit[static_cast<int64_t>(b) * p.L + tok] + p.b_g);
          const int64_t orow = ((static_cast<int64_t>(b) * p.L + tok) * p.H + h) * D;
          const __nv_bfloat16* y = p.y_lr + orow;
          __nv_bfloat16* dst = p.out + orow;
#pragma unroll
          for (int c = 0; c < D; c += 8) {
            float yv[8], ov[8];
            {
              const uint4 u = __ldcs(reinterpret_cast<const uint4*>(y + c));
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 f2 = __bfloat1622float2(h[i]);
                yv[2 * i] = f2.x;
                yv[2 * i + 1] = f2.y;
              }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
              ov[i] = fmaf(gate, yv[i], __uint_as_float(ob[c + i]) * inv * p.rms_sp[c + i]);
            uint4 u;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(ov[2 * i], ov[2 * i + 1]);
            __stcs(reinterpret_cast<uint4*>(dst + c), u);
          }
        }
      }
      g += n;
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
  prm.scale_log2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(s->d)));
  const char* pol = getenv("ROPESLR_KV_EVICT_LAST");
  prm.kv_evict_last = (pol != nullptr && pol[0] == '1') ? 1 : 0;
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
