// K2 + K4: block-sparse softmax attention on the 5th-generation tensor cores
// with the fused RoPeSLR epilogue (mechanism.py:321-326 and 437-451).
//
// Two kernels share the warp layout below: sparse_attn_tc_kernel keeps a
// running row max (online softmax, two O accumulators); the default,
// sparse_attn_fixed_kernel (further down), fixes each row's exponent
// reference per unit from one probe score and needs neither the max nor the
// rescale.  ROPESLR_K2=online selects the first.
//
// One persistent CTA per SM walks work units (bh, query block) in head-major
// order, so the ~150 CTAs in flight read the K/V blocks of one or two heads
// and those stay resident in the 126 MB L2 (at block 64 the fixed-reference
// kernel's units are pairs of adjacent query blocks over the union of their
// selections: see sparse_attn_fixed_kernel, UNI).  Per unit:
//
//   warp 0  TMA producer   Q tile once per unit, then K_j for every selected
//                          key block j (contiguous [block, 128] boxes of the
//                          [B*H, L, d] tensors, 128-byte swizzle) into a
//                          3-stage ring (4 for block 64).
//   warp 3  TMA producer   V_j, its own ring (a V slot frees only after its
//                          PV, so it must not hold back the K prefetch).
//   warp 1  MMA issuer     S_b = Q K_j^T into TMEM buffer b = j & 1 (SS-MMA),
//                          O += P_b V_j as a TS-MMA reading P from TMEM;
//                          tcgen05.commit releases smem stages and signals.
//   warp 2  TMEM owner     alloc / dealloc of the 512 columns.
//   warps 4-7, 8-11        two softmax warpgroups splitting every key block
//                          by columns: WG w owns keys [w*B/2, (w+1)*B/2) of
//                          each S tile, one query row per thread.  Row max =
//                          max of the two halves (exchanged through shared
//                          memory), exp2-domain softmax with the lazy
//                          (threshold 2^8) rescale of O, bf16 P written back
//                          over S_b.  Both warpgroups work on every tile, so
//                          a tile's softmax takes half the time it would on
//                          one warpgroup and overlaps the MMAs of the next.
//                          Epilogue: O / l, RMSNorm * rms_sparse, +
//                          sigmoid(g_logit + b_g) * y_lr, bf16 store; WG w
//                          finalises O columns [64w, 64w + 64).
//
// TMEM columns: S_0, S_1, S_2 at [0,128), [128,256), [256,384); O [384,512).
// Shared memory (block 128): Q 32K, K 3x32K, V 3x32K = 224 KiB.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

// -DROPESLR_K2_MEASURE=1 (scripts/build_variant.sh) compiles the
// measurement switches into the fixed-reference kernel; the product build
// leaves them out (their branches cost 1.6% at config 3).
#ifndef ROPESLR_K2_MEASURE
#define ROPESLR_K2_MEASURE 0
#endif

namespace ropeslr {

int launch_sparse_attention_simt(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                                 const int32_t* idx, int kmax, const int32_t* cnt, const int32_t* perm,
                                 float* o_sparse, cudaStream_t st);

namespace tc {

using namespace sm100;

constexpr int D = 128;   // head dim handled by this kernel
constexpr int M = 128;   // MMA rows (query rows per tile)
constexpr int kThreads = 640;  // 4 control warps + 4 softmax warpgroups (two pairs)
constexpr uint32_t O_COL = 256;  // TMEM columns: S_0 [0,128), S_1 [128,256), O_0 [256,384), O_1 [384,512)
// setmaxnreg moves registers inside the CTA's own pool, which holds what the
// launch allotted: 96 per thread (65536 / 640, rounded down to 8) x 640.
constexpr int kLaunchRegs = 96;
constexpr int kCtrlRegs = 56;       // per thread, control warpgroup (TMA, MMA, TMEM)
constexpr int kSoftmaxRegs = 104;   // per thread, softmax warpgroups
static_assert(kCtrlRegs * 128 + kSoftmaxRegs * 512 <= kLaunchRegs * kThreads, "register pool overcommitted");

template <int BLK>
struct Layout {
  static constexpr int Q_BYTES = M * D * 2;
  static constexpr int KV_BYTES = BLK * D * 2;
  static constexpr int KST = BLK == 128 ? 2 : 4;  // K ring depth (a K slot frees as soon as its QK^T lands)
  static constexpr int VST = BLK == 128 ? 3 : 4;  // V ring depth (a V slot frees only after its PV)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  static constexpr int OFF_XCH = OFF_V + VST * KV_BYTES;  // row-max / epilogue exchange, 4 KiB
  static constexpr int OFF_BAR = OFF_XCH + 4096;
  static constexpr int NBAR = 2 * KST + 2 * VST + 12;
  static constexpr int BYTES = OFF_BAR + NBAR * 8 + 16;
  // dynamic smem starts 1024-aligned (after the driver's 1 KiB reservation);
  // the kernel traps if that ever changes
  static constexpr int ALLOC = BYTES;
  static_assert(ALLOC <= 227 * 1024, "shared memory budget");
};

// Barrier indices.  Tile t belongs to softmax pair p = t & 1.
template <int BLK>
struct Bars {
  static constexpr int KST = Layout<BLK>::KST, VST = Layout<BLK>::VST;
  static constexpr int Q_FULL = 0, Q_EMPTY = 1;
  static constexpr int K_FULL = 2, K_EMPTY = K_FULL + KST;
  static constexpr int V_FULL = K_EMPTY + KST, V_EMPTY = V_FULL + VST;
  static constexpr int S_FULL = V_EMPTY + VST;  // +p: S_p = Q K_t^T landed
  static constexpr int P_FULL = S_FULL + 2;     // +p: both warpgroups of pair p wrote P_p
  static constexpr int O_FULL = P_FULL + 2;
  static constexpr int O_EMPTY = O_FULL + 1;
  static constexpr int COUNT = O_EMPTY + 1;
  static_assert(COUNT <= Layout<BLK>::NBAR, "barrier count");
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
  const int32_t* order;  // nullable: unit schedule (schedule_units_kernel), position -> unit
  const __nv_bfloat16* kmat;  // K itself (fixed-reference kernel: the probe key)
  // fixed-reference kernel: units whose exponent reference failed (see
  // sparse_attn_fixed_kernel) are appended to flag_list once (unit_flag
  // dedupes), and the running-max kernel recomputes them, reading its unit
  // count from num_units_dev
  int* unit_flag;
  int* flag_count;
  int32_t* flag_list;
  const int* num_units_dev;
  float scale_log2;
  const __nv_bfloat16* y_lr;
  const float* g_logit;
  float b_g;
  const float* rms_sp;
  float eps;
  __nv_bfloat16* out;
  float* out_f32;  // when set, the fused output is stored as float32 here instead of bf16 into out
  float* o_sparse;
  int out_H;   // heads per token row of out / y_lr (>= H when a head chunk writes into a wider row)
  int out_h0;  // first head of this call inside that row
  int qb0;  // query-block range of this call (nq > 0): positions map to units
  int nq;   // (bh, qb0 + pos % nq), bh = pos / nq; nq == 0: every query block
  int kv_evict_last;
  // query-block pairs (block 64, union_pairs_kernel): units are (bh, pair)
  // of 128 query rows; idx / cnt / kmax / nb describe the pairs' union key
  // lists, ubits [unit][kmax] which query block of the pair selected each
  // entry (bit 0: the first, bit 1: the second), nb_orig the query blocks
  const uint8_t* ubits;
  int nb_orig;
  int qlo, qhi;  // pairs: the query blocks [qlo, qhi) this call writes (a range may split a pair)
  int debug_mode;  // measurement only: 0 normal; 2 every K/V load reads block 0; 3 no K/V TMA;
                   // 4 no MMAs (fixed-reference kernel: only in a build with -DROPESLR_K2_MEASURE=1)
  long long* trace;  // TRACE
};

// Unit (bh * nb + qb) at schedule position pos: the longest-first order or a
// fallback list when given, else the query-block range of the call.
__device__ __forceinline__ int64_t unit_at(const Params& p, int64_t pos) {
  if (p.order != nullptr) return p.order[pos];
  if (p.nq > 0) return (pos / p.nq) * p.nb + p.qb0 + pos % p.nq;
  return pos;
}

// Fused output of one row's 32 columns [col0, col0 + 32): the normalised
// sparse branch O/l * rsqrt(mean + eps) * rms_sparse (ob holds O/l, inv the
// rsqrt) plus sigmoid(g_logit + b_g) * y_lr (mechanism.py:437-451), stored
// as bf16 into out or as float32 into out_f32.  16 columns per step: one
// 256-bit load of y_lr and one (bf16) or two (f32) 256-bit stores, a full
// sector per access.
__device__ __forceinline__ void store_fused_row(const Params& p, int64_t orow, const uint32_t (&ob)[32], float inv,
                                                float gate, int col0) {
  const __nv_bfloat16* y = p.y_lr + orow;
#pragma unroll
  for (int i = 0; i < 32; i += 16) {
    uint32_t uy[8];
    asm volatile("ld.global.cs.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(uy[0]), "=r"(uy[1]), "=r"(uy[2]), "=r"(uy[3]), "=r"(uy[4]), "=r"(uy[5]), "=r"(uy[6]),
                   "=r"(uy[7])
                 : "l"(y + i));
    float o[16];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float2 yv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uy[e]));
      o[2 * e] = fmaf(gate, yv.x, __uint_as_float(ob[i + 2 * e]) * inv * p.rms_sp[col0 + i + 2 * e]);
      o[2 * e + 1] = fmaf(gate, yv.y, __uint_as_float(ob[i + 2 * e + 1]) * inv * p.rms_sp[col0 + i + 2 * e + 1]);
    }
    if (p.out_f32 != nullptr) {
      float* dst = p.out_f32 + orow + i;
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf)
        asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 8 * hlf),
                     "r"(__float_as_uint(o[8 * hlf])), "r"(__float_as_uint(o[8 * hlf + 1])),
                     "r"(__float_as_uint(o[8 * hlf + 2])), "r"(__float_as_uint(o[8 * hlf + 3])),
                     "r"(__float_as_uint(o[8 * hlf + 4])), "r"(__float_as_uint(o[8 * hlf + 5])),
                     "r"(__float_as_uint(o[8 * hlf + 6])), "r"(__float_as_uint(o[8 * hlf + 7]))
                     : "memory");
    } else {
      uint32_t uo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
        uo[e] = *reinterpret_cast<uint32_t*>(&h2);
      }
      asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p.out + orow + i), "r"(uo[0]),
                   "r"(uo[1]), "r"(uo[2]), "r"(uo[3]), "r"(uo[4]), "r"(uo[5]), "r"(uo[6]), "r"(uo[7])
                   : "memory");
    }
  }
}

#ifdef ROPESLR_WATCHDOG
__device__ volatile unsigned long long* g_watchdog;  // host-mapped
// Debug builds: a wait that spins for more than ~2 s records (once per
// waiter) who waited on what into host-mapped memory, then keeps waiting.
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, uint64_t* bars0, int line) {
  const long long t0 = clock64();
  bool reported = false;
  while (!mbar_try_wait(bar, parity)) {
    if (!reported && clock64() - t0 > 4000000000LL) {
      reported = true;
      const unsigned long long slot = atomicAdd(const_cast<unsigned long long*>(&g_watchdog[0]), 1ull);
      if (slot < 30) {
        volatile unsigned long long* e = g_watchdog + 2 + slot * 4;
        e[0] = blockIdx.x;
        e[1] = threadIdx.x;
        e[2] = static_cast<unsigned long long>(bar - bars0) | (static_cast<unsigned long long>(parity) << 32);
        e[3] = line;
        __threadfence_system();
      }
    }
  }
}
#define mbar_wait(b, ph) mbar_wait_wd((b), (ph), bars, __LINE__)
#endif

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
  // q + (n << 23) (ptxas fuses the shift-add into one LEA)
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}

// Fraction of the exponentials computed on the FMA pipe: pairs i with
// (i % POLY_DEN) < POLY_NUM (the rest go to the MUFU).
#ifndef ROPESLR_RESCALE_THRESHOLD
#define ROPESLR_RESCALE_THRESHOLD 8.f
#endif
#ifndef ROPESLR_PREFETCH
#define ROPESLR_PREFETCH 0
#endif
#ifndef ROPESLR_POLY_NUM
#define ROPESLR_POLY_NUM 1
#endif
#ifndef ROPESLR_POLY_DEN
#define ROPESLR_POLY_DEN 4
#endif

// Softmax of one key block by one pair of warpgroups, split by key
// columns: warpgroup w of the pair owns keys [w*BLK/2, (w+1)*BLK/2), one
// query row per thread, its half row already in registers.
//
// half_max: this half's max (masked past the end of the sequence when
// RAGGED), exchanged with the partner warpgroup through shared memory; the
// pair barrier also guarantees both halves of S have been read before
// either warpgroup overwrites S with P.
template <int BLK, bool RAGGED>
__device__ __forceinline__ float half_max(uint32_t (&sr)[BLK / 2], int valid, float* xmax_mine,
                                          const float* xmax_other, int bar_id) {
  constexpr int HB = BLK / 2;
  if (RAGGED) {
#pragma unroll
    for (int c = 0; c < HB; ++c)
      if (c >= valid) sr[c] = __float_as_uint(-INFINITY);
  }
  float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int c = 0; c < HB; c += 8) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      mq[q] = fmaxf(mq[q], fmaxf(__uint_as_float(sr[c + 2 * q]), __uint_as_float(sr[c + 2 * q + 1])));
  }
  const float lmx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
  *xmax_mine = lmx;
  named_bar_sync(bar_id, 256);
  return fmaxf(lmx, *xmax_other);
}

// half_exp: P = 2^(s*scale - m) as bf16 pairs written over S (P column c
// holds keys 2c, 2c+1), 16 columns per TMEM store; returns this half's sum.
template <int BLK>
__device__ __forceinline__ float half_exp(const uint32_t (&sr)[BLK / 2], uint32_t tPh, float scale_log2,
                                          float m_run) {
  constexpr int HB = BLK / 2;
  const float2 sc2 = make_float2(scale_log2, scale_log2);
  const float2 nm2 = make_float2(-m_run, -m_run);
  float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int h = 0; h < HB / 32; ++h) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 x2 = __ffma2_rn(
          make_float2(__uint_as_float(sr[h * 32 + 2 * i]), __uint_as_float(sr[h * 32 + 2 * i + 1])), sc2, nm2);
      float2 e2;
      if ((i % ROPESLR_POLY_DEN) < ROPESLR_POLY_NUM) {
        e2 = ex2_poly2(x2);  // FMA-pipe exp2 for a fraction of the scores: offloads the MUFU
      } else {
        e2.x = ex2_approx(x2.x);
        e2.y = ex2_approx(x2.y);
      }
      sum2 = __fadd2_rn(sum2, e2);
      __nv_bfloat162 hb = __floats2bfloat162_rn(e2.x, e2.y);
      pk[i] = *reinterpret_cast<uint32_t*>(&hb);
    }
    tmem_st16(tPh + h * 16, pk);
  }
  return sum2.x + sum2.y;
}

template <int BLK>
__global__ void __launch_bounds__(kThreads, 1)
    sparse_attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ Params p) {
  using Lay = Layout<BLK>;
  using Bx = Bars<BLK>;
  constexpr int KST = Lay::KST, VST = Lay::VST;
  constexpr int HB = BLK / 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Lay::OFF_BAR + Lay::NBAR * 8);
  float* xch = reinterpret_cast<float*>(smem + Lay::OFF_XCH);  // 1024 floats

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < Bx::COUNT; ++i) {
      uint32_t count = 1;
      if (i == Bx::P_FULL || i == Bx::P_FULL + 1) count = 256;
      if (i == Bx::O_EMPTY) count = 512;
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
  const int64_t nunits = p.num_units_dev ? static_cast<int64_t>(*p.num_units_dev) : p.num_units;

  if (warp < 4) {
    setmaxnreg_dec<kCtrlRegs>();
    if (warp == 0 || warp == 3) {
      if (elect_one_sync()) {
        // ------------------------------------------- TMA producers
        // warp 0: Q and K; warp 3: V (a V slot frees only after its PV, so
        // it must not hold back the K prefetch).
        const bool is_k = (warp == 0);
        const int st = is_k ? KST : VST;
        const uint64_t pol_kv = p.kv_evict_last ? policy_evict_last() : policy_evict_normal();
        const uint64_t pol_q = policy_evict_first();
        const CUtensorMap* map = is_k ? &tmK : &tmV;
        uint8_t* ring = is_k ? sK : sV;
        const int full = is_k ? Bx::K_FULL : Bx::V_FULL;
        const int empty = is_k ? Bx::K_EMPTY : Bx::V_EMPTY;
        uint32_t g = 0, uc = 0;
        for (int64_t pos = blockIdx.x; pos < nunits; pos += gridDim.x, ++uc) {
          const int64_t u = unit_at(p, pos);
          const int bh = static_cast<int>(u / p.nb);
          const int n = p.cnt[u];
          const int32_t* irow = p.idx + u * p.kmax;
          if (is_k) {
            const int qb = static_cast<int>(u % p.nb);
            mbar_wait(&bars[Bx::Q_EMPTY], (uc & 1) ^ 1);
            mbar_arrive_expect_tx(&bars[Bx::Q_FULL], 2 * BLK * 128);
            tma_load_3d_hint(sQ, &tmQ, &bars[Bx::Q_FULL], 0, qb * BLK, bh, pol_q);
            tma_load_3d_hint(sQ + M * 128, &tmQ, &bars[Bx::Q_FULL], 64, qb * BLK, bh, pol_q);
          }
          for (int j = 0; j < n; ++j, ++g) {
            const int kb = p.debug_mode == 2 ? 0 : irow[j];
            const int s = g % st;
            const uint32_t ph = (g / st) & 1;
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
      // Global tile t belongs to softmax pair p = t & 1: S_p = Q K_t^T
      // (SS-MMA into TMEM columns [128p, +BLK)); the pair overwrites S_p with
      // P_p (bf16 pairs, columns [128p, +BLK/2)); O_p += P_p V_t (TS-MMA, A
      // from TMEM, O_p at columns [256 + 128p, +128)).  Issue order per unit:
      // QK(0), QK(1), then [PV(j-2), QK(j)], then PV(n-2), PV(n-1): QK(j)
      // overwrites what PV(j-2) reads, the tensor pipe executes a CTA's MMAs
      // in issue order, and S_FULL's commit after QK(j) also covers PV(j-2),
      // so a pair may rescale O_p as soon as it sees S_p.
      constexpr uint32_t idesc_qk = idesc_bf16_f32(M, BLK, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(M, D, false, true);
      const uint64_t dQ = desc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dK0 = desc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dV0 = desc_sw128(smem_u32(sV), BLK * 128, 1024);
      const bool leader = elect_one_sync();
      uint32_t g = 0, uc = 0;
      for (int64_t pos = blockIdx.x; pos < nunits; pos += gridDim.x, ++uc) {
        const int64_t u = unit_at(p, pos);
        const int n = p.cnt[u];
        mbar_wait(&bars[Bx::Q_FULL], uc & 1);
        tc_fence_after();
        for (int j = 0; j < n + 2; ++j) {
          if (j >= 2) {
            const uint32_t t = g + j - 2;
            const int s = t % VST;
            const int pr = t & 1;
            mbar_wait(&bars[Bx::V_FULL + s], (t / VST) & 1);
            mbar_wait(&bars[Bx::P_FULL + pr], (t >> 1) & 1);
            if (j == 2) mbar_wait(&bars[Bx::O_EMPTY], (uc & 1) ^ 1);
            tc_fence_after();
            if (leader) {
              const uint64_t dV = dV0 + static_cast<uint64_t>((s * Lay::KV_BYTES) >> 4);
#pragma unroll
              for (int kk = 0; kk < BLK / 16; ++kk) {
                const uint64_t db = dV + static_cast<uint64_t>((kk * 2048) >> 4);
                mma_bf16_ts(tmem + O_COL + pr * 128, tmem + pr * 128 + kk * 8, db, idesc_pv,
                            (j >= 4 || kk > 0) ? 1u : 0u);
              }
              mma_commit(&bars[Bx::V_EMPTY + s]);
            }
            __syncwarp();
          }
          if (j < n) {
            const uint32_t t = g + j;
            const int s = t % KST;
            const int pr = t & 1;
            mbar_wait(&bars[Bx::K_FULL + s], (t / KST) & 1);
            tc_fence_after();
            if (leader) {
              const uint64_t dK = dK0 + static_cast<uint64_t>((s * Lay::KV_BYTES) >> 4);
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint64_t da = dQ + static_cast<uint64_t>(((kk >> 2) * (M * 128) + (kk & 3) * 32) >> 4);
                const uint64_t db = dK + static_cast<uint64_t>(((kk >> 2) * (BLK * 128) + (kk & 3) * 32) >> 4);
                mma_bf16_ss(tmem + pr * 128, da, db, idesc_qk, kk > 0 ? 1u : 0u);
              }
              mma_commit(&bars[Bx::K_EMPTY + s]);
              mma_commit(&bars[Bx::S_FULL + pr]);
              if (j == n - 1) mma_commit(&bars[Bx::Q_EMPTY]);
            }
            __syncwarp();
          }
        }
        if (leader) mma_commit(&bars[Bx::O_FULL]);
        __syncwarp();
        g += n;
      }
    }
  } else {
    setmaxnreg_inc<kSoftmaxRegs>();
    // ------------------------------------ softmax warpgroups + epilogue
    const int q = (warp - 4) >> 2;                 // softmax warpgroup 0..3
    const int pr = q >> 1;                         // pair: tiles t with t & 1 == pr
    const int w = q & 1;                           // key-column half within the pair
    const int row = (threadIdx.x - 128) & 127;     // query row == TMEM lane
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t tS = lane_addr + pr * 128;
    const uint32_t tOh = lane_addr + O_COL + pr * 128 + w * (D / 2);
    // rows >= BLK of the 128-row MMA tile are padding (block 64)
    const bool rows_live = BLK >= M || (warp & 3) * 32 < BLK;
    uint32_t g = 0, uc = 0;
    for (int64_t pos = blockIdx.x; pos < nunits; pos += gridDim.x, ++uc) {
      const int64_t u = unit_at(p, pos);
      const int bh = static_cast<int>(u / p.nb);
      const int qb = static_cast<int>(u % p.nb);
      const int n = p.cnt[u];
      const int32_t* irow = p.idx + u * p.kmax;
      const int qrows = block_size(p.L, BLK, qb);
      float m_run = -INFINITY, l_run = 0.f;
      // this pair's tiles of the unit: j = j0, j0 + 2, ...
      const int j0 = (pr - static_cast<int>(g & 1)) & 1;
      for (int j = j0; j < n; j += 2) {
        const uint32_t t = g + j;
        const int kreal = block_size(p.L, BLK, irow[j]);
        mbar_wait(&bars[Bx::S_FULL + pr], (t >> 1) & 1);
        tc_fence_after();
        const bool trc = ROPESLR_K2_MEASURE && p.trace && blockIdx.x == 0 && row == 0 && t < 64;
        if (trc) p.trace[(w * 64 + t) * 4 + 0] = clock64();
        float* xm = xch + (pr * 2 + ((t >> 1) & 1)) * 256;  // [pair][tile parity][wg][row]
        if (!rows_live) {
          // block 64: TMEM lanes 64-127 hold the zero query rows of the MMA
          // tile; their warps only keep the pair barrier and P_FULL counts
          named_bar_sync(1 + pr, 256);
          tc_fence_before();
          mbar_arrive(&bars[Bx::P_FULL + pr]);
          continue;
        }
        uint32_t sr[HB];
#pragma unroll
        for (int c = 0; c < HB / 32; ++c) tmem_ld32(tS + w * HB + c * 32, sr + c * 32);
        tmem_wait_ld();
        const int valid = kreal - w * HB;
        float mx = valid < HB ? half_max<BLK, true>(sr, valid, xm + w * 128 + row, xm + (w ^ 1) * 128 + row, 1 + pr)
                              : half_max<BLK, false>(sr, HB, xm + w * 128 + row, xm + (w ^ 1) * 128 + row, 1 + pr);
        mx *= p.scale_log2;
        // lazy rescale: the running max moves only when it grows by more
        // than 2^8 (both warpgroups of the pair take the same decision)
        float alpha = 1.f;
        if (j == j0) {
          m_run = mx;
        } else if (mx > m_run + ROPESLR_RESCALE_THRESHOLD) {
          alpha = ex2_approx(m_run - mx);
          l_run *= alpha;
          m_run = mx;
        }
        l_run += half_exp<BLK>(sr, tS + w * (HB / 2), p.scale_log2, m_run);
        // tcgen05.ld / st are warp-collective: the rescale runs for the whole
        // warp when any of its rows needs it (alpha == 1 for the others).
        // PV(t-2), the last writer of O_p, completed before S_p landed.
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < D / 64; ++c) {
            uint32_t o[32];
            tmem_ld32(tOh + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tOh + c * 32, o);
          }
        }
        if (trc) p.trace[(w * 64 + t) * 4 + 1] = clock64();
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars[Bx::P_FULL + pr]);
        if (trc) p.trace[(w * 64 + t) * 4 + 2] = clock64();
      }
      g += n;
      // ---------------------------------------------- fused epilogue
      // merge the two pairs' partial softmaxes: O = sum_p O_p 2^(m_p - m) / l;
      // warpgroup q finalises output columns [32q, 32q + 32) of its row
      mbar_wait(&bars[Bx::O_FULL], uc & 1);
      tc_fence_after();
      named_bar_sync(3, 512);  // every pair's last max exchange has been read
      float2* xml = reinterpret_cast<float2*>(xch);  // [4 wg][128] (m, l_half)
      xml[q * 128 + row] = make_float2(m_run, l_run);
      named_bar_sync(3, 512);
      const float2 a0 = xml[0 * 128 + row], a1 = xml[1 * 128 + row];
      const float2 b0 = xml[2 * 128 + row], b1 = xml[3 * 128 + row];
      const float mA = a0.x, lA = a0.y + a1.y, mB = b0.x, lB = b0.y + b1.y;
      const float mm = fmaxf(mA, mB);
      const float fA = mA == -INFINITY ? 0.f : ex2_approx(mA - mm);
      const float fB = mB == -INFINITY ? 0.f : ex2_approx(mB - mm);
      const float inv_l = 1.f / (lA * fA + lB * fB);
      const float sA = fA * inv_l, sB = fB * inv_l;
      uint32_t ob[32];
      {
        uint32_t tb[32];
        tmem_ld32(lane_addr + O_COL + q * 32, ob);
        tmem_ld32(lane_addr + O_COL + 128 + q * 32, tb);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          // an O_p with no tile in this unit holds stale data: weight 0, and
          // never multiply it (it could be inf / NaN)
          const float oa = sA != 0.f ? __uint_as_float(ob[i]) * sA : 0.f;
          const float obb = sB != 0.f ? __uint_as_float(tb[i]) * sB : 0.f;
          ob[i] = __float_as_uint(oa + obb);
        }
      }
      tc_fence_before();
      mbar_arrive(&bars[Bx::O_EMPTY]);
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) ss = fmaf(__uint_as_float(ob[i]), __uint_as_float(ob[i]), ss);
      named_bar_sync(3, 512);  // the (m, l) exchange has been read
      xch[q * 128 + row] = ss;
      named_bar_sync(3, 512);
      ss = (xch[row] + xch[128 + row]) + (xch[256 + row] + xch[384 + row]);
      named_bar_sync(3, 512);  // the exchange area is free for the next unit
      const bool live = row < qrows;
      if (!live) continue;
      const int64_t flat = static_cast<int64_t>(qb) * BLK + row;
      const int64_t tok = p.perm ? p.perm[flat] : flat;
      const int b = bh / p.H, h = bh % p.H;
      const float inv = 1.f / sqrtf(ss / static_cast<float>(D) + p.eps);
      const int col0 = q * 32;
      if (p.o_sparse) {
        float* dst = p.o_sparse + (static_cast<int64_t>(bh) * p.L + tok) * D + col0;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + i) = make_float4(__uint_as_float(ob[i]), __uint_as_float(ob[i + 1]),
                                                            __uint_as_float(ob[i + 2]), __uint_as_float(ob[i + 3]));
      }
      if (p.out || p.out_f32) {
        const float gate = sigmoidf_stable(p.g_logit[static_cast<int64_t>(b) * p.L + tok] + p.b_g);
        const int64_t orow = ((static_cast<int64_t>(b) * p.L + tok) * p.out_H + p.out_h0 + h) * D + col0;
        store_fused_row(p, orow, ob, inv, gate, col0);
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

// ---------------------------------------------------------------------------
// K2 + K4, fixed-reference variant.  Same warp roles, rings and alternating
// softmax pairs as sparse_attn_tc_kernel, but every query row uses ONE
// exponent reference m for the whole unit instead of a running max:
//
//   m_i = s_i0 + 64          (log2 domain)
//
// with s_i0 the scaled score of a probe key, the first key of the unit's
// first selected block.  Softmax is shift-invariant, so O / l is the same
// quantity as with the running max; only the range of P = 2^(s - m) moves:
// the row max lies at or above s_i0, so the largest P is at least 2^-64 (P
// of keys more than 62 binary orders below the row max flush to zero,
// weights < 2^-62 of the max key's that fp32 / bf16 could not resolve in the
// output anyway), and P stays finite while the row max is within ~160 binary
// orders (110 nats) of s_i0.  The epilogue checks every row's l against
// [2^-100, 2^110]; a unit outside goes to the running-max kernel, which
// recomputes the flagged units in the same stream (see launch_fixed).
// Without a running max there is no per-tile row max, no max exchange
// between the two warpgroups of a pair and no O rescale, hence one O
// accumulator shared by both pairs; each warpgroup works on its key half of
// a tile with no synchronisation with its partner: it writes its P half over
// the first half of its own S columns, and the PV MMA reads A from those two
// column ranges.  The freed TMEM holds Q (QK^T becomes a TS-MMA).
//
// TMEM columns: S_0 [0,128), S_1 [128,256), O [256,384), Q_0/Q_1 [384,512).
namespace fx {
constexpr uint32_t O_COL = 256;
constexpr uint32_t Q_COL = 384;  // Q_0 [384, 448), Q_1 [448, 512): the A operand of QK^T, per unit parity
template <int BLK>
struct FBars : Bars<BLK> {
  static constexpr int QT_FULL = Bars<BLK>::COUNT;  // this unit's Q is in TMEM (16 softmax warps)
  static constexpr int COUNT = QT_FULL + 1;
};
template <int BLK>
struct Layout {
  using Base = tc::Layout<BLK>;
  static constexpr int Q_BYTES = Base::Q_BYTES, KV_BYTES = Base::KV_BYTES;
  static constexpr int KST = Base::KST, VST = Base::VST;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  // [2 unit parity][4 wg][128 rows] float2 (spare, probe partial) 8 KiB,
  // then l partials [4][128] 2 KiB, then RMS partials [4][128] 2 KiB
  static constexpr int OFF_XQ = OFF_V + VST * KV_BYTES;
  static constexpr int OFF_XL = OFF_XQ + 8192;
  static constexpr int OFF_XS = OFF_XL + 2048;
  static constexpr int OFF_BAR = OFF_XS + 2048;
  static constexpr int NBAR = 2 * KST + 2 * VST + 12;
  static constexpr int BYTES = OFF_BAR + NBAR * 8 + 16;
  static constexpr int ALLOC = BYTES;
  static_assert(ALLOC <= 227 * 1024, "shared memory budget");
};
}  // namespace fx

// BLK = keys per tile (the S tile width); KB = block size (query rows of a
// unit, keys of a selected block).  KB == BLK: one selected block per tile.
// KB = 64 with BLK = 128 ("paired" block 64): a tile is two consecutive
// selected blocks stacked in one 128-row K / V slot (the second masked out
// when the count is odd), so block 64 runs the 128-key pipeline with half
// the per-tile barrier round trips.
// UNI (block 64 only): a unit is a pair of adjacent query blocks, 128 rows
// filling the MMA, over the union of their selected key blocks; each row
// masks the entries its own query block did not select (ubits), so every
// row attends exactly its own selection.  Adjacent query blocks of real
// attention share most of their selections (90-95% in the config-4 DiT's
// layers), so a unit streams about half the K / V tiles of the two
// 64-row units it replaces.
template <int BLK, int KB, bool UNI = false>
__global__ void __launch_bounds__(kThreads, 1)
    sparse_attn_fixed_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                             const __grid_constant__ CUtensorMap tmV, const __grid_constant__ Params p) {
  using Lay = fx::Layout<BLK>;
  using Bx = fx::FBars<BLK>;
  static_assert(Bx::COUNT <= Lay::NBAR, "barrier count");
  static_assert(KB == BLK || (KB == 64 && BLK == 128), "tile shapes");
  constexpr int KST = Lay::KST, VST = Lay::VST;
  constexpr int HB = BLK / 2;   // keys per warpgroup of a pair
  constexpr int KK = BLK / 16;  // K steps of the PV MMA
  constexpr int TPB = BLK / KB;  // selected blocks per tile
  constexpr int QR = UNI ? M : KB;  // query rows of a unit
  static_assert(!UNI || (KB == 64 && BLK == 128), "query-block pairs: paired block 64 only");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Lay::OFF_BAR + Lay::NBAR * 8);
  float2* xq = reinterpret_cast<float2*>(smem + Lay::OFF_XQ);
  float* xl = reinterpret_cast<float*>(smem + Lay::OFF_XL);
  float* xs = reinterpret_cast<float*>(smem + Lay::OFF_XS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < Bx::COUNT; ++i) {
      uint32_t count = 1;
      if (i == Bx::P_FULL || i == Bx::P_FULL + 1) count = 8;  // one arrival per warp of the pair
      if (i == Bx::O_EMPTY) count = 512;
      if (i == Bx::Q_EMPTY || i == Bx::QT_FULL) count = 16;  // every softmax warp: Q read / stored to TMEM
      mbar_init(&bars[i], count);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  if (KB < M && !UNI && warp >= 4 && warp < 8) {
    const int t = threadIdx.x - 128;
    for (int half = 0; half < 2; ++half) {
      uint4* z = reinterpret_cast<uint4*>(sQ + half * (M * 128) + KB * 128);
      for (int i = t; i < (M - KB) * 128 / 16; i += 128) z[i] = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp < 4) {
    setmaxnreg_dec<kCtrlRegs>();
    if (warp == 0 || warp == 3) {
      if (elect_one_sync()) {
        // ------------------------------------------- TMA producers (as v7)
        const bool is_k = (warp == 0);
        const int st = is_k ? KST : VST;
        const uint64_t pol_kv = p.kv_evict_last ? policy_evict_last() : policy_evict_normal();
        const uint64_t pol_q = policy_evict_first();
        const CUtensorMap* map = is_k ? &tmK : &tmV;
        uint8_t* ring = is_k ? sK : sV;
        const int full = is_k ? Bx::K_FULL : Bx::V_FULL;
        const int empty = is_k ? Bx::K_EMPTY : Bx::V_EMPTY;
        uint32_t g = 0, uc = 0;
        for (int64_t pos = blockIdx.x; pos < p.num_units; pos += gridDim.x, ++uc) {
          const int64_t u = unit_at(p, pos);
          const int bh = static_cast<int>(u / p.nb);
          const int n = p.cnt[u];
          const int nt = (n + TPB - 1) / TPB;
          const int32_t* irow = p.idx + u * p.kmax;
          if (is_k) {
            const int qb = static_cast<int>(u % p.nb);
            mbar_wait(&bars[Bx::Q_EMPTY], (uc & 1) ^ 1);
            mbar_arrive_expect_tx(&bars[Bx::Q_FULL], 2 * QR * 128);
            tma_load_3d_hint(sQ, &tmQ, &bars[Bx::Q_FULL], 0, qb * QR, bh, pol_q);
            tma_load_3d_hint(sQ + M * 128, &tmQ, &bars[Bx::Q_FULL], 64, qb * QR, bh, pol_q);
          }
          for (int j = 0; j < nt; ++j, ++g) {
            const int s = g % st;
            const uint32_t ph = (g / st) & 1;
            uint8_t* dst = ring + s * Lay::KV_BYTES;
            mbar_wait(&bars[empty + s], ph ^ 1);
#if ROPESLR_K2_MEASURE
            if (p.debug_mode == 3) {  // measurement build only: no K/V bytes at all
              mbar_arrive(&bars[full + s]);
              continue;
            }
#endif
            mbar_arrive_expect_tx(&bars[full + s], Lay::KV_BYTES);
#pragma unroll
            for (int b = 0; b < TPB; ++b) {
              // an odd count's missing partner block: reload the first one
              // (its columns are masked) so the byte count stays fixed
#if ROPESLR_K2_MEASURE
              const int kb = p.debug_mode == 2 ? 0 : irow[TPB * j + b < n ? TPB * j + b : TPB * j];
#else
              const int kb = irow[TPB * j + b < n ? TPB * j + b : TPB * j];
#endif
              tma_load_3d_hint(dst + b * KB * 128, map, &bars[full + s], 0, kb * KB, bh, pol_kv);
              tma_load_3d_hint(dst + BLK * 128 + b * KB * 128, map, &bars[full + s], 64, kb * KB, bh, pol_kv);
            }
          }
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------ MMA issuer
      // As v7 (QK(0), QK(1), then [PV(j-2), QK(j)]), with one O: PV(t)
      // accumulates into O whatever the pair; its A operand is the pair's
      // two P halves, at columns [128p, +BLK/4) and [128p + BLK/2, +BLK/4).
      constexpr uint32_t idesc_qk = idesc_bf16_f32(M, BLK, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(M, D, false, true);
      const uint64_t dK0 = desc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dV0 = desc_sw128(smem_u32(sV), BLK * 128, 1024);
      const bool leader = elect_one_sync();
      uint32_t g = 0, uc = 0;
      for (int64_t pos = blockIdx.x; pos < p.num_units; pos += gridDim.x, ++uc) {
        const int64_t u = unit_at(p, pos);
        const int n = (p.cnt[u] + TPB - 1) / TPB;  // tiles
        const uint32_t tQ = tmem + fx::Q_COL + (uc & 1) * (D / 2);
        mbar_wait(&bars[Bx::QT_FULL], uc & 1);
        tc_fence_after();
        for (int j = 0; j < n + 2; ++j) {
          if (j >= 2) {
            const uint32_t t = g + j - 2;
            const int s = t % VST;
            const int pr = t & 1;
            mbar_wait(&bars[Bx::V_FULL + s], (t / VST) & 1);
            mbar_wait(&bars[Bx::P_FULL + pr], (t >> 1) & 1);
            if (j == 2) mbar_wait(&bars[Bx::O_EMPTY], (uc & 1) ^ 1);
            tc_fence_after();
            if (leader) {
              const uint64_t dV = dV0 + static_cast<uint64_t>((s * Lay::KV_BYTES) >> 4);
              if (!ROPESLR_K2_MEASURE || p.debug_mode != 4) {  // mode 4 (measurement build): no MMAs
#pragma unroll
                for (int kk = 0; kk < KK; ++kk) {
                  const uint64_t db = dV + static_cast<uint64_t>((kk * 2048) >> 4);
                  const uint32_t a = tmem + pr * 128 + (kk / (KK / 2)) * HB + (kk % (KK / 2)) * 8;
                  mma_bf16_ts(tmem + fx::O_COL, a, db, idesc_pv, (j > 2 || kk > 0) ? 1u : 0u);
                }
              }
              mma_commit(&bars[Bx::V_EMPTY + s]);
            }
            __syncwarp();
          }
          if (j < n) {
            const uint32_t t = g + j;
            const int s = t % KST;
            const int pr = t & 1;
            mbar_wait(&bars[Bx::K_FULL + s], (t / KST) & 1);
            tc_fence_after();
            if (leader) {
              const uint64_t dK = dK0 + static_cast<uint64_t>((s * Lay::KV_BYTES) >> 4);
              if (!ROPESLR_K2_MEASURE || p.debug_mode != 4) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                  // A = Q from TMEM (TS-MMA): only K is read from shared memory
                  const uint64_t db = dK + static_cast<uint64_t>(((kk >> 2) * (BLK * 128) + (kk & 3) * 32) >> 4);
                  mma_bf16_ts(tmem + pr * 128, tQ + kk * 8, db, idesc_qk, kk > 0 ? 1u : 0u);
                }
              }
              mma_commit(&bars[Bx::K_EMPTY + s]);
              mma_commit(&bars[Bx::S_FULL + pr]);
            }
            __syncwarp();
          }
        }
        if (leader) mma_commit(&bars[Bx::O_FULL]);
        __syncwarp();
        g += n;
      }
    }
  } else {
    setmaxnreg_inc<kSoftmaxRegs>();
    // ------------------------------------ softmax warpgroups + epilogue
    const int q = (warp - 4) >> 2;                 // softmax warpgroup 0..3
    const int pr = q >> 1;                         // pair: tiles t with t & 1 == pr
    const int w = q & 1;                           // key half within the pair
    const int row = (threadIdx.x - 128) & 127;     // query row == TMEM lane
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t tS = lane_addr + pr * 128 + w * HB;  // this warpgroup's S columns; its P over their first half
    const uint32_t tOq = lane_addr + fx::O_COL + q * (D / 4);
    const bool rows_live = UNI || KB >= M || (warp & 3) * 32 < KB;
    // this thread's quarter of its Q row in the 128B-swizzled tile: d in
    // [32q, 32q + 32) = 16-byte chunks 4(q&1) .. 4(q&1)+3 of half q>>1
    const uint8_t* qrow = sQ + (q >> 1) * (M * 128) + row * 128;
    // prep(unit at position pos, parity uc): wait for its Q tile, store this
    // thread's quarter of its Q row into TMEM buffer uc & 1 (the A operand of
    // QK^T: column c holds d = 2c, 2c+1), publish its part of the probe dot
    // product, free the shared-memory tile
    auto prep = [&](int64_t pos, uint32_t uc) {
      const int64_t u = unit_at(p, pos);
      const int bh = static_cast<int>(u / p.nb);
      const int32_t* irow = p.idx + u * p.kmax;
      mbar_wait(&bars[Bx::Q_FULL], uc & 1);
      const __nv_bfloat16* krow =
          p.kmat + (static_cast<int64_t>(bh) * p.L + static_cast<int64_t>(irow[0]) * KB) * D + q * 32;
      float dot = 0.f;
      uint32_t qw[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int chunk = ((q & 1) * 4 + c) ^ (row & 7);
        const uint4 qv = *reinterpret_cast<const uint4*>(qrow + chunk * 16);
        const uint4 kv = __ldg(reinterpret_cast<const uint4*>(krow + c * 8));
        qw[4 * c] = qv.x;
        qw[4 * c + 1] = qv.y;
        qw[4 * c + 2] = qv.z;
        qw[4 * c + 3] = qv.w;
        const __nv_bfloat162* qh = reinterpret_cast<const __nv_bfloat162*>(&qv);
        const __nv_bfloat162* kh = reinterpret_cast<const __nv_bfloat162*>(&kv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 a = __bfloat1622float2(qh[e]), b = __bfloat1622float2(kh[e]);
          dot = fmaf(a.x, b.x, fmaf(a.y, b.y, dot));
        }
      }
      tmem_st16(lane_addr + fx::Q_COL + (uc & 1) * (D / 2) + q * 16, qw);
      xq[((uc & 1) * 4 + q) * 128 + row] = make_float2(0.f, dot);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bars[Bx::QT_FULL]);
        mbar_arrive(&bars[Bx::Q_EMPTY]);
      }
    };
    uint32_t g = 0, uc = 0;
    if (blockIdx.x < p.num_units) prep(blockIdx.x, 0);
    for (int64_t pos = blockIdx.x; pos < p.num_units; pos += gridDim.x, ++uc) {
      const int64_t u = unit_at(p, pos);
      const int bh = static_cast<int>(u / p.nb);
      const int qb = static_cast<int>(u % p.nb);
      const int nblk = p.cnt[u];
      const int n = (nblk + TPB - 1) / TPB;  // tiles
      const int32_t* irow = p.idx + u * p.kmax;
      const int qrows = block_size(p.L, QR, qb);
      // ---- the unit's exponent reference m (see the header)
      named_bar_sync(2, 512);
      float m_ref;
      {
        const float2* xr = xq + (uc & 1) * 512 + row;
        const float2 a0 = xr[0], a1 = xr[128], a2 = xr[256], a3 = xr[384];
        m_ref = ((a0.y + a1.y) + (a2.y + a3.y)) * p.scale_log2 + 64.f;
      }
      float l_run = 0.f;
      // pairs: this warp's selection bits for the entries its warpgroup
      // takes (w, w + 2, ...), the first 64 of them in two registers
      uint32_t sel_lo = 0xffffffffu, sel_hi = 0xffffffffu;
      if (UNI) {
        const int half = row >> 6;
        const uint8_t* ub = p.ubits + u * p.kmax;
        const int e0 = 2 * lane + w, e1 = 2 * (lane + 32) + w;
        sel_lo = __ballot_sync(0xffffffffu, e0 < nblk && ((ub[e0] >> half) & 1));
        sel_hi = __ballot_sync(0xffffffffu, e1 < nblk && ((ub[e1] >> half) & 1));
      }
      const int j0 = (pr - static_cast<int>(g & 1)) & 1;
      for (int j = j0; j < n; j += 2) {
        const uint32_t t = g + j;
        mbar_wait(&bars[Bx::S_FULL + pr], (t >> 1) & 1);
        tc_fence_after();
        if (rows_live) {
          // real keys in this warpgroup's half of the tile
          int valid;
          if (TPB == 1) {
            valid = block_size(p.L, BLK, irow[j]) - w * HB;
          } else {
            const int jb = TPB * j + w;  // the selected block this half holds
            valid = jb < nblk ? block_size(p.L, KB, irow[jb]) : 0;
            // a pair's union entry that this row's query block did not select
            if (UNI && valid > 0) {
              const bool sel = j < 32 ? (sel_lo >> j) & 1u
                             : j < 64 ? (sel_hi >> (j - 32)) & 1u
                                      : (p.ubits[u * p.kmax + jb] >> (row >> 6)) & 1;
              if (!sel) valid = 0;
            }
          }
          if (valid <= 0) {
            // nothing of this half is attended (warp-uniform: an unselected
            // pair entry, or an odd count's missing partner): P = 0, no exps
            const uint32_t zero[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
            for (int c = 0; c < HB / 32; ++c) tmem_st16(tS + c * 16, zero);
          } else {
            uint32_t sr[HB];
#pragma unroll
            for (int c = 0; c < HB / 32; ++c) tmem_ld32(tS + c * 32, sr + c * 32);
            tmem_wait_ld();
            if (valid < HB) {
#pragma unroll
              for (int c = 0; c < HB; ++c)
                if (c >= valid) sr[c] = __float_as_uint(-INFINITY);
            }
            l_run += half_exp<BLK>(sr, tS, p.scale_log2, m_ref);
          }
          tmem_wait_st();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[Bx::P_FULL + pr]);
      }
      g += n;
      // the next unit's Q goes to the other TMEM buffer now, so its first
      // QK^T overlaps this unit's epilogue
      if (pos + gridDim.x < p.num_units) prep(pos + gridDim.x, uc + 1);
      // ---------------------------------------------- fused epilogue
      // l = the four warpgroups' partial sums; warpgroup q finalises output
      // columns [32q, 32q + 32) of its row
      mbar_wait(&bars[Bx::O_FULL], uc & 1);
      tc_fence_after();
      uint32_t ob[32];
      tmem_ld32(tOq, ob);
      xl[q * 128 + row] = l_run;
      named_bar_sync(3, 512);
      const float l_all = (xl[row] + xl[128 + row]) + (xl[256 + row] + xl[384 + row]);
      const float inv_l = 1.f / l_all;
      // the reference m was too low (P, l and O headed for overflow) or too
      // high (every P flushed): hand the unit to the running-max kernel
      // pairs: rows of a query block outside the call's range are neither checked nor stored
      const int qrow_blk = UNI ? 2 * qb + (row >> 6) : 0;
      const bool in_range = !UNI || (qrow_blk >= p.qlo && qrow_blk < p.qhi);
      const bool bad = rows_live && row < qrows && in_range &&
                       !(l_all >= 7.9e-31f && l_all <= 1.29e33f);  // [2^-100, 2^110]
      if (__any_sync(0xffffffffu, bad) && lane == 0 && p.flag_count != nullptr) {
        if (UNI) {  // the running-max kernel recomputes the pair's query blocks as plain units
          for (int e = 0; e < 2; ++e) {
            const int qq = 2 * qb + e;
            const int64_t uo = static_cast<int64_t>(bh) * p.nb_orig + qq;
            if (qq >= p.qlo && qq < p.qhi && atomicExch(p.unit_flag + uo, 1) == 0)
              p.flag_list[atomicAdd(p.flag_count, 1)] = static_cast<int32_t>(uo);
          }
        } else if (atomicExch(p.unit_flag + u, 1) == 0) {
          p.flag_list[atomicAdd(p.flag_count, 1)] = static_cast<int32_t>(u);
        }
      }
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars[Bx::O_EMPTY]);
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float o = __uint_as_float(ob[i]) * inv_l;
        ob[i] = __float_as_uint(o);
        ss = fmaf(o, o, ss);
      }
      xs[q * 128 + row] = ss;
      named_bar_sync(3, 512);
      ss = (xs[row] + xs[128 + row]) + (xs[256 + row] + xs[384 + row]);
      const bool live = row < qrows && in_range;
      if (!live) continue;
      const int64_t flat = static_cast<int64_t>(qb) * QR + row;
      const int64_t tok = p.perm ? p.perm[flat] : flat;
      const int b = bh / p.H, h = bh % p.H;
      const float inv = 1.f / sqrtf(ss / static_cast<float>(D) + p.eps);
      const int col0 = q * 32;
      if (p.o_sparse) {
        float* dst = p.o_sparse + (static_cast<int64_t>(bh) * p.L + tok) * D + col0;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + i) = make_float4(__uint_as_float(ob[i]), __uint_as_float(ob[i + 1]),
                                                            __uint_as_float(ob[i + 2]), __uint_as_float(ob[i + 3]));
      }
      if (p.out || p.out_f32) {
        const float gate = sigmoidf_stable(p.g_logit[static_cast<int64_t>(b) * p.L + tok] + p.b_g);
        const int64_t orow = ((static_cast<int64_t>(b) * p.L + tok) * p.out_H + p.out_h0 + h) * D + col0;
        store_fused_row(p, orow, ob, inv, gate, col0);
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

// Longest-first unit schedule for variable per-row block counts (the `keep`
// rule, decomposition.py:105-111).  The persistent kernel's CTA c takes
// positions c, c + G, c + 2G, ...; here, per head (so the CTAs in flight
// still share one head's K/V in L2), the head's units are ranked by
// descending selected-block count (ties by block id) and laid out over the
// positions in snake order (full rounds of G alternate direction), which
// balances the CTAs' total work.  One CTA per (batch, head).
__global__ void schedule_units_kernel(const int32_t* __restrict__ cnt, int nb, int64_t num_units, int G,
                                      int32_t* __restrict__ order) {
  extern __shared__ int32_t sc[];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * nb;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sc[i] = cnt[base + i];
  __syncthreads();
  const int64_t full_rounds = num_units / G;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    const int c = sc[i];
    int rank = 0;
    for (int j = 0; j < nb; ++j) {
      const int cj = sc[j];
      rank += (cj > c) | ((cj == c) & (j < i));
    }
    const int64_t pos = base + rank;
    const int64_t r = pos / G;
    int64_t slot = pos % G;
    if ((r & 1) && r < full_rounds) slot = G - 1 - slot;
    order[r * G + slot] = static_cast<int32_t>(base + i);
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
#ifdef ROPESLR_WATCHDOG
  {
    static unsigned long long* hbuf = nullptr;
    if (!hbuf) {
      cudaHostAlloc(&hbuf, 4096, cudaHostAllocMapped);
      void* dptr = nullptr;
      cudaHostGetDevicePointer(&dptr, hbuf, 0);
      cudaMemcpyToSymbol(g_watchdog, &dptr, sizeof(dptr));
    }
    // (the pointer is set before this launch on the first call: re-launch note below)
    for (int i = 0; i < 60; ++i) {
      if (cudaStreamQuery(st) == cudaSuccess) break;
      usleep(100000);
      if (hbuf[0]) {
        usleep(500000);
        fprintf(stderr, "WATCHDOG %llu waiters (S_FULL=%d P_FULL=%d O_FULL=%d O_EMPTY=%d V_FULL=%d K_FULL=%d)\n",
                hbuf[0], Bars<BLK>::S_FULL, Bars<BLK>::P_FULL, Bars<BLK>::O_FULL,
                Bars<BLK>::O_EMPTY, Bars<BLK>::V_FULL, Bars<BLK>::K_FULL);
        for (unsigned long long k = 0; k < hbuf[0] && k < 30; ++k)
          fprintf(stderr, "  block %llu thread %llu barrier %llu parity %llu line %llu\n", hbuf[2 + k * 4],
                  hbuf[3 + k * 4], hbuf[4 + k * 4] & 0xffffffffull, hbuf[4 + k * 4] >> 32, hbuf[5 + k * 4]);
        fflush(stderr);
        break;
      }
    }
  }
#endif
#if ROPESLR_K2_MEASURE
  if (prm.trace) {  // measurement build only: clock64 trace of CTA 0 (scripts/exp_k2.py)
    long long h[2 * 64 * 4];
    if (cudaMemcpyAsync(h, prm.trace, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    const char* path = getenv("ROPESLR_K2_TRACE");
    if (FILE* f = path ? fopen(path, "w") : nullptr) {
      for (int i = 0; i < 128; ++i)
        fprintf(f, "%d %d %lld %lld %lld\n", i / 64, i % 64, h[i * 4] ? h[i * 4] - h[0] : -1,
                h[i * 4 + 1] ? h[i * 4 + 1] - h[0] : -1, h[i * 4 + 2] ? h[i * 4 + 2] - h[0] : -1);
      fclose(f);
    }
  }
#endif
  return launch_status();
}

// The fixed-reference kernel, then the running-max kernel over its flagged units.
template <int BLK, int KB, bool UNI = false>
static int launch_fixed(const ropeslr_shape* s, const void* q, const void* k, const void* v, Params prm,
                        int* fallback, cudaStream_t st, const Params* plain = nullptr) {
  const int64_t BH = s->B * s->H;
  // fallback area: [unit_flag: all B*H*nb units][count: 1][list]; flags are
  // indexed by (plain, 64-row) unit, which neither a query-block range nor
  // the pairing renumbers
  const int64_t nu_all = BH * (UNI ? prm.nb_orig : prm.nb);
  prm.unit_flag = fallback;
  prm.flag_count = fallback + nu_all;
  prm.flag_list = fallback + nu_all + 1;
  if (cudaMemsetAsync(fallback, 0, (nu_all + 1) * sizeof(int), st) != cudaSuccess) return ROPESLR_ERR_LAUNCH;
  prm.kmat = static_cast<const __nv_bfloat16*>(k);
  CUtensorMap mq, mk, mv;
  if (!make_map(&mq, q, BH, s->L, UNI ? M : KB) || !make_map(&mk, k, BH, s->L, KB) ||
      !make_map(&mv, v, BH, s->L, KB))
    return ROPESLR_ERR_LAUNCH;
  auto kfn = sparse_attn_fixed_kernel<BLK, KB, UNI>;
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, fx::Layout<BLK>::ALLOC) != cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  const int64_t grid = prm.num_units < num_sms() ? prm.num_units : num_sms();
  kfn<<<static_cast<unsigned>(grid), kThreads, fx::Layout<BLK>::ALLOC, st>>>(mq, mk, mv, prm);
  if (int e = launch_status()) return e;
  if (ROPESLR_K2_MEASURE && prm.debug_mode >= 2) return ROPESLR_OK;  // measurement modes: the fixed kernel alone
  // the running-max kernel over the flagged units (usually none: its CTAs
  // read a zero count and retire); after a pair launch they are plain units
  Params fb = UNI ? *plain : prm;
  fb.nq = 0;
  fb.order = prm.flag_list;
  fb.num_units_dev = prm.flag_count;
  fb.unit_flag = nullptr;
  fb.flag_count = nullptr;
  fb.flag_list = nullptr;
  return launch_tc<KB>(s, q, k, v, fb, st);
}

// Union key lists of query-block pairs (2p, 2p + 1): one warp per pair; the
// two lists are ascending and duplicate-free, so an element's place in the
// union is (its index) + (the other list's elements below it) - (the shared
// elements below it): one binary search per element and a warp prefix count
// of the shared ones, no sequential merge.  A last unpaired block (odd nb)
// keeps its own list.
__device__ __forceinline__ int lower_bound_i32(const int32_t* __restrict__ a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Places the elements of X (n) among those of Y (m) in the union: out
// position i + #(Y < x_i) - #(shared elements of X before i), the bit of X
// set and the bit of Y too when x_i is shared; returns the shared count.
// skip_shared: X is the second list, whose shared elements the first list
// already wrote.
__device__ __forceinline__ int place_list(const int32_t* __restrict__ X, int n, const int32_t* __restrict__ Y, int m,
                                          uint8_t bit_x, uint8_t bit_y, bool skip_shared, int32_t* __restrict__ out,
                                          uint8_t* __restrict__ bits, int lane) {
  int carry = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    int x = 0, ry = 0;
    bool shared = false;
    if (i < n) {
      x = X[i];
      ry = lower_bound_i32(Y, m, x);
      shared = ry < m && Y[ry] == x;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, shared);
    const int before = carry + __popc(bal & ((1u << lane) - 1u));
    if (i < n && !(skip_shared && shared)) {
      const int pos = i + ry - before;
      out[pos] = x;
      bits[pos] = static_cast<uint8_t>(bit_x | (shared ? bit_y : 0));
    }
    carry += __popc(bal);
  }
  return carry;
}

__global__ void union_pairs_kernel(const int32_t* __restrict__ idx, int kmax, const int32_t* __restrict__ cnt,
                                   int nb, int npairs, int64_t nunits, int ukmax, int32_t* __restrict__ uidx,
                                   int32_t* __restrict__ ucnt, uint8_t* __restrict__ ubits) {
  const int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (u >= nunits) return;
  const int64_t bh = u / npairs;
  const int pr = static_cast<int>(u % npairs);
  const int64_t ua = bh * nb + 2 * pr;
  const int32_t* A = idx + ua * kmax;
  const int na = cnt[ua];
  const bool has_b = 2 * pr + 1 < nb;
  const int32_t* B = has_b ? idx + (ua + 1) * kmax : A;
  const int nbb = has_b ? cnt[ua + 1] : 0;
  int32_t* out = uidx + u * ukmax;
  uint8_t* bits = ubits + u * ukmax;
  const int shared = place_list(A, na, B, nbb, 1, 2, false, out, bits, lane);
  place_list(B, nbb, A, na, 2, 1, true, out, bits, lane);
  if (lane == 0) ucnt[u] = na + nbb - shared;
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
  if (s->qb_begin != 0 || s->qb_end != 0) {
    const int64_t nb = ceil_div(s->L, s->block);
    if (s->qb_begin < 0 || s->qb_end <= s->qb_begin || s->qb_end > nb) return ROPESLR_ERR_SHAPE;
  }
  if (!device_is_sm100()) return ROPESLR_ERR_ARCH;
  return ROPESLR_OK;
}

static int resolve_impl(const ropeslr_shape* s, int impl) {
  if (impl == ROPESLR_IMPL_AUTO) return tc::tc_eligible(s) ? ROPESLR_IMPL_TCGEN05 : ROPESLR_IMPL_SIMT;
  if (impl == ROPESLR_IMPL_TCGEN05 && !tc::tc_eligible(s)) return -1;
  if (impl != ROPESLR_IMPL_SIMT && impl != ROPESLR_IMPL_TCGEN05) return -1;
  return impl;
}

// workspace of the fixed-reference path: [schedule: NU][fallback: 2 NU + 1],
// then for block 64 the query-block pairs' union lists:
// [ucnt: BH * npairs][uidx: BH * npairs * nb][ubits: BH * npairs * nb bytes]
static size_t pair_area_offset(const ropeslr_shape* s) {
  const size_t nu = static_cast<size_t>(s->B * s->H * ceil_div(s->L, s->block));
  return ((3 * nu + 1) * sizeof(int32_t) + 255) / 256 * 256;
}
static size_t pair_area_bytes(const ropeslr_shape* s) {
  if (s->block != 64) return 0;
  const size_t nb = static_cast<size_t>(ceil_div(s->L, s->block)), np = (nb + 1) / 2;
  const size_t units = static_cast<size_t>(s->B * s->H) * np;
  return units * sizeof(int32_t) + units * nb * sizeof(int32_t) + units * nb;
}

static int launch_fixed_dispatch(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                                 const tc::Params& prm, void* ws, cudaStream_t st) {
  int* fallback = static_cast<int*>(ws) + s->B * s->H * prm.nb;
  if (s->block == 128) return tc::launch_fixed<128, 128>(s, q, k, v, prm, fallback, st);
  // block 64: two selected blocks per 128-key tile unless ROPESLR_PAIR64=0
  if (!tuning().pair64) return tc::launch_fixed<64, 64>(s, q, k, v, prm, fallback, st);
  if (tuning().pairs64) {
    // units of two adjacent query blocks over the union of their selections
    const int64_t BH = s->B * s->H;
    const int nb = prm.nb, npairs = (nb + 1) / 2;
    const int ukmax = 2 * prm.kmax < nb ? 2 * prm.kmax : nb;
    const int64_t units = BH * npairs;
    uint8_t* area = static_cast<uint8_t*>(ws) + pair_area_offset(s);
    int32_t* ucnt = reinterpret_cast<int32_t*>(area);
    int32_t* uidx = ucnt + units;
    uint8_t* ubits = reinterpret_cast<uint8_t*>(uidx + units * ukmax);
    tc::union_pairs_kernel<<<static_cast<unsigned>(ceil_div(units * 32, 256)), 256, 0, st>>>(
        prm.idx, prm.kmax, prm.cnt, nb, npairs, units, ukmax, uidx, ucnt, ubits);
    if (cudaGetLastError() != cudaSuccess) return ROPESLR_ERR_LAUNCH;
    tc::Params up = prm;
    up.idx = uidx;
    up.cnt = ucnt;
    up.kmax = ukmax;
    up.nb = npairs;
    up.num_units = units;
    up.ubits = ubits;
    up.nb_orig = nb;
    up.order = nullptr;
    up.qlo = 0;
    up.qhi = nb;
    if (prm.nq > 0) {
      // a query-block range: the pairs it touches; rows of a split pair's
      // other block are left alone
      up.qlo = prm.qb0;
      up.qhi = prm.qb0 + prm.nq;
      up.qb0 = prm.qb0 / 2;
      up.nq = (up.qhi - 1) / 2 - up.qb0 + 1;
      up.num_units = BH * up.nq;
    }
    // the union sizes range from k to 2k: longest-first over the pairs
    const int64_t G = up.num_units < num_sms() ? up.num_units : num_sms();
    if (prm.nq == 0 && tuning().schedule && npairs <= 8192) {
      int32_t* order = static_cast<int32_t*>(ws);
      tc::schedule_units_kernel<<<static_cast<unsigned>(BH), 512, npairs * sizeof(int32_t), st>>>(
          ucnt, npairs, units, static_cast<int>(G), order);
      if (cudaGetLastError() != cudaSuccess) return ROPESLR_ERR_LAUNCH;
      up.order = order;
    }
    return tc::launch_fixed<128, 64, true>(s, q, k, v, up, fallback, st, &prm);
  }
  return tc::launch_fixed<128, 64>(s, q, k, v, prm, fallback, st);
}

// K2 flavour for the tcgen05 path: the fixed-reference kernel unless
// ROPESLR_K2=online asks for the running-max (v7) kernel.
static bool use_fixed_reference() { return !tuning().k2_online; }

static int launch_tc_dispatch(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                              const tc::Params& prm, cudaStream_t st) {
  return s->block == 128 ? tc::launch_tc<128>(s, q, k, v, prm, st) : tc::launch_tc<64>(s, q, k, v, prm, st);
}

static tc::Params base_params(const ropeslr_shape* s, const int32_t* idx, int kmax, const int32_t* cnt,
                              const int32_t* perm, cudaStream_t st) {
  tc::Params prm{};
  prm.idx = idx;
  prm.cnt = cnt;
  prm.kmax = kmax;
  prm.nb = static_cast<int>(ceil_div(s->L, s->block));
  prm.H = static_cast<int>(s->H);
  prm.L = s->L;
  prm.num_units = s->B * s->H * prm.nb;
  if (s->qb_end > s->qb_begin) {  // a query-block range (validated by check_attn_args)
    prm.qb0 = s->qb_begin;
    prm.nq = s->qb_end - s->qb_begin;
    prm.num_units = s->B * s->H * prm.nq;
  }
  prm.perm = perm;
  prm.order = nullptr;
  prm.kmat = nullptr;
  prm.unit_flag = nullptr;
  prm.flag_count = nullptr;
  prm.flag_list = nullptr;
  prm.num_units_dev = nullptr;
  prm.out_H = static_cast<int>(s->H);
  prm.out_h0 = 0;
  prm.scale_log2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(s->d)));
  // K/V tiles are re-read by many query blocks of the head: keep them in L2
  // (evict_last) ahead of the streamed Q / y_lr / out; ROPESLR_KV_EVICT_LAST=0
  // turns the hint off
  prm.kv_evict_last = tuning().kv_evict_last ? 1 : 0;
  prm.debug_mode = 0;
  prm.trace = nullptr;
#if ROPESLR_K2_MEASURE
  // measurement build only (scripts/build_variant.sh): K2 mode switches and the clock64 trace
  const char* dbg = getenv("ROPESLR_DEBUG_MODE");
  prm.debug_mode = dbg ? atoi(dbg) : 0;
  static long long* tbuf = nullptr;
  if (getenv("ROPESLR_K2_TRACE")) {
    if (!tbuf && cudaMalloc(&tbuf, 2 * 64 * 4 * 8) != cudaSuccess) tbuf = nullptr;
    if (tbuf && cudaMemsetAsync(tbuf, 0, 2 * 64 * 4 * 8, st) == cudaSuccess) prm.trace = tbuf;
  }
#endif
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
  if (which == ROPESLR_IMPL_SIMT) {
    if (s->qb_end > s->qb_begin) return ROPESLR_ERR_SHAPE;  // query-block ranges: tcgen05 path only
    return launch_sparse_attention_simt(s, q, k, v, idx, kmax, cnt, row_perm, o_sparse, cs);
  }
  tc::Params prm = base_params(s, idx, kmax, cnt, row_perm, cs);
  prm.o_sparse = o_sparse;
  return launch_tc_dispatch(s, q, k, v, prm, cs);
}

namespace ropeslr {
constexpr int kMaxScheduledBlocks = 8192;  // larger nb: identity order (the O(nb^2) ranking gets slow)
static int64_t num_units_of(const ropeslr_shape* s) { return s->B * s->H * ceil_div(s->L, s->block); }

// The longest-first unit schedule into the workspace's first num_units
// int32 (ROPESLR_SCHEDULE=0 turns it off).  On skewed `keep` inputs (1 to
// 397 blocks per row, 12 heads of the Wan shape, scripts/exp_keep.py) it is
// 19-20% faster with the fixed-reference kernel; on uniform top-k counts it
// is neutral.
static int schedule_units(const ropeslr_shape* s, const int32_t* cnt, tc::Params& prm, void* ws, cudaStream_t cs) {
  if (!tuning().schedule || prm.nq > 0 || prm.nb > kMaxScheduledBlocks) return ROPESLR_OK;
  // top-k rows (index rows narrower than nb) all hold k blocks: balanced by
  // construction, so the identity order is as good and the ranking is skipped
  if (prm.kmax < prm.nb) return ROPESLR_OK;
  const int64_t G = prm.num_units < num_sms() ? prm.num_units : num_sms();
  int32_t* order = static_cast<int32_t*>(ws);
  tc::schedule_units_kernel<<<static_cast<unsigned>(s->B * s->H), 512, prm.nb * sizeof(int32_t), cs>>>(
      cnt, prm.nb, prm.num_units, static_cast<int>(G), order);
  if (cudaGetLastError() != cudaSuccess) return ROPESLR_ERR_LAUNCH;
  prm.order = order;
  return ROPESLR_OK;
}
}  // namespace ropeslr

extern "C" size_t ropeslr_attend_workspace_bytes(const ropeslr_shape* s, int32_t impl) {
  if (!s) return 0;
  const int which = resolve_impl(s, impl);
  if (which == ROPESLR_IMPL_SIMT) return static_cast<size_t>(s->B * s->H * s->L * s->d) * sizeof(float);
  // tcgen05 path: the longest-first unit schedule, then the fallback area of
  // the fixed-reference kernel, then (block 64) the query-block pairs' lists
  return pair_area_offset(s) + pair_area_bytes(s);
}

namespace ropeslr {
// K2 + K4 (tcgen05 path only) writing heads [out_h0, out_h0 + H) of
// out / y_lr rows that hold out_H heads: a head chunk of a wider forward
// (forward_host.cu).
int attend_fused_tc_strided(const ropeslr_shape* s, const void* q, const void* k, const void* v, const int32_t* idx,
                            int32_t kmax, const int32_t* cnt, const void* y_lr, const float* g_logit, float b_g,
                            const float* rms_sparse, float eps, void* out, int out_H, int out_h0, void* ws,
                            size_t ws_bytes, cudaStream_t stream) {
  int st = check_attn_args(s, q, k, v, idx, kmax, cnt);
  if (st) return st;
  if (!tc::tc_eligible(s)) return ROPESLR_ERR_VALUE;
  if (out_h0 < 0 || out_h0 + s->H > out_H) return ROPESLR_ERR_SHAPE;
  if (!y_lr || !g_logit || !rms_sparse || !out) return ROPESLR_ERR_NULL;
  // the fused epilogue moves y_lr / out rows with 256-bit accesses
  if (!aligned32(y_lr) || !aligned32(out)) return ROPESLR_ERR_ALIGN;
  tc::Params prm = base_params(s, idx, kmax, cnt, nullptr, stream);
  prm.y_lr = static_cast<const __nv_bfloat16*>(y_lr);
  prm.g_logit = g_logit;
  prm.b_g = b_g;
  prm.rms_sp = rms_sparse;
  prm.eps = eps;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.out_H = out_H;
  prm.out_h0 = out_h0;
  if (ws && ws_bytes >= ropeslr_attend_workspace_bytes(s, ROPESLR_IMPL_TCGEN05)) {
    if (int e = schedule_units(s, cnt, prm, ws, stream)) return e;
    if (use_fixed_reference()) return launch_fixed_dispatch(s, q, k, v, prm, ws, stream);
  }
  return launch_tc_dispatch(s, q, k, v, prm, stream);
}
bool attend_tc_eligible(const ropeslr_shape* s) { return tc::tc_eligible(s); }
}  // namespace ropeslr

namespace ropeslr {
int fuse_output(const ropeslr_shape* s, const float* o_sparse, const void* y_lr, const float* g_logit, float b_g,
                const float* rms_sparse, float eps, void* out, int out_dtype, cudaStream_t stream_);
}

extern "C" int ropeslr_attend_fused(const ropeslr_shape* s, const void* q, const void* k, const void* v,
                                    const int32_t* idx, int32_t kmax, const int32_t* cnt, const int32_t* row_perm,
                                    const void* y_lr, const float* g_logit, float b_g, const float* rms_sparse,
                                    float eps, void* out, int32_t out_dtype, float* o_sparse, int32_t impl, void* ws,
                                    size_t ws_bytes, void* stream) {
  int st = check_attn_args(s, q, k, v, idx, kmax, cnt);
  if (st) return st;
  if (!y_lr || !g_logit || !rms_sparse || !out) return ROPESLR_ERR_NULL;
  if (!(eps > 0.f)) return ROPESLR_ERR_VALUE;
  if (out_dtype != s->dtype && out_dtype != ROPESLR_F32) return ROPESLR_ERR_DTYPE;
  const int which = resolve_impl(s, impl);
  if (which < 0) return ROPESLR_ERR_VALUE;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  if (o_sparse && !aligned16(o_sparse)) return ROPESLR_ERR_ALIGN;
  if (which == ROPESLR_IMPL_SIMT) {
    if (s->qb_end > s->qb_begin) return ROPESLR_ERR_SHAPE;  // query-block ranges: tcgen05 path only
    if (!aligned16(y_lr) || !aligned16(out)) return ROPESLR_ERR_ALIGN;
    float* osp = o_sparse;
    if (osp == nullptr) {
      if (!ws || ws_bytes < ropeslr_attend_workspace_bytes(s, impl)) return ROPESLR_ERR_WORKSPACE;
      osp = static_cast<float*>(ws);
    }
    st = launch_sparse_attention_simt(s, q, k, v, idx, kmax, cnt, row_perm, osp, cs);
    if (st) return st;
    return fuse_output(s, osp, y_lr, g_logit, b_g, rms_sparse, eps, out, out_dtype, cs);
  }
  // the fused epilogue moves y_lr / out rows with 256-bit accesses
  if (!aligned32(y_lr) || !aligned32(out)) return ROPESLR_ERR_ALIGN;
  tc::Params prm = base_params(s, idx, kmax, cnt, row_perm, cs);
  prm.y_lr = static_cast<const __nv_bfloat16*>(y_lr);
  prm.g_logit = g_logit;
  prm.b_g = b_g;
  prm.rms_sp = rms_sparse;
  prm.eps = eps;
  if (out_dtype == ROPESLR_F32)
    prm.out_f32 = static_cast<float*>(out);
  else
    prm.out = static_cast<__nv_bfloat16*>(out);
  prm.o_sparse = o_sparse;
  if (ws && ws_bytes >= ropeslr_attend_workspace_bytes(s, impl)) {
    if (int e = schedule_units(s, cnt, prm, ws, cs)) return e;
  }
  if (use_fixed_reference() && ws && ws_bytes >= ropeslr_attend_workspace_bytes(s, impl))
    return launch_fixed_dispatch(s, q, k, v, prm, ws, cs);
  return launch_tc_dispatch(s, q, k, v, prm, cs);
}
