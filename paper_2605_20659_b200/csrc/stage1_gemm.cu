// The float32 GEMMs of the Stage-I step (training.py; mechanism.py:456-488)
// on the tcgen05 tensor cores with float32-grade accuracy: every operand is
// split into bf16 hi + lo parts (a = hi + lo, |lo| <= 2^-9 |a|) and
//
//   A B ~= A_hi B_hi + A_hi B_lo + A_lo B_hi      (float32 accumulation),
//
// which keeps ~16 significant bits of every product (the dropped A_lo B_lo
// term is 2^-18 relative), three MMAs per 16-wide k-step.  The shapes are the
// compensator's: a long token dimension L and small K, N in {64, 128}.
//
//   rows  C[h] = epi(A[h] B[h]):  A [H, L, K] row-major, B [H, K, N] (small),
//         C [H, L, N]; one 128-token tile per MMA, B's hi / lo images in
//         shared memory for the whole CTA; epilogues: none, sigmoid
//         (h1 = sigma(x_hat W_A)), or the sigmoid derivative of a given
//         tensor (dz1 = (dz2 W_B^T) * h1 (1 - h1));
//   gram  C[h] = sum_l A[h][l]^T B[h][l]:  A [H, L, 128], B [H, L, N]; per
//         CTA a chunk of tokens accumulated in TMEM (both operands
//         MN-major, the reduction runs over the tile's tokens), partials
//         reduced over the chunks in fixed order (deterministic), optionally
//         transposed and added into the output.
//
// Operands are loaded as float32 by the converter warps (16-byte loads),
// split and written in the 128B-swizzled layout the UMMA descriptors read.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace ropeslr {
namespace s1g {

using namespace sm100;

constexpr int M = 128;  // tokens per tile (rows kernel) / MMA M

// Chunk c (8 bf16) of row r of a [rows x C] bf16 tile in 64-column atoms of
// rows x 128 B, 128B-swizzled.
__device__ __forceinline__ uint32_t sw_off(int rows, int r, int c) {
  return (c >> 3) * (rows * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4);
}

__device__ __forceinline__ void split8(const float* f, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 a = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    const float2 af = __bfloat1622float2(a);
    const __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i] - af.x, f[2 * i + 1] - af.y);
    h[i] = *reinterpret_cast<const uint32_t*>(&a);
    l[i] = *reinterpret_cast<const uint32_t*>(&b);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ void load8(const float* p, bool valid, float* f) {
  if (valid) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = 0.f;
  }
}

// Convert a [128 x C] float32 tile (rows row0.., row stride C, rows >= nrows
// zero) into swizzled bf16 hi / lo tiles; NT threads, thread t.  All of a
// thread's loads are issued before the conversions, so a tile's bytes are in
// flight at once.
template <int C, int NT>
__device__ __forceinline__ void convert_tile(const float* src, int64_t row0, int64_t nrows, uint8_t* hi, uint8_t* lo,
                                             int t) {
  constexpr int CH = C / 8;             // chunks per row
  constexpr int PER = M * CH / NT;      // chunks per thread
  static_assert(M * CH % NT == 0, "tile chunks split evenly");
  float f[PER][8];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = t + i * NT;
    const int r = e / CH, c = e % CH;
    load8(src + (row0 + r) * C + c * 8, row0 + r < nrows, f[i]);
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = t + i * NT;
    const int r = e / CH, c = e % CH;
    uint4 h, l;
    split8(f[i], h, l);
    const uint32_t off = sw_off(M, r, c);
    *reinterpret_cast<uint4*>(hi + off) = h;
    *reinterpret_cast<uint4*>(lo + off) = l;
  }
}

enum Epi { EPI_NONE = 0, EPI_SIGMOID = 1, EPI_DSIG = 2 };

struct RowsArgs {
  CUtensorMap mC;    // C as [H][L][N] float32, box [32 columns, 32 rows, 1], 128-byte swizzle
  CUtensorMap mAux;  // aux, the same way (EPI_DSIG)
  const float* A;    // [H, L, K]
  const float* B;    // [H, K, N], or [H, N, K] when b_trans (B^T given)
  const float* aux;  // EPI_DSIG: h1 [H, L, N]
  float* C;          // [H, L, N]
  int64_t L;
  int H;
  int b_trans;
  int epi;
  int ntiles;  // ceil(L / 128) per head
};

template <int K, int N>
struct RowsLay {
  static constexpr int F_BYTES = M / 2 * K * 4;  // one float32 staging half tile (64 rows, bulk copy target)
  static constexpr int A_BYTES = M * K * 2;   // one of hi / lo
  static constexpr int B_BYTES = N * K * 2;
  static constexpr int EW = (K == 128 && N == 128) ? 4 : 8;       // epilogue warps (two per TMEM lane quarter)
  static constexpr int FST = K == 128 ? 2 : 4;                    // staging half-tile stages
  static constexpr int AST = K == 128 ? 1 : 2;                   // converted A stages
  static constexpr int O_BYTES = 32 * 128;      // an epilogue warp's [32 rows x 32 columns] float32 store box
  static constexpr int OFF_F = 0;
  static constexpr int OFF_A = OFF_F + FST * F_BYTES;          // [AST][hi, lo]
  static constexpr int OFF_B = OFF_A + AST * 2 * A_BYTES;      // [hi, lo] K-major [N rows][K]
  static constexpr int OFF_O = OFF_B + 2 * B_BYTES;            // [EW warps][2 buffers] store boxes
  static constexpr int OFF_BAR = OFF_O + 2 * EW * O_BYTES;
  static constexpr int THREADS = 256 + EW * 32 + 64;           // converters, epilogue, MMA, bulk copies
  static constexpr int W_MMA = 8 + EW, W_LOAD = 9 + EW;
  static constexpr int BYTES = OFF_BAR + 34 * 8;
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

constexpr int kConv = 256;  // converter threads (warps 0-7)

// A float32 A tile is one contiguous run of rows (row stride K): warp 13
// moves it into a staging ring in two 64-row bulk copies, so the bytes in
// flight do not depend on registers; the converter warps split it from
// shared memory into the swizzled bf16 hi / lo operand tiles.
template <int K, int N>
__global__ void __launch_bounds__(RowsLay<K, N>::THREADS, 1) stage1_rows_kernel(const __grid_constant__ RowsArgs a) {
  using Lay = RowsLay<K, N>;
  constexpr int FST = Lay::FST, AST = Lay::AST;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  uint8_t* sF = smem + Lay::OFF_F;
  uint8_t* sA = smem + Lay::OFF_A;
  uint8_t* sB = smem + Lay::OFF_B;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* ffull = bars;        // [4]
  uint64_t* fempty = bars + 4;   // [4]
  uint64_t* afull = bars + 8;    // [2]
  uint64_t* aempty = bars + 10;  // [2]
  uint64_t* accf = bars + 12;    // [2]
  uint64_t* acce = bars + 14;    // [2]
  uint64_t* obar = bars + 16;    // [EW warps][2 boxes]: the aux box landed (EPI_DSIG)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 32);
  // the CTA's tiles: one contiguous range, so B (per head) changes at most
  // a couple of times
  const int64_t total = static_cast<int64_t>(a.H) * a.ntiles;
  const int64_t beg = total * blockIdx.x / gridDim.x, end = total * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(&ffull[i], 1);
      mbar_init(&fempty[i], kConv);
    }
    for (int i = 0; i < 2 * Lay::EW; ++i) mbar_init(&obar[i], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], kConv);
      mbar_init(&aempty[i], 1);
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], Lay::EW * 32);
    }
    fence_mbar_init();
  }
  if (warp == Lay::W_MMA) {
    tmem_alloc(tmem_slot, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == Lay::W_LOAD) {
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      uint32_t hc = 0;  // half tiles issued
      for (int64_t pos = beg; pos < end; ++pos) {
        const int h = static_cast<int>(pos / a.ntiles);
        const int tile = static_cast<int>(pos % a.ntiles);
        for (int hf = 0; hf < 2; ++hf, ++hc) {
          const int s = hc % FST;
          if (hc >= FST) mbar_wait_sleep(&fempty[s], ((hc / FST) - 1) & 1);
          const int64_t row0 = static_cast<int64_t>(tile) * M + hf * (M / 2);
          const int64_t left = a.L - row0;
          const int rows = static_cast<int>(left <= 0 ? 0 : left < M / 2 ? left : M / 2);
          const uint32_t bytes = static_cast<uint32_t>(rows) * K * 4;
          mbar_arrive_expect_tx(&ffull[s], bytes);
          if (rows > 0)
            bulk_load_1d(sF + s * Lay::F_BYTES, a.A + (static_cast<int64_t>(h) * a.L + row0) * K, bytes, &ffull[s],
                         pol);
        }
      }
    }
  } else if (warp < kConv / 32) {
    constexpr int CH = K / 8, PER = M * CH / kConv;
    int cur_h = -1;
    uint32_t it = 0;
    for (int64_t pos = beg; pos < end; ++pos, ++it) {
      const int h = static_cast<int>(pos / a.ntiles);
      const int tile = static_cast<int>(pos % a.ntiles);
      const int sa = it % AST;
      if (it >= AST) mbar_wait_sleep(&aempty[sa], ((it / AST) - 1) & 1);
      if (h != cur_h) {
        // B of head h as K-major [N rows][K] hi / lo images; every MMA on the
        // previous head's B has completed (aempty of the previous tile)
        if (it >= 1) mbar_wait_sleep(&aempty[(it - 1) % AST], ((it - 1) / AST) & 1);
        asm volatile("bar.sync 2, %0;" ::"n"(kConv) : "memory");
        const float* B = a.B + static_cast<int64_t>(h) * K * N;
        for (int e = threadIdx.x; e < N * (K / 8); e += kConv) {
          const int n = e / (K / 8), c = e % (K / 8);
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int k = c * 8 + i;
            f[i] = a.b_trans ? B[static_cast<int64_t>(n) * K + k] : B[static_cast<int64_t>(k) * N + n];
          }
          uint4 hv, lv;
          split8(f, hv, lv);
          const uint32_t off = sw_off(N, n, c);
          *reinterpret_cast<uint4*>(sB + off) = hv;
          *reinterpret_cast<uint4*>(sB + Lay::B_BYTES + off) = lv;
        }
        cur_h = h;
      }
      const int64_t nrows = a.L - static_cast<int64_t>(tile) * M;
      uint8_t* hi = sA + sa * 2 * Lay::A_BYTES;
      uint8_t* lo = hi + Lay::A_BYTES;
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        const uint32_t hc = 2 * it + hf;
        const int sf = hc % FST;
        mbar_wait_sleep(&ffull[sf], (hc / FST) & 1);
        const float* src = reinterpret_cast<const float*>(sF + sf * Lay::F_BYTES);
#pragma unroll 4
        for (int i = 0; i < PER / 2; ++i) {
          const int e = threadIdx.x + i * kConv;
          const int rh = e / CH, c = e % CH, r = hf * (M / 2) + rh;
          float f[8];
          if (r < nrows) {
            const float4 x0 = *reinterpret_cast<const float4*>(src + rh * K + c * 8);
            const float4 x1 = *reinterpret_cast<const float4*>(src + rh * K + c * 8 + 4);
            f[0] = x0.x; f[1] = x0.y; f[2] = x0.z; f[3] = x0.w; f[4] = x1.x; f[5] = x1.y; f[6] = x1.z; f[7] = x1.w;
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = 0.f;
          }
          uint4 hv, lv;
          split8(f, hv, lv);
          const uint32_t off = sw_off(M, r, c);
          *reinterpret_cast<uint4*>(hi + off) = hv;
          *reinterpret_cast<uint4*>(lo + off) = lv;
        }
        mbar_arrive(&fempty[sf]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&afull[sa]);
    }
  } else if (warp == Lay::W_MMA) {
    constexpr uint32_t idesc = idesc_bf16_f32(M, N, false, false);
    const bool leader = elect_one();
    uint32_t it = 0;
    for (int64_t pos = beg; pos < end; ++pos, ++it) {
      const int sa = it % AST, ab = it & 1;
      mbar_wait_sleep(&afull[sa], (it / AST) & 1);
      if (it >= 2) mbar_wait_sleep(&acce[ab], ((it >> 1) - 1) & 1);
      tc_fence_after();
      if (leader) {
        const uint64_t dAh = desc_sw128(smem_u32(sA + sa * 2 * Lay::A_BYTES), 16, 1024);
        const uint64_t dAl = desc_sw128(smem_u32(sA + sa * 2 * Lay::A_BYTES + Lay::A_BYTES), 16, 1024);
        const uint64_t dBh = desc_sw128(smem_u32(sB), 16, 1024);
        const uint64_t dBl = desc_sw128(smem_u32(sB + Lay::B_BYTES), 16, 1024);
        const uint32_t acc = tmem + ab * 128;
#pragma unroll
        for (int kk = 0; kk < K / 16; ++kk) {
          const uint32_t ka = ((kk & 3) * 32 + (kk >> 2) * (M * 128)) >> 4;
          const uint32_t kb = ((kk & 3) * 32 + (kk >> 2) * (N * 128)) >> 4;
          mma_bf16_ss(acc, dAh + ka, dBh + kb, idesc, kk > 0 ? 1u : 0u);
          mma_bf16_ss(acc, dAh + ka, dBl + kb, idesc, 1u);
          mma_bf16_ss(acc, dAl + ka, dBh + kb, idesc, 1u);
        }
        mma_commit(&aempty[sa]);
        mma_commit(&accf[ab]);
      }
      __syncwarp();
    }
  } else {
    // epilogue warps 8 ..: TMEM lane quarter warp % 4 = token row; with 8
    // warps, warp 8 + q and 12 + q share a quarter (even / odd chunks).  Each
    // 32-column chunk goes TMEM -> registers -> (epilogue) -> a swizzled
    // [32 rows x 128 B] box in shared memory -> one TMA store (coalesced;
    // rows past L are clipped by the tensor map), two boxes in flight.
    // EPI_DSIG's h1 box arrives in the same buffer by a TMA load.
    const int q4 = warp & 3, lane = threadIdx.x & 31, ew = warp - 8;
    constexpr int CSTEP = Lay::EW / 4;  // chunks of a warp: c0, c0 + CSTEP, ...
    const int c0 = ew >> 2;
    uint8_t* obuf = smem + Lay::OFF_O + ew * 2 * Lay::O_BYTES;
    const bool dsig = a.epi == EPI_DSIG;
    uint32_t it = 0, nst = 0;
    for (int64_t pos = beg; pos < end; ++pos, ++it) {
      const int h = static_cast<int>(pos / a.ntiles);
      const int tile = static_cast<int>(pos % a.ntiles);
      const int ab = it & 1;
      const int row0 = tile * M + q4 * 32;
      mbar_wait_sleep(&accf[ab], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = c0; c < N / 32; c += CSTEP, ++nst) {
        uint8_t* box = obuf + (nst & 1) * Lay::O_BYTES;
        uint64_t* ob = &obar[ew * 2 + (nst & 1)];
        // the box written two stores ago has been read out
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          if (dsig) {
            mbar_arrive_expect_tx(ob, Lay::O_BYTES);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
                "%5}], [%2];" ::"r"(smem_u32(box)),
                "l"(reinterpret_cast<uint64_t>(&a.mAux)), "r"(smem_u32(ob)), "r"(c * 32), "r"(row0), "r"(h)
                : "memory");
          }
        }
        uint32_t u[32];
        tmem_ld32(tmem + ab * 128 + (static_cast<uint32_t>(q4 * 32) << 16) + c * 32, u);
        tmem_wait_ld();
        if (c + CSTEP >= N / 32) {
          tc_fence_before();
          mbar_arrive(&acce[ab]);
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(u[j]);
        if (a.epi == EPI_SIGMOID) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __frcp_rn(1.f + __expf(-v[j]));
        } else if (dsig) {
          mbar_wait(ob, (nst >> 1) & 1);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 g = *reinterpret_cast<const float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4));
            v[4 * j] *= g.x * (1.f - g.x);
            v[4 * j + 1] *= g.y * (1.f - g.y);
            v[4 * j + 2] *= g.z * (1.f - g.z);
            v[4 * j + 3] *= g.w * (1.f - g.w);
          }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
              make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&a.mC)),
                       "r"(smem_u32(box)), "r"(c * 32), "r"(row0), "r"(h)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == Lay::W_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// ------------------------------------------------------------------ gram
struct GramArgs {
  const float* A;   // [H, L, 128]
  const float* B;   // [H, L, N]
  float* partial;   // [H, nchunks, 128, N]
  int64_t L;
  int H;
  int ntiles;       // ceil(L / 128)
  int tiles_per_cta;
  int nchunks;
};

template <int N>
struct GramLay {
  static constexpr int A_BYTES = M * 128 * 2;  // one of hi / lo: [128 tok][128 cols]
  static constexpr int B_BYTES = M * N * 2;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int ST = N == 128 ? 1 : 2;  // stages that fit in 227 KiB
  static constexpr int OFF_BAR = ST * STAGE;
  static constexpr int BYTES = OFF_BAR + 8 * 8;
};

constexpr int kGramConv = 256;
constexpr int kGramThreads = kGramConv + 32;  // + warp 8: MMA, TMEM

template <int N>
__global__ void __launch_bounds__(kGramThreads, 1) stage1_gram_kernel(const __grid_constant__ GramArgs a) {
  using Lay = GramLay<N>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int h = blockIdx.y, chunk = blockIdx.x;
  const int t0 = chunk * a.tiles_per_cta;
  const int n = max(0, min(a.ntiles, t0 + a.tiles_per_cta) - t0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* full = bars;       // [2]
  uint64_t* empty = bars + 2;  // [2]
  uint64_t* done = bars + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], kGramConv);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 8) {
    tmem_alloc(tmem_slot, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const float* A = a.A + static_cast<int64_t>(h) * a.L * 128;
  const float* B = a.B + static_cast<int64_t>(h) * a.L * N;
  if (warp < 8) {
    for (int i = 0; i < n; ++i) {
      const int s = i % Lay::ST;
      if (i >= Lay::ST) mbar_wait_sleep(&empty[s], ((i / Lay::ST) - 1) & 1);
      uint8_t* st = smem + s * Lay::STAGE;
      const int64_t row0 = static_cast<int64_t>(t0 + i) * M;
      convert_tile<128, kGramConv>(A, row0, a.L, st, st + Lay::A_BYTES, threadIdx.x);
      convert_tile<N, kGramConv>(B, row0, a.L, st + 2 * Lay::A_BYTES, st + 2 * Lay::A_BYTES + Lay::B_BYTES,
                                 threadIdx.x);
      fence_proxy_async_smem();
      mbar_arrive(&full[s]);
    }
  } else {
    // D[m][n] = sum_tok A[tok][m] B[tok][n]: both operands MN-major, K = tokens
    constexpr uint32_t idesc = idesc_bf16_f32(M, N, true, true);
    const bool leader = elect_one();
    for (int i = 0; i < n; ++i) {
      const int s = i % Lay::ST;
      mbar_wait_sleep(&full[s], (i / Lay::ST) & 1);
      tc_fence_after();
      if (leader) {
        uint8_t* st = smem + s * Lay::STAGE;
        const uint64_t dAh = desc_sw128(smem_u32(st), M * 128, 1024);
        const uint64_t dAl = desc_sw128(smem_u32(st + Lay::A_BYTES), M * 128, 1024);
        const uint64_t dBh = desc_sw128(smem_u32(st + 2 * Lay::A_BYTES), M * 128, 1024);
        const uint64_t dBl = desc_sw128(smem_u32(st + 2 * Lay::A_BYTES + Lay::B_BYTES), M * 128, 1024);
#pragma unroll
        for (int kk = 0; kk < M / 16; ++kk) {
          const uint64_t k2 = static_cast<uint64_t>((kk * 2048) >> 4);
          mma_bf16_ss(tmem, dAh + k2, dBh + k2, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_bf16_ss(tmem, dAh + k2, dBl + k2, idesc, 1u);
          mma_bf16_ss(tmem, dAl + k2, dBh + k2, idesc, 1u);
        }
        mma_commit(&empty[s]);
        if (i == n - 1) mma_commit(done);
      }
      __syncwarp();
    }
  }
  // the chunk's partial: TMEM lane m = row m of A^T B
  __syncthreads();
  if (warp < 4) {
    const int m = threadIdx.x;
    float* dst = a.partial + ((static_cast<int64_t>(h) * a.nchunks + chunk) * M + m) * N;
    if (n > 0) {
      mbar_wait_sleep(done, 0);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < N / 32; ++c) {
        uint32_t u[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, u);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(dst + c * 32 + j) =
              make_float4(__uint_as_float(u[j]), __uint_as_float(u[j + 1]), __uint_as_float(u[j + 2]),
                          __uint_as_float(u[j + 3]));
      }
    } else {
      for (int j = 0; j < N; ++j) dst[j] = 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

// out[h] (+)= sum over chunks (fixed order) of partial [h][chunk][128][N],
// transposed ([N][128]) when trans.
template <int N>
__global__ void __launch_bounds__(256) stage1_gram_reduce_kernel(const float* __restrict__ partial, int nchunks,
                                                                 int trans, int accumulate, float* __restrict__ out) {
  const int h = blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const int m = e / N, n = e % N;
  const float* src = partial + static_cast<int64_t>(h) * nchunks * M * N + e;
  float s = 0.f;
  for (int c = 0; c < nchunks; ++c) s += src[static_cast<int64_t>(c) * M * N];
  float* dst = out + static_cast<int64_t>(h) * M * N + (trans ? static_cast<int64_t>(n) * M + m : e);
  *dst = accumulate ? *dst + s : s;
}

static int gram_chunks(int H, int ntiles) {
  int c = num_sms() / (H > 0 ? H : 1);
  if (c < 1) c = 1;
  if (c > ntiles) c = ntiles;
  return c;
}

}  // namespace s1g
}  // namespace ropeslr

using namespace ropeslr;

namespace ropeslr {
namespace s1g {
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
}  // namespace s1g
}  // namespace ropeslr

extern "C" int ropeslr_stage1_gemm_rows(int64_t H, int64_t L, int32_t K, int32_t N, const float* A, const float* B,
                                        int32_t b_trans, int32_t epi, const float* aux, float* C, void* stream) {
  if (!A || !B || !C || (epi == s1g::EPI_DSIG && !aux)) return ROPESLR_ERR_NULL;
  if (H < 1 || L < 1 || !((K == 64 || K == 128) && (N == 64 || N == 128))) return ROPESLR_ERR_SHAPE;
  if (epi < 0 || epi > 2) return ROPESLR_ERR_VALUE;
  if (!aligned16(A) || !aligned16(C) || (aux && !aligned16(aux))) return ROPESLR_ERR_ALIGN;
  s1g::RowsArgs a{};
  a.A = A;
  a.B = B;
  a.aux = aux;
  a.C = C;
  a.L = L;
  a.H = static_cast<int>(H);
  a.b_trans = b_trans;
  a.epi = epi;
  a.ntiles = static_cast<int>(ceil_div(L, s1g::M));
  {
    auto enc = s1g::encode_fn();
    if (enc == nullptr) return ROPESLR_ERR_LAUNCH;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(H)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(N) * 4, static_cast<cuuint64_t>(L) * N * 4};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&a.mC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, C, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return ROPESLR_ERR_LAUNCH;
    if (aux != nullptr &&
        enc(&a.mAux, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(aux), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return ROPESLR_ERR_LAUNCH;
  }
  const int64_t total = H * a.ntiles;
  const unsigned grid = static_cast<unsigned>(total < num_sms() ? total : num_sms());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define ROPESLR_ROWS(K_, N_)                                                                                 \
  {                                                                                                          \
    auto kfn = s1g::stage1_rows_kernel<K_, N_>;                                                              \
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, s1g::RowsLay<K_, N_>::BYTES) != \
        cudaSuccess)                                                                                         \
      return ROPESLR_ERR_LAUNCH;                                                                             \
    kfn<<<grid, s1g::RowsLay<K_, N_>::THREADS, s1g::RowsLay<K_, N_>::BYTES, st>>>(a);                                    \
  }
  if (K == 128 && N == 64) ROPESLR_ROWS(128, 64)
  else if (K == 64 && N == 128) ROPESLR_ROWS(64, 128)
  else if (K == 128 && N == 128) ROPESLR_ROWS(128, 128)
  else ROPESLR_ROWS(64, 64)
#undef ROPESLR_ROWS
  return launch_status();
}

extern "C" size_t ropeslr_stage1_gram_workspace_bytes(int64_t H, int64_t L, int32_t N) {
  if (H < 1 || L < 1 || (N != 64 && N != 128)) return 0;
  const int nch = s1g::gram_chunks(static_cast<int>(H), static_cast<int>(ceil_div(L, s1g::M)));
  return static_cast<size_t>(H) * nch * s1g::M * N * sizeof(float);
}

extern "C" int ropeslr_stage1_gemm_gram(int64_t H, int64_t L, int32_t N, const float* A, const float* B, float* out,
                                        int32_t transpose, int32_t accumulate, void* workspace, size_t ws_bytes,
                                        void* stream) {
  if (!A || !B || !out) return ROPESLR_ERR_NULL;
  if (H < 1 || L < 1 || (N != 64 && N != 128)) return ROPESLR_ERR_SHAPE;
  if (!aligned16(A) || !aligned16(B)) return ROPESLR_ERR_ALIGN;
  if (!workspace || ws_bytes < ropeslr_stage1_gram_workspace_bytes(H, L, N)) return ROPESLR_ERR_WORKSPACE;
  s1g::GramArgs a{};
  a.A = A;
  a.B = B;
  a.partial = static_cast<float*>(workspace);
  a.L = L;
  a.H = static_cast<int>(H);
  a.ntiles = static_cast<int>(ceil_div(L, s1g::M));
  a.nchunks = s1g::gram_chunks(a.H, a.ntiles);
  a.tiles_per_cta = static_cast<int>(ceil_div(a.ntiles, a.nchunks));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid(static_cast<unsigned>(a.nchunks), static_cast<unsigned>(H));
  const dim3 rgrid(static_cast<unsigned>(ceil_div(s1g::M * N, 256)), static_cast<unsigned>(H));
  if (N == 64) {
    if (cudaFuncSetAttribute(s1g::stage1_gram_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             s1g::GramLay<64>::BYTES) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    s1g::stage1_gram_kernel<64><<<grid, s1g::kGramThreads, s1g::GramLay<64>::BYTES, st>>>(a);
    if (int e = launch_status()) return e;
    s1g::stage1_gram_reduce_kernel<64><<<rgrid, 256, 0, st>>>(a.partial, a.nchunks, transpose, accumulate, out);
  } else {
    if (cudaFuncSetAttribute(s1g::stage1_gram_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             s1g::GramLay<128>::BYTES) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    s1g::stage1_gram_kernel<128><<<grid, s1g::kGramThreads, s1g::GramLay<128>::BYTES, st>>>(a);
    if (int e = launch_status()) return e;
    s1g::stage1_gram_reduce_kernel<128><<<rgrid, 256, 0, st>>>(a.partial, a.nchunks, transpose, accumulate, out);
  }
  return launch_status();
}
