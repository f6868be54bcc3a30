// K3 `linear` mode on tcgen05 with the 3D absolute-PE injection inside the
// kernels: the linear compensator of mechanism.py:33-36, 347-362, fed by the
// backbone projections of x_hat = x + alpha * PE (mechanism.py:429-432).
//
// The caller supplies the frozen projections of the plain token features,
// q_lin / k_lin / v_lin = x W_{q,k,v}[h] ([B, H, L, d] bf16; a DiT computes
// them for its own attention anyway).  The PE part of x_hat W is
// parameter-only and axis-separable,
//
//   (alpha * PE[p]) W = T[t] + T[x] + T[y],  T_axis = (alpha * P_axis) W,
//
// so ropeslr_linear_tables folds it once into per-axis [n_axis, d] tables
// per head and tensor (and the gate into per-axis scalars); the kernels add
// three table rows per token on the way through:
//
//   state   (one CTA per (head, token chunk))  TMA K, V tiles -> phi(k + T_k)
//           in place in shared memory -> tcgen05 S += phi(K)^T V, then the
//           PE part of V (T_v rows, written into V's buffer once that MMA
//           is done; adding it to the bf16 v would round it away) -> S +=
//           phi(K)^T T_v
//           (M = d, N = d, K = 128 tokens, both operands MN-major) into
//           TMEM, z = sum phi(k) in registers (fixed-order reduction over
//           the token slots at the end); the chunk's [d, d | z] partial
//           goes to the workspace;
//   reduce  partials summed in fixed chunk order (float64), written as the
//           apply GEMM's B operand image [S | z] / L (K-major,
//           128B-swizzled, fp16);
//   apply   (one CTA per (head, token chunk))  TMA Q tiles -> phi(q + T_q)
//           in place as fp16 -> tcgen05 [phi(Q) S | phi(Q) z] (fp16 x fp16,
//           N = 144) into a double-buffered TMEM accumulator; the epilogue
//           warps divide by max(phi(q) . z, 1e-8), RMS-normalise with
//           rms_lowrank and store y_lr (bf16) and optionally o_lr (f32);
//   gate    g_logit = x . w_g over the local columns + G[t] + G[x] + G[y]
//           (one warp per token: X is read once, no per-element PE gather).
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace ropeslr {
namespace lnu {

using namespace sm100;

constexpr int D = 128;                  // head dim
constexpr int M = 128;                  // tokens per tile
constexpr int HALF = M * 128;           // 16 KiB: one 64-column half of a tile (TMA box)
constexpr int TILE = 2 * HALF;          // 32 KiB
constexpr int TAB_PITCH = 272;          // bytes per bf16 table row: 128 values + 16 B (conflict-free rows)
constexpr int NB = 144;                 // apply GEMM N: 128 numerators + the denominator column + pad
constexpr int BHALF = NB * 128;         // 18 KiB: one 64-wide K half of the B image
constexpr int BIMG = 2 * BHALF;         // 36 KiB: the fp16 image
constexpr int NPART = NB;               // columns of a state partial: S row (128) | z | pad
constexpr float kFloor = 1e-8f;         // mechanism.py:347

__device__ __forceinline__ float elu1(float v) { return v > 0.f ? v + 1.f : __expf(v); }

// Chunk c (0..15: 8 bf16 each) of row r of a TMA-loaded [128 x 128] tile,
// two 64-column halves in the 128B-swizzled layout.
template <int ROWS = M>
__device__ __forceinline__ uint4* tile_chunk(uint8_t* tile, int r, int c) {
  return reinterpret_cast<uint4*>(tile + (c >> 3) * (ROWS * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

// In place on chunks [c0, c0 + NC) of row r of a tile: v + T[rt] + T[rx] +
// T[ry] (tables optional), then phi when PHI; rows of tokens beyond L become
// zero.  Several threads share a row (each its own chunk range), so the
// CUDA-core work of a tile spreads over many warps.
__device__ __forceinline__ float2 bf16x2_to_f32x2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}

// phi(k) = elu(k) + 1 = exp(min(k, 0)) + max(k, 0) (mechanism.py:33-36),
// branch-free: exp(0) = 1 supplies the +1 of the positive side.  With
// 2 min(k, 0) = k - |k| and 2 max(k, 0) = k + |k| (both exact) the work
// stays on the FMA pipe (|k| is an operand modifier) instead of four
// min / max on the ALU; bit-identical to the min / max form.
__device__ __forceinline__ float2 phi2(float2 k) {
  const float2 ak = make_float2(fabsf(k.x), fabsf(k.y));
  const float2 neg2 = __fadd2_rn(k, make_float2(-ak.x, -ak.y));  // 2 min(k, 0)
  const float2 pos2 = __fadd2_rn(k, ak);  // 2 max(k, 0)
  const float2 e = __fmul2_rn(neg2, make_float2(0.72134752044448170f, 0.72134752044448170f));  // log2(e) / 2
  float2 r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(e.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(e.y));
  return __ffma2_rn(pos2, make_float2(0.5f, 0.5f), r);
}

// In place on chunks [c0, c0 + NC) of row r of a tile: v + (T[rt] + T[rx] +
// T[ry]) (tables optional; the three table rows are summed in bf16x2, their
// sum is small against v and is rounded once more with v to bf16 anyway),
// then phi when PHI; rows of tokens beyond L become zero.  Several threads
// share a row (each its own chunk range), so the CUDA-core work of a tile
// spreads over many warps.  ACC: add the phi values to acc (z = sum phi(k)).
// F16OUT: store fp16 instead of bf16 (the apply GEMM runs fp16 x fp16).
template <bool PHI, int NC, bool ACC = false, bool F16OUT = false, int ROWS = M>
__device__ __forceinline__ void transform_row(uint8_t* tile, int r, int c0, bool valid, const uint8_t* tab, int rt,
                                              int rx, int ry, float (*acc)[NC * 8] = nullptr, int rot = 0) {
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) {
    // rot: visit the chunks rotated (two threads of a row on the two halves
    // then land in different bank groups of the swizzled tile)
    const int c = c0 + ((cc + rot) & (NC - 1));
    uint4* p = tile_chunk<ROWS>(tile, r, c);
    if (!valid) {
      *p = make_uint4(0, 0, 0, 0);
      continue;
    }
    uint4 u = *p;
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t t[4] = {0u, 0u, 0u, 0u};
    if (tab != nullptr) {
      const uint4 a = *reinterpret_cast<const uint4*>(tab + rt * TAB_PITCH + c * 16);
      const uint4 b = *reinterpret_cast<const uint4*>(tab + rx * TAB_PITCH + c * 16);
      const uint4 e = *reinterpret_cast<const uint4*>(tab + ry * TAB_PITCH + c * 16);
      const uint32_t aa[4] = {a.x, a.y, a.z, a.w}, bb[4] = {b.x, b.y, b.z, b.w}, ee[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 s2 = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&aa[i]),
                                    *reinterpret_cast<const __nv_bfloat162*>(&bb[i]));
        s2 = __hadd2(s2, *reinterpret_cast<const __nv_bfloat162*>(&ee[i]));
        t[i] = *reinterpret_cast<uint32_t*>(&s2);
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = bf16x2_to_f32x2(w[i]);
      if (tab != nullptr) f = __fadd2_rn(f, bf16x2_to_f32x2(t[i]));
      if (PHI) f = phi2(f);
      if (ACC) {
        (*acc)[cc * 8 + 2 * i] += f.x;
        (*acc)[cc * 8 + 2 * i + 1] += f.y;
      }
      if (F16OUT) {
        __half2 h2 = __floats2half2_rn(f.x, f.y);
        o[i] = *reinterpret_cast<uint32_t*>(&h2);
      } else {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(f.x, f.y);
        o[i] = *reinterpret_cast<uint32_t*>(&h2);
      }
    }
    *p = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Chunks [c0, c0 + NC) of row r of a tile := T[rt] + T[rx] + T[ry] (bf16x2
// sums), zero for tokens beyond L: the PE part of V as its own MMA operand.
// V itself stays the exact bf16 input: adding a table value much smaller than
// v's bf16 spacing and rounding again would drop it systematically.
template <int NC, int ROWS = M>
__device__ __forceinline__ void table_row(uint8_t* tile, int r, int c0, bool valid, const uint8_t* tab, int rt, int rx,
                                          int ry) {
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) {
    const int c = c0 + cc;
    uint4* p = tile_chunk<ROWS>(tile, r, c);
    if (!valid) {
      *p = make_uint4(0, 0, 0, 0);
      continue;
    }
    const uint4 a = *reinterpret_cast<const uint4*>(tab + rt * TAB_PITCH + c * 16);
    const uint4 b = *reinterpret_cast<const uint4*>(tab + rx * TAB_PITCH + c * 16);
    const uint4 e = *reinterpret_cast<const uint4*>(tab + ry * TAB_PITCH + c * 16);
    const uint32_t aa[4] = {a.x, a.y, a.z, a.w}, bb[4] = {b.x, b.y, b.z, b.w}, ee[4] = {e.x, e.y, e.z, e.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 s2 = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&aa[i]),
                                  *reinterpret_cast<const __nv_bfloat162*>(&bb[i]));
      s2 = __hadd2(s2, *reinterpret_cast<const __nv_bfloat162*>(&ee[i]));
      o[i] = *reinterpret_cast<uint32_t*>(&s2);
    }
    *p = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

struct Grid3 {
  int T, Hg, Wg;
  // table rows of token l: t, T + x, T + Hg + y (32-bit: L < 2^31 on this path)
  __device__ __forceinline__ void rows(int64_t l, int& rt, int& rx, int& ry) const {
    const uint32_t u = static_cast<uint32_t>(l);
    const uint32_t row = u / static_cast<uint32_t>(Wg);
    rt = static_cast<int>(row / static_cast<uint32_t>(Hg));
    rx = T + static_cast<int>(row - static_cast<uint32_t>(rt) * Hg);
    ry = T + Hg + static_cast<int>(u - row * static_cast<uint32_t>(Wg));
  }
};

struct StateArgs {
  int64_t L;
  int H;
  Grid3 g;
  int use_pe;
  int nrows;
  int ntiles;           // ceil(L / SR)
  int tiles_per_cta;
  int nchunks;
  const uint8_t* tables;    // [H][3][nrows][TAB_PITCH] bf16 (q, k, v): the rows of t read here
  float* partial;       // [BH][nchunks][128][NPART]: phi(K)^T (V + T_xy,v) per chunk
  float* phi_t;         // [BH][nchunks][T][128]: sum of phi(k) over the chunk's tokens of each t
};

// The state pass in 64-token stages, three deep.  TMA brings K, V and the
// stage's 64 rows of the (x, y) tables of k and v (T_xy[x W + y] = T_x[x] +
// T_y[y], rows repeated past H W so a stage never wraps); the transform
// warps turn K into phi(k + T_k) in place (the MMA's A tile), and V and
// T_xy,v sit side by side as one N = 256 B operand: S_v | S_xy = phi(K)^T
// [V | T_xy,v] in one MMA per k-step.  The t part of the PE: phi(k + T_k) takes
// T_t,k[t] from shared memory, and sum_l phi(k_l) T_t,v[t(l)] = sum_t (sum
// over the tokens of t of phi(k)) T_t,v[t]: the per-t sums go out with the
// chunk (phi_t) and the reduce kernel adds their products with T_t,v
// (float32 tables).
constexpr int SR = 64;                 // tokens per state stage
constexpr int SHALF = SR * 128;        // 8 KiB: one 64-column half of a stage tile
constexpr int STILE = 2 * SHALF;       // 16 KiB
constexpr int SST = 3;                 // state ring depth
// smem: [SST][K -> phi(K) | V | Txy_v | Txy_k] | T_t,k rows | flush buffer [16 warps][128] | barriers
struct StateLay {
  static constexpr int STAGE = 4 * STILE;
  static constexpr int OFF_TAB = SST * STAGE;
  __host__ __device__ static int off_phi(int T) { return OFF_TAB + ((T * TAB_PITCH + 127) / 128) * 128; }
  __host__ __device__ static int off_bar(int T) { return off_phi(T) + 16 * D * 4; }
  __host__ __device__ static int bytes(int T) { return off_bar(T) + (4 * SST + 2) * 8 + 16; }
};

constexpr int kStateXf = 512;                 // transform threads: 8 per token row, 2 chunks each
constexpr int kStateThreads = kStateXf + 64;  // + warp 16 TMA, warp 17 MMA + TMEM
constexpr int kStateTma = kStateXf / 32, kStateMma = kStateTma + 1;

__global__ void __launch_bounds__(kStateThreads, 1)
    linear_state_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmXY, const __grid_constant__ StateArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int bh = blockIdx.y, chunk = blockIdx.x;
  const int h = bh % a.H;
  const int T = a.g.T, HW = a.g.Hg * a.g.Wg;
  const int t0 = chunk * a.tiles_per_cta;
  const int t1 = min(a.ntiles, t0 + a.tiles_per_cta);
  const int n = max(0, t1 - t0);
  uint8_t* sTab = smem + StateLay::OFF_TAB;
  float* sRed = reinterpret_cast<float*>(smem + StateLay::off_phi(T));  // [16 warps][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + StateLay::off_bar(T));
  uint64_t* full = bars;                 // [SST] TMA (K, V, Txy_v, Txy_k) landed
  uint64_t* ready = bars + SST;          // [SST] phi(K) written
  uint64_t* empty = bars + 2 * SST;      // [SST] MMA done with the stage
  uint64_t* done = bars + 3 * SST;       // MMA -> readout
  uint64_t* tabf = done + 1;             // T_t,k rows landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tabf + 1);
  const bool pe = a.use_pe != 0;
  auto stage = [&](int s) { return smem + s * StateLay::STAGE; };  // K -> phi(K) | V | Txy_v | Txy_k

  if (threadIdx.x == 0) {
    for (int i = 0; i < SST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&ready[i], kStateXf);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    mbar_init(tabf, 1);
    fence_mbar_init();
  }
  if (warp == kStateMma) {
    tmem_alloc(tmem_slot, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kStateTma) {
    if (elect_one()) {
      if (pe) {
        const uint8_t* gk = a.tables + (static_cast<int64_t>(h) * 3 + 1) * a.nrows * TAB_PITCH;  // k, rows 0..T-1
        mbar_arrive_expect_tx(tabf, T * TAB_PITCH);
        bulk_load_1d(sTab, gk, T * TAB_PITCH, tabf, policy_evict_last());
      }
      const uint64_t pol = policy_evict_first(), pol_t = policy_evict_last();
      for (int i = 0; i < n; ++i) {
        const int s = i % SST;
        if (i >= SST) mbar_wait_sleep(&empty[s], ((i / SST) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], (pe ? 4 : 2) * STILE);
        const int row = (t0 + i) * SR;
        uint8_t* st = stage(s);
        tma_load_3d_hint(st, &tmK, &full[s], 0, row, bh, pol);
        tma_load_3d_hint(st + SHALF, &tmK, &full[s], 64, row, bh, pol);
        tma_load_3d_hint(st + STILE, &tmV, &full[s], 0, row, bh, pol);
        tma_load_3d_hint(st + STILE + SHALF, &tmV, &full[s], 64, row, bh, pol);
        if (pe) {
          const int xy0 = row % HW;
          tma_load_3d_hint(st + 2 * STILE, &tmXY, &full[s], 0, xy0, 2 * h + 1, pol_t);
          tma_load_3d_hint(st + 2 * STILE + SHALF, &tmXY, &full[s], 64, xy0, 2 * h + 1, pol_t);
          tma_load_3d_hint(st + 3 * STILE, &tmXY, &full[s], 0, xy0, 2 * h, pol_t);
          tma_load_3d_hint(st + 3 * STILE + SHALF, &tmXY, &full[s], 64, xy0, 2 * h, pol_t);
        }
      }
    }
  } else if (warp == kStateMma) {
    // per stage: [S_v | S_xy] += phi(K)^T [V | T_xy,v] (N = 256 with PE)
    const uint32_t idesc_s = pe ? idesc_bf16_f32(M, 2 * D, true, true) : idesc_bf16_f32(M, D, true, true);
    const bool leader = elect_one();
    for (int i = 0; i < n; ++i) {
      const int s = i % SST;
      mbar_wait_sleep(&full[s], (i / SST) & 1);
      mbar_wait_sleep(&ready[s], (i / SST) & 1);
      tc_fence_after();
      if (leader) {
        uint8_t* st = stage(s);
        const uint64_t dA = desc_sw128(smem_u32(st), SHALF, 1024);
        const uint64_t dB = desc_sw128(smem_u32(st + STILE), SHALF, 1024);
#pragma unroll
        for (int kk = 0; kk < SR / 16; ++kk)
          mma_bf16_ss(tmem, dA + static_cast<uint64_t>((kk * 2048) >> 4), dB + static_cast<uint64_t>((kk * 2048) >> 4),
                      idesc_s, (i > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
        if (i == n - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    // transform warps: 8 threads per token row (chunks c0 and c0 + 8: the 8
    // threads of a row, one shared-memory phase, touch 8 distinct 16-byte
    // bank groups of the swizzled tile).  The phi sums accumulate per thread
    // for the CTA's current t; when a stage reaches a new t every thread
    // takes part in a fixed-order reduction over the 64 row slots (shuffles
    // within a warp, then the 16 warps in order), written straight to phi_t,
    // so the result does not depend on timing; the phi of a token of a later
    // t in that stage is recomputed from its registers for its own t.
    const int r = threadIdx.x >> 3, c0 = threadIdx.x & 7, lane = threadIdx.x & 31, xw = threadIdx.x >> 5;
    float* gphi = a.phi_t + (static_cast<int64_t>(bh) * a.nchunks + chunk) * T * D;
    for (int e = threadIdx.x; e < T * D; e += kStateXf) gphi[e] = 0.f;
    asm volatile("bar.sync 1, %0;" ::"n"(kStateXf) : "memory");
    if (pe) mbar_wait_sleep(tabf, 0);
    float zacc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) zacc[j] = 0.f;
    // the phi sums of t over the slots, into phi_t[t]: v (this thread's 16 columns)
    auto reduce_to = [&](int tt, const float (&v)[16]) {
      float w[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        w[j] = v[j];
        w[j] += __shfl_down_sync(0xffffffffu, w[j], 16);
        w[j] += __shfl_down_sync(0xffffffffu, w[j], 8);
      }
      if (lane < 8) {
#pragma unroll
        for (int j = 0; j < 16; ++j) sRed[xw * D + c0 * 8 + (j < 8 ? j : 64 + j - 8)] = w[j];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kStateXf) : "memory");
      if (threadIdx.x < D) {
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += sRed[q * D + threadIdx.x];
        gphi[tt * D + threadIdx.x] = acc;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kStateXf) : "memory");
    };
    // token of this slot in stage i: l = (t0 + i) SR + r; its t, stepped
    int64_t l = static_cast<int64_t>(t0) * SR + r;
    int tt = static_cast<int>(l / HW), xy = static_cast<int>(l - static_cast<int64_t>(tt) * HW);
    int cta_t = static_cast<int>((static_cast<int64_t>(t0) * SR) / HW);  // the CTA's current t
    for (int i = 0; i < n; ++i) {
      const int s = i % SST;
      const bool valid = l < a.L;
      mbar_wait_sleep(&full[s], (i / SST) & 1);
      const uint8_t* trow = pe ? sTab + tt * TAB_PITCH : nullptr;
      uint8_t* at = stage(s);
      uint4 kc[2], tc[2], bc[2];
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        kc[cc] = *tile_chunk<SR>(at, r, c0 + 8 * cc);
        tc[cc] = pe ? *tile_chunk<SR>(at + 3 * STILE, r, c0 + 8 * cc) : make_uint4(0, 0, 0, 0);
        bc[cc] = pe ? *reinterpret_cast<const uint4*>(trow + (c0 + 8 * cc) * 16) : make_uint4(0, 0, 0, 0);
      }
      // phi of element pair e of chunk cc of this slot's token
      auto phi_at = [&](int cc, int e) {
        const uint32_t wv = e == 0 ? kc[cc].x : e == 1 ? kc[cc].y : e == 2 ? kc[cc].z : kc[cc].w;
        float2 f = bf16x2_to_f32x2(wv);
        if (pe) {
          const uint32_t av = e == 0 ? tc[cc].x : e == 1 ? tc[cc].y : e == 2 ? tc[cc].z : tc[cc].w;
          const uint32_t bv = e == 0 ? bc[cc].x : e == 1 ? bc[cc].y : e == 2 ? bc[cc].z : bc[cc].w;
          f = __fadd2_rn(f, __fadd2_rn(bf16x2_to_f32x2(bv), bf16x2_to_f32x2(av)));
        }
        return phi2(f);
      };
      const bool mine = valid && tt == cta_t;  // this token's phi belongs to the CTA's current t
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        uint4* p = tile_chunk<SR>(at, r, c0 + 8 * cc);
        if (!valid) {
          *p = make_uint4(0, 0, 0, 0);
          continue;
        }
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = phi_at(cc, e);
          if (mine) {
            zacc[cc * 8 + 2 * e] += f.x;
            zacc[cc * 8 + 2 * e + 1] += f.y;
          }
          __nv_bfloat162 h2 = __floats2bfloat162_rn(f.x, f.y);
          o[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
        *p = make_uint4(o[0], o[1], o[2], o[3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&ready[s]);
      // did this stage reach past the CTA's t?  (uniform: the stage's last valid token)
      const int64_t last = min(static_cast<int64_t>(t0 + i + 1) * SR, a.L) - 1;
      const int t_last = static_cast<int>(last / HW);
      if (t_last != cta_t) {
        // rare: close the current t, then each later t of this stage (phi of
        // the tokens of that t recomputed from the registers)
        for (int tq = cta_t; tq <= t_last; ++tq) {
          if (tq > cta_t) {
#pragma unroll
            for (int j = 0; j < 16; ++j) zacc[j] = 0.f;
            if (valid && tt == tq) {
#pragma unroll
              for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = phi_at(cc, e);
                  zacc[cc * 8 + 2 * e] = f.x;
                  zacc[cc * 8 + 2 * e + 1] = f.y;
                }
            }
          }
          if (tq < t_last) reduce_to(tq, zacc);
        }
        cta_t = t_last;
      }
      l += SR;
      xy += SR;
      while (xy >= HW) {
        xy -= HW;
        ++tt;
      }
    }
    if (n > 0) reduce_to(cta_t, zacc);
  }
  if (warp < 4) {  // warps 0-3 read TMEM lanes 0-127 (the rows of S) out: S_v + S_xy
    const int r = threadIdx.x;
    float* dst = a.partial + ((static_cast<int64_t>(bh) * a.nchunks + chunk) * D + r) * NPART;
    if (n > 0) {
      mbar_wait_sleep(done, 0);
      tc_fence_after();
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32], w[32];
        tmem_ld32(lane_base + c * 32, v);
        if (pe) tmem_ld32(lane_base + 128 + c * 32, w);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                 __uint_as_float(v[j + 3]));
          if (pe) {
            o.x += __uint_as_float(w[j]);
            o.y += __uint_as_float(w[j + 1]);
            o.z += __uint_as_float(w[j + 2]);
            o.w += __uint_as_float(w[j + 3]);
          }
          *reinterpret_cast<float4*>(dst + c * 32 + j) = o;
        }
      }
    } else {
      for (int j = 0; j < D; ++j) dst[j] = 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kStateMma) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// Sum the chunk partials (fixed order, float64) and write the apply GEMM's B
// operand: B[n][k] = S[k][n] / L for n < 128, B[128][k] = z[k] / L, zero rows
// above, with S = sum_chunks phi(K)^T (V + T_xy,v) + sum_t Phi[t]^T T_t,v[t]
// (Phi[t] = the chunks' phi_t summed; float32 T_t,v) and z = sum_t Phi[t];
// K-major, two 64-wide K halves of [144 rows x 128 B], 128B-swizzled as a
// 1024-aligned shared-memory copy expects, in fp16.  The common 1/L cancels
// in phi(q) S / phi(q) z and keeps z (a sum of L positive terms) inside
// fp16's range; fp16's 11-bit significand keeps S and z to ~5e-4, against
// bf16's 2^-9 for the phi(q) operand it meets in the MMA.  Also S and z in
// float32, unscaled (state [BH][128][NPART]), for inspection.
// phi_tot[bh][t][k] = sum over the chunks of phi_t (fixed order, float64).
__global__ void __launch_bounds__(128) linear_phi_sum_kernel(const float* __restrict__ phi_t, int nchunks, int T,
                                                             double* __restrict__ phi_tot) {
  const int bh = blockIdx.x, t = blockIdx.y, k = threadIdx.x;
  const float* p = phi_t + (static_cast<int64_t>(bh) * nchunks * T + t) * D + k;
  double acc = 0.0;
  for (int c = 0; c < nchunks; ++c) acc += p[static_cast<int64_t>(c) * T * D];
  phi_tot[(static_cast<int64_t>(bh) * T + t) * D + k] = acc;
}

// grid (BH, D / 8): block = 8 rows k of S (one per warp), lanes over the
// columns n (coalesced partial loads); T_t,v and the block's Phi rows are
// staged in shared memory.
__global__ void __launch_bounds__(256) linear_reduce_image_kernel(const float* __restrict__ partial,
                                                                  const double* __restrict__ phi_tot, int nchunks, int T,
                                                                  int H, const float* __restrict__ tf, int nrows,
                                                                  double inv_L, uint8_t* __restrict__ bimg,
                                                                  float* __restrict__ state) {
  extern __shared__ double sRed[];  // T_t,v [T][128] | Phi [8][T]
  double* sTv = sRed;
  double* sPhi = sRed + T * D;
  const int bh = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.y * 8 + warp;
  // T_t,v rows (float32 tables [H][3][nrows][128], tensor 2 = v, rows 0..T-1)
  const float* tv = tf != nullptr ? tf + (static_cast<int64_t>(bh % H) * 3 + 2) * nrows * D : nullptr;
  for (int e = threadIdx.x; e < T * D; e += blockDim.x) sTv[e] = tv != nullptr ? static_cast<double>(tv[e]) : 0.0;
  for (int e = threadIdx.x; e < 8 * T; e += blockDim.x)
    sPhi[e] = phi_tot[(static_cast<int64_t>(bh) * T + e % T) * D + blockIdx.y * 8 + e / T];
  __syncthreads();
  const float* src = partial + static_cast<int64_t>(bh) * nchunks * D * NPART;
  uint8_t* img = bimg + static_cast<int64_t>(bh) * BIMG;
  const double* ph = sPhi + warp * T;
  for (int n = lane; n < NB; n += 32) {
    double acc = 0.0;
    if (n < 128) {
      for (int c = 0; c < nchunks; ++c) acc += src[(static_cast<int64_t>(c) * D + k) * NPART + n];
      if (tv != nullptr)
        for (int t = 0; t < T; ++t) acc += ph[t] * sTv[t * D + n];
    } else if (n == 128) {
      for (int t = 0; t < T; ++t) acc += ph[t];
    }
    if (state != nullptr && n <= 128) state[(static_cast<int64_t>(bh) * D + k) * NPART + n] = static_cast<float>(acc);
    const int half = k >> 6, ch = (k & 63) >> 3, el = k & 7;
    const int off = half * BHALF + n * 128 + ((ch ^ (n & 7)) << 4) + el * 2;
    *reinterpret_cast<__half*>(img + off) = __float2half_rn(static_cast<float>(acc * inv_L));
  }
}

struct ApplyArgs {
  int64_t L;
  int H;
  Grid3 g;
  int use_pe;
  int nrows;
  int ntiles;
  int tiles_per_cta;
  const uint8_t* tables;  // [H][3][nrows][TAB_PITCH]
  const uint8_t* bimg;    // [BH][BIMG] fp16
  const float* rms_lr;
  float eps;
  __nv_bfloat16* y_lr;    // [B, L, H, d]
  float* o_lr;            // [B, H, L, d] nullable
};

// smem: Q ring (4 x 32 KiB) | B image (36 KiB) | T_q | rms | row sums | barriers
constexpr int QST = 4;  // Q ring depth
struct ApplyLay {
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_B = OFF_Q + QST * TILE;
  static constexpr int OFF_TAB = OFF_B + BIMG;
  __host__ __device__ static int off_rms(int nrows) { return OFF_TAB + ((nrows * TAB_PITCH + 127) / 128) * 128; }
  __host__ __device__ static int off_xs(int nrows) { return off_rms(nrows) + D * 4; }
  __host__ __device__ static int off_bar(int nrows) { return off_xs(nrows) + 2 * M * 4; }
  __host__ __device__ static int bytes(int nrows) { return off_bar(nrows) + (3 * QST + 5) * 8 + 16; }
};

constexpr int kApplyXf = 256;   // transform threads: 2 per token row, 8 chunks each (warps 0-7)
constexpr int kApplyEpi = 256;  // epilogue threads (warps 8-15): lane quarter warp % 4, tile parity (warp - 8) / 4
constexpr int kApplyTma = (kApplyXf + kApplyEpi) / 32, kApplyMma = kApplyTma + 1;
constexpr int kApplyThreads = kApplyXf + kApplyEpi + 64;

__global__ void __launch_bounds__(kApplyThreads, 1)
    linear_apply_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ ApplyArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int bh = blockIdx.y;
  const int h = bh % a.H, b = bh / a.H;
  const int t0 = blockIdx.x * a.tiles_per_cta;
  const int t1 = min(a.ntiles, t0 + a.tiles_per_cta);
  const int n = max(0, t1 - t0);
  uint8_t* sQ = smem + ApplyLay::OFF_Q;
  uint8_t* sB = smem + ApplyLay::OFF_B;
  uint8_t* sTab = smem + ApplyLay::OFF_TAB;
  float* sRms = reinterpret_cast<float*>(smem + ApplyLay::off_rms(a.nrows));
  float(*xs)[M] = reinterpret_cast<float(*)[M]>(smem + ApplyLay::off_xs(a.nrows));  // per-half row sums of squares
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ApplyLay::off_bar(a.nrows));
  uint64_t* full = bars;              // [QST] TMA -> transform
  uint64_t* ready = bars + QST;       // [QST] transform -> MMA
  uint64_t* empty = bars + 2 * QST;   // [QST] MMA -> TMA
  uint64_t* accf = bars + 3 * QST;    // [2] MMA -> epilogue
  uint64_t* acce = accf + 2;          // [2] epilogue -> MMA
  uint64_t* init = acce + 2;          // B image + table landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(init + 1);
  const int tab_bytes = a.nrows * TAB_PITCH;

  if (threadIdx.x == 0) {
    for (int i = 0; i < QST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&ready[i], kApplyXf);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], kApplyEpi / 2);
    }
    mbar_init(init, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < D; i += blockDim.x) sRms[i] = a.rms_lr[i];
  if (warp == kApplyMma) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kApplyTma) {
    if (elect_one()) {
      const uint8_t* gtab = a.tables + (static_cast<int64_t>(h) * 3) * tab_bytes;
      mbar_arrive_expect_tx(init, BIMG + (a.use_pe ? tab_bytes : 0));
      bulk_load_1d(sB, a.bimg + static_cast<int64_t>(bh) * BIMG, BIMG, init, policy_evict_last());
      if (a.use_pe) bulk_load_1d(sTab, gtab, tab_bytes, init, policy_evict_last());
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < n; ++i) {
        const int s = i % QST;
        if (i >= QST) mbar_wait_sleep(&empty[s], ((i / QST) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], TILE);
        const int row = (t0 + i) * M;
        tma_load_3d_hint(sQ + s * TILE, &tmQ, &full[s], 0, row, bh, pol);
        tma_load_3d_hint(sQ + s * TILE + HALF, &tmQ, &full[s], 64, row, bh, pol);
      }
    }
  } else if (warp == kApplyMma) {
    constexpr uint32_t idesc = idesc_f16_f32(M, NB, false, false);
    const bool leader = elect_one();
    mbar_wait_sleep(init, 0);
    const uint64_t dB = desc_sw128(smem_u32(sB), 16, 1024);
    for (int i = 0; i < n; ++i) {
      const int s = i % QST, ab = i & 1;
      mbar_wait_sleep(&ready[s], (i / QST) & 1);
      if (i >= 2) mbar_wait_sleep(&acce[ab], ((i >> 1) - 1) & 1);
      tc_fence_after();
      if (leader) {
        const uint64_t dA = desc_sw128(smem_u32(sQ + s * TILE), 16, 1024);
        const uint32_t acc_t = tmem + ab * 256;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ka = ((kk & 3) * 32 + (kk >> 2) * HALF) >> 4;
          const uint32_t kb = ((kk & 3) * 32 + (kk >> 2) * BHALF) >> 4;
          mma_f16_ss(acc_t, dA + ka, dB + kb, idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(&empty[s]);
        mma_commit(&accf[ab]);
      }
      __syncwarp();
    }
  } else if (warp < kApplyXf / 32) {
    // transform: 2 threads per token row, 8 of its 16 chunks each
    const int r = threadIdx.x >> 1, c0 = (threadIdx.x & 1) * 8;
    const uint8_t* tq = nullptr;
    if (a.use_pe) {
      mbar_wait_sleep(init, 0);
      tq = sTab;
    }
    for (int i = 0; i < n; ++i) {
      const int s = i % QST;
      mbar_wait_sleep(&full[s], (i / QST) & 1);
      const int64_t l = static_cast<int64_t>(t0 + i) * M + r;
      const bool valid = l < a.L;
      int rt = 0, rx = 0, ry = 0;
      if (valid) a.g.rows(l, rt, rx, ry);
      transform_row<true, 8, false, true>(sQ + s * TILE, r, c0, valid, tq, rt, rx, ry, nullptr, c0 >> 1);
      fence_proxy_async_smem();
      mbar_arrive(&ready[s]);
    }
  } else {
    // epilogue: row r = TMEM lane (warp % 4) * 32 + lane; warps 8-11 take
    // the even tiles (accumulator 0), warps 12-15 the odd ones (accumulator
    // 1), each whole rows of 128 columns: no exchange between warps
    const int q4 = warp & 3, par = (warp - kApplyXf / 32) >> 2;
    const int r = q4 * 32 + (threadIdx.x & 31);
    for (int i = par; i < n; i += 2) {
      const int ab = par;
      mbar_wait_sleep(&accf[ab], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t base = tmem + ab * 256 + (static_cast<uint32_t>(q4 * 32) << 16);
      // two passes over TMEM (the row's columns are not held in registers):
      // the sum of squares, then the normalised stores
      uint32_t den_u[2];
      tmem_ld2(base + 128, den_u);
      tmem_wait_ld();
      const float inv_den = 1.f / fmaxf(__uint_as_float(den_u[0]), kFloor);
      // sum of squares of the raw row (the 1 / den factor applied once, squared)
      float ss = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(base + c * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) ss = fmaf(__uint_as_float(v[j]), __uint_as_float(v[j]), ss);
      }
      const int64_t l = static_cast<int64_t>(t0 + i) * M + r;
      const bool live = l < a.L;
      const float inv = rsqrtf(ss * (inv_den * inv_den) / static_cast<float>(D) + a.eps);
      const float scale = inv_den * inv;  // o / den, RMS-normalised
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(base + c * 32, v);
        tmem_wait_ld();
        if (c == 3) {
          tc_fence_before();
          mbar_arrive(&acce[ab]);
        }
        if (!live) continue;
        const int cb = c * 32;
        if (a.o_lr != nullptr) {
          float* dst = a.o_lr + (static_cast<int64_t>(bh) * a.L + l) * D + cb;
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) =
                make_float4(__uint_as_float(v[j]) * inv_den, __uint_as_float(v[j + 1]) * inv_den,
                            __uint_as_float(v[j + 2]) * inv_den, __uint_as_float(v[j + 3]) * inv_den);
        }
        __nv_bfloat16* dst = a.y_lr + ((static_cast<int64_t>(b) * a.L + l) * a.H + h) * D + cb;
#pragma unroll
        for (int j = 0; j < 32; j += 16) {
          uint32_t u[8];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const float4 w4 = *reinterpret_cast<const float4*>(sRms + cb + j + 2 * e);
            __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(v[j + 2 * e]) * scale * w4.x,
                                                      __uint_as_float(v[j + 2 * e + 1]) * scale * w4.y);
            __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(v[j + 2 * e + 2]) * scale * w4.z,
                                                      __uint_as_float(v[j + 2 * e + 3]) * scale * w4.w);
            u[e] = *reinterpret_cast<uint32_t*>(&h0);
            u[e + 1] = *reinterpret_cast<uint32_t*>(&h1);
          }
          asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + j), "r"(u[0]),
                       "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7])
                       : "memory");
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kApplyMma) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- tables
// T[h][z][row][j] = sum_c alpha[c] P_axis[row][c] W_z[h][c][j] over all
// D_total columns (x_hat W with x_hat the full token row), rounded to bf16
// into padded rows.  grid (ceil(nrows / 16), 3 H), 128 threads (column j).
__global__ void __launch_bounds__(128) linear_fold_kernel(const float* __restrict__ pe_t, const float* __restrict__ pe_x,
                                                          const float* __restrict__ pe_y,
                                                          const float* __restrict__ alpha,
                                                          const float* __restrict__ wq, const float* __restrict__ wk,
                                                          const float* __restrict__ wv, int64_t Dt, int T, int Hg,
                                                          int Wg, uint8_t* __restrict__ tables,
                                                          float* __restrict__ tf) {
  constexpr int RT = 16, CK = 32;
  __shared__ float sp[RT][CK];
  const int nrows = T + Hg + Wg;
  const int r0 = blockIdx.x * RT;
  const int h = blockIdx.y / 3, z = blockIdx.y % 3;
  const float* W = (z == 0 ? wq : z == 1 ? wk : wv) + static_cast<int64_t>(h) * Dt * D;
  const int j = threadIdx.x;
  float acc[RT];
#pragma unroll
  for (int i = 0; i < RT; ++i) acc[i] = 0.f;
  for (int64_t c0 = 0; c0 < Dt; c0 += CK) {
    for (int e = threadIdx.x; e < RT * CK; e += blockDim.x) {
      const int rr = e / CK, cc = e % CK;
      const int row = r0 + rr;
      const int64_t c = c0 + cc;
      float v = 0.f;
      if (row < nrows && c < Dt) {
        const float* src = row < T ? pe_t + static_cast<int64_t>(row) * Dt
                         : row < T + Hg ? pe_x + static_cast<int64_t>(row - T) * Dt
                                        : pe_y + static_cast<int64_t>(row - T - Hg) * Dt;
        v = alpha[c] * src[c];
      }
      sp[rr][cc] = v;
    }
    __syncthreads();
    const int ck = static_cast<int>(Dt - c0 < CK ? Dt - c0 : CK);
    for (int cc = 0; cc < ck; ++cc) {
      const float w = W[(c0 + cc) * D + j];
#pragma unroll
      for (int i = 0; i < RT; ++i) acc[i] = fmaf(sp[i][cc], w, acc[i]);
    }
    __syncthreads();
  }
  uint8_t* out = tables + (static_cast<int64_t>(h) * 3 + z) * nrows * TAB_PITCH;
  float* outf = tf + (static_cast<int64_t>(h) * 3 + z) * nrows * D;
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int row = r0 + i;
    if (row < nrows) {
      reinterpret_cast<__nv_bfloat16*>(out + row * TAB_PITCH)[j] = __float2bfloat16_rn(acc[i]);
      outf[row * D + j] = acc[i];
    }
  }
}

// The (x, y) tables of k and v: Txy[h][z - 1][i][j] = bf16(T_x[x] + T_y[y]) in
// float32, x = (i mod HW) / W, y = i mod W, for i < HW + SR (a stage's 64
// rows never wrap).  grid (ceil(rows / 8), 2 H), 128 threads (column j).
__global__ void __launch_bounds__(128) linear_xy_kernel(const float* __restrict__ tf, int T, int Hg, int Wg, int nrows,
                                                        int xye, __nv_bfloat16* __restrict__ xy) {
  const int h = blockIdx.y >> 1, z = 1 + (blockIdx.y & 1);
  const float* src = tf + (static_cast<int64_t>(h) * 3 + z) * nrows * D;
  __nv_bfloat16* dst = xy + (static_cast<int64_t>(h) * 2 + (z - 1)) * xye * D;
  const int HW = Hg * Wg, j = threadIdx.x;
  for (int i = blockIdx.x * 8; i < min(xye, blockIdx.x * 8 + 8); ++i) {
    const int u = i % HW, x = u / Wg, y = u % Wg;
    dst[static_cast<int64_t>(i) * D + j] = __float2bfloat16_rn(src[(T + x) * D + j] + src[(T + Hg + y) * D + j]);
  }
}

// G[row] = sum over the local columns of alpha P_axis[row] w_g (float32).
__global__ void __launch_bounds__(256) linear_gate_fold_kernel(const float* __restrict__ pe_t,
                                                               const float* __restrict__ pe_x,
                                                               const float* __restrict__ pe_y,
                                                               const float* __restrict__ alpha,
                                                               const float* __restrict__ w_g, int64_t Dt, int64_t c0,
                                                               int64_t ncols, int T, int Hg, float* __restrict__ G) {
  __shared__ float red[8];
  const int row = blockIdx.x;
  const float* src = row < T ? pe_t + static_cast<int64_t>(row) * Dt
                   : row < T + Hg ? pe_x + static_cast<int64_t>(row - T) * Dt
                                  : pe_y + static_cast<int64_t>(row - T - Hg) * Dt;
  float s = 0.f;
  for (int64_t c = c0 + threadIdx.x; c < c0 + ncols; c += blockDim.x) s = fmaf(alpha[c] * src[c], w_g[c], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    G[row] = t;
  }
}

// g_logit[b, l] = x[b, l, local cols] . w_g[local cols] + G[t] + G[x] + G[y]
// (no bias: the fused epilogue adds it after any head-parallel all-reduce).
// One warp per token; 16-byte loads of X.
__global__ void __launch_bounds__(256) linear_gate_kernel(const __nv_bfloat16* __restrict__ x, int64_t row_stride,
                                                          const float* __restrict__ w_g, int64_t ncols, int64_t BL,
                                                          int64_t L, Grid3 g, const float* __restrict__ G,
                                                          float* __restrict__ g_logit) {
  const int64_t tok = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (tok >= BL) return;
  const __nv_bfloat16* row = x + tok * row_stride;
  float s = 0.f;
#pragma unroll 4
  for (int64_t c = lane * 8; c < ncols; c += 256) {
    float f[8];
    uint4 u;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
        : "l"(row + c));
    bf16x8_to_f32(u, f);
    const float4 wa = *reinterpret_cast<const float4*>(w_g + c);
    const float4 wb = *reinterpret_cast<const float4*>(w_g + c + 4);
    s = fmaf(f[0], wa.x, s);
    s = fmaf(f[1], wa.y, s);
    s = fmaf(f[2], wa.z, s);
    s = fmaf(f[3], wa.w, s);
    s = fmaf(f[4], wb.x, s);
    s = fmaf(f[5], wb.y, s);
    s = fmaf(f[6], wb.z, s);
    s = fmaf(f[7], wb.w, s);
  }
  s = warp_sum(s);
  if (lane == 0) {
    if (G != nullptr) {
      int rt, rx, ry;
      g.rows(tok % L, rt, rx, ry);
      s += (G[rt] + G[rx]) + G[ry];
    }
    g_logit[tok] = s;
  }
}

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

// [BH, L, 128] bf16 as a 3-D tensor, box [64 cols, 128 rows, 1], 128B swizzle;
// rows past L read as zero.
static bool make_map(CUtensorMap* m, const void* base, int64_t BH, int64_t L, int rows = M) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(BH)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(L) * D * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(rows), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int nrows_of(const ropeslr_token_args* t) { return t->grid_t + t->grid_h + t->grid_w; }

// The tables buffer: per-axis bf16 rows [H][3][nrows][TAB_PITCH] | gate
// scalars G [nrows] | per-axis float32 rows [H][3][nrows][128] | the (x, y)
// tables of k and v [H][2][HW + SR][128] bf16.
struct TabLay {
  size_t ax, g, tf, xy, total;
  int xye;
};
static size_t up256(size_t x);
static TabLay tab_layout(int64_t H, const ropeslr_token_args* t) {
  const int nr = nrows_of(t);
  TabLay y{};
  y.xye = t->grid_h * t->grid_w + SR;
  y.ax = 0;
  y.g = up256(static_cast<size_t>(H) * 3 * nr * TAB_PITCH);
  y.tf = y.g + up256(static_cast<size_t>(nr) * 4);
  y.xy = y.tf + up256(static_cast<size_t>(H) * 3 * nr * D * 4);
  y.total = y.xy + up256(static_cast<size_t>(H) * 2 * y.xye * D * 2);
  return y;
}

// CTAs per head: one wave over all heads (one CTA per SM; BH * chunks <= SMs
// when BH <= SMs, so no tail wave).
static int chunks_per_head(int64_t BH, int ntiles) {
  int64_t c = num_sms() / BH;
  if (c > ntiles) c = ntiles;
  return static_cast<int>(c < 1 ? 1 : c);
}

static size_t up256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace lnu
}  // namespace ropeslr

using namespace ropeslr;

static bool linear_pe_eligible(const ropeslr_shape* s, const ropeslr_token_args* t) {
  if (!s || !t || s->dtype != ROPESLR_BF16 || s->d != lnu::D || s->L >= (1LL << 31)) return false;
  const int nr = lnu::nrows_of(t);
  return lnu::StateLay::bytes(t->grid_t) <= 227 * 1024 && lnu::ApplyLay::bytes(nr) <= 227 * 1024 &&
         t->grid_t * (lnu::D + 8) * 8 <= 200 * 1024;
}

extern "C" size_t ropeslr_linear_tables_bytes(const ropeslr_shape* s, const ropeslr_token_args* t) {
  if (!linear_pe_eligible(s, t)) return 0;
  return lnu::tab_layout(s->H, t).total;
}

extern "C" int ropeslr_linear_tables(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_q,
                                     const float* w_k, const float* w_v, void* tables, size_t tables_bytes,
                                     void* stream) {
  if (!s || !t || !tables) return ROPESLR_ERR_NULL;
  if (!linear_pe_eligible(s, t)) return ROPESLR_ERR_SHAPE;
  if (t->token_offset != 0) return ROPESLR_ERR_SHAPE;
  if (tables_bytes < ropeslr_linear_tables_bytes(s, t)) return ROPESLR_ERR_WORKSPACE;
  if (!t->use_pe) return ROPESLR_OK;  // no PE: the tables are not read
  if (!w_q || !w_k || !w_v || !t->pe_t || !t->pe_x || !t->pe_y || !t->alpha || !t->w_g) return ROPESLR_ERR_NULL;
  if (t->d_model < (t->head_offset + s->H) * s->d) return ROPESLR_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nr = lnu::nrows_of(t);
  const lnu::TabLay ly = lnu::tab_layout(s->H, t);
  uint8_t* tab = static_cast<uint8_t*>(tables);
  float* tf = reinterpret_cast<float*>(tab + ly.tf);
  lnu::linear_fold_kernel<<<dim3(static_cast<unsigned>(ceil_div(nr, 16)), static_cast<unsigned>(3 * s->H)), 128, 0,
                            st>>>(t->pe_t, t->pe_x, t->pe_y, t->alpha, w_q, w_k, w_v, t->d_model, t->grid_t,
                                  t->grid_h, t->grid_w, tab, tf);
  if (int e = launch_status()) return e;
  lnu::linear_xy_kernel<<<dim3(static_cast<unsigned>(ceil_div(ly.xye, 8)), static_cast<unsigned>(2 * s->H)), 128, 0,
                          st>>>(tf, t->grid_t, t->grid_h, t->grid_w, nr, ly.xye,
                                reinterpret_cast<__nv_bfloat16*>(tab + ly.xy));
  if (int e = launch_status()) return e;
  float* G = reinterpret_cast<float*>(tab + ly.g);
  lnu::linear_gate_fold_kernel<<<nr, 256, 0, st>>>(t->pe_t, t->pe_x, t->pe_y, t->alpha, t->w_g, t->d_model,
                                                   t->head_offset * s->d, s->H * s->d, t->grid_t, t->grid_h, G);
  return launch_status();
}

extern "C" size_t ropeslr_linear_pe_workspace_bytes(const ropeslr_shape* s, const ropeslr_token_args* t) {
  if (!linear_pe_eligible(s, t)) return 0;
  const int64_t BH = s->B * s->H;
  const int ntiles = static_cast<int>(ceil_div(s->L, lnu::M));
  const int nch = lnu::chunks_per_head(BH, ntiles);
  return lnu::up256(static_cast<size_t>(BH) * nch * lnu::D * lnu::NPART * 4) +
         lnu::up256(static_cast<size_t>(BH) * lnu::BIMG) +
         lnu::up256(static_cast<size_t>(BH) * nch * t->grid_t * lnu::D * 4) +
         lnu::up256(static_cast<size_t>(BH) * t->grid_t * lnu::D * 8);
}

extern "C" int ropeslr_linear_branch_pe(const ropeslr_shape* s, const ropeslr_token_args* t, const void* q_lin,
                                        const void* k_lin, const void* v_lin, const void* tables,
                                        const float* rms_lowrank, float eps, void* y_lr, float* o_lr,
                                        float* g_logit, float* state, void* ws, size_t ws_bytes, void* stream) {
  if (!s || !t || !q_lin || !k_lin || !v_lin || !tables || !rms_lowrank || !y_lr || !t->x || !t->w_g)
    return ROPESLR_ERR_NULL;
  if (s->B < 1 || s->H < 1 || s->L < 1) return ROPESLR_ERR_SHAPE;
  if (!linear_pe_eligible(s, t)) return ROPESLR_ERR_SHAPE;
  if (static_cast<int64_t>(t->grid_t) * t->grid_h * t->grid_w != s->L || t->token_offset != 0)
    return ROPESLR_ERR_SHAPE;
  if (!(eps > 0.f)) return ROPESLR_ERR_VALUE;
  if (!aligned16(q_lin) || !aligned16(k_lin) || !aligned16(v_lin) || !aligned16(tables) || !aligned32(y_lr) ||
      !aligned16(t->x) || t->x_row_stride % 8 || (o_lr && !aligned16(o_lr)) || (state && !aligned16(state)))
    return ROPESLR_ERR_ALIGN;
  if (!ws || ws_bytes < ropeslr_linear_pe_workspace_bytes(s, t)) return ROPESLR_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t BH = s->B * s->H;
  const int nr = lnu::nrows_of(t);
  const int ntiles = static_cast<int>(ceil_div(s->L, lnu::M));
  const int nch = lnu::chunks_per_head(BH, ntiles);
  const int tpc = static_cast<int>(ceil_div(ntiles, nch));
  float* partial = static_cast<float*>(ws);
  uint8_t* bimg = static_cast<uint8_t*>(ws) + lnu::up256(static_cast<size_t>(BH) * nch * lnu::D * lnu::NPART * 4);
  float* phi_t = reinterpret_cast<float*>(bimg + lnu::up256(static_cast<size_t>(BH) * lnu::BIMG));
  double* phi_tot = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(phi_t) +
                                              lnu::up256(static_cast<size_t>(BH) * nch * t->grid_t * lnu::D * 4));
  const uint8_t* tab = static_cast<const uint8_t*>(tables);
  const lnu::TabLay ly = lnu::tab_layout(s->H, t);
  const float* G = reinterpret_cast<const float*>(tab + ly.g);
  lnu::Grid3 g{t->grid_t, t->grid_h, t->grid_w};

  CUtensorMap mq, mk, mv, mxy;
  if (!lnu::make_map(&mq, q_lin, BH, s->L) || !lnu::make_map(&mk, k_lin, BH, s->L, lnu::SR) ||
      !lnu::make_map(&mv, v_lin, BH, s->L, lnu::SR) ||
      !lnu::make_map(&mxy, tab + ly.xy, 2 * s->H, ly.xye, lnu::SR))
    return ROPESLR_ERR_LAUNCH;
  // state
  lnu::StateArgs sa{};
  sa.L = s->L;
  sa.H = static_cast<int>(s->H);
  sa.g = g;
  sa.use_pe = t->use_pe;
  sa.nrows = nr;
  // the state pass walks the same token chunks in 64-token stages
  sa.ntiles = static_cast<int>(ceil_div(s->L, lnu::SR));
  sa.tiles_per_cta = tpc * (lnu::M / lnu::SR);
  sa.nchunks = nch;
  sa.tables = tab;
  sa.partial = partial;
  sa.phi_t = phi_t;
  const int ssm = lnu::StateLay::bytes(t->grid_t);
  if (cudaFuncSetAttribute(lnu::linear_state_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm) != cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  lnu::linear_state_kernel<<<dim3(nch, static_cast<unsigned>(BH)), lnu::kStateThreads, ssm, st>>>(mk, mv, mxy, sa);
  if (int e = launch_status()) return e;
  const int rsm = t->grid_t * (lnu::D + 8) * 8;
  if (rsm > 48 * 1024 && cudaFuncSetAttribute(lnu::linear_reduce_image_kernel,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, rsm) != cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  lnu::linear_phi_sum_kernel<<<dim3(static_cast<unsigned>(BH), static_cast<unsigned>(t->grid_t)), lnu::D, 0, st>>>(
      phi_t, nch, t->grid_t, phi_tot);
  if (int e = launch_status()) return e;
  lnu::linear_reduce_image_kernel<<<dim3(static_cast<unsigned>(BH), lnu::D / 8), 256, rsm, st>>>(
      partial, phi_tot, nch, t->grid_t, static_cast<int>(s->H), t->use_pe ? reinterpret_cast<const float*>(tab + ly.tf)
                                                                        : nullptr,
      nr, 1.0 / static_cast<double>(s->L), bimg, state);
  if (int e = launch_status()) return e;
  // apply
  lnu::ApplyArgs aa{};
  aa.L = s->L;
  aa.H = static_cast<int>(s->H);
  aa.g = g;
  aa.use_pe = t->use_pe;
  aa.nrows = nr;
  aa.ntiles = ntiles;
  aa.tiles_per_cta = tpc;
  aa.tables = tab;
  aa.bimg = bimg;
  aa.rms_lr = rms_lowrank;
  aa.eps = eps;
  aa.y_lr = static_cast<__nv_bfloat16*>(y_lr);
  aa.o_lr = o_lr;
  const int asm_ = lnu::ApplyLay::bytes(nr);
  if (cudaFuncSetAttribute(lnu::linear_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, asm_) != cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  lnu::linear_apply_kernel<<<dim3(nch, static_cast<unsigned>(BH)), lnu::kApplyThreads, asm_, st>>>(mq, aa);
  if (int e = launch_status()) return e;
  // gate
  if (g_logit != nullptr) {
    const int64_t BL = s->B * s->L;
    lnu::linear_gate_kernel<<<static_cast<unsigned>(ceil_div(BL, 8)), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(t->x), t->x_row_stride, t->w_g + t->head_offset * s->d, s->H * s->d, BL,
        s->L, g, t->use_pe ? G : nullptr, g_logit);
    if (int e = launch_status()) return e;
    return scan_nonfinite(g_logit, false, BL, t->nonfinite, ROPESLR_NONFINITE_X, st);
  }
  return ROPESLR_OK;
}
