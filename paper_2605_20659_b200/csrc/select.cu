// K1: block routing of the RoPeSLR sparse branch.
//
// Restates mechanism.py:305-320 (+ the attended-pair count of :326) for flat,
// possibly ragged blocks on the GPU:
//   pool      mean of each block's Q and K rows, accumulated in float64
//             (mechanism.py:306-308).  Sums of <= block bf16/f32 values are
//             exact in float64 for realistic data, so the pooled means match
//             the NumPy oracle bit for bit before the division by the count.
//   scores    (pooled_q @ pooled_k^T) / sqrt(d) in float64 (mechanism.py:309).
//   select    stable descending order of the block softmax (ties -> lower
//             block index, mechanism.py:317), then top-k or count_for_mass
//             (decomposition.py:105-111); emits the ascending index list the
//             attention kernel walks (mechanism.py:321 `sorted(chosen)`).
// All three are HBM/L2-bound; see DESIGN.md for the byte counts.
#include <cuda_runtime.h>
#include <math.h>

#include <stdlib.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace ropeslr {

// exp(x) of a float64 is 0 below this: a block whose score is that far below
// the row max has probability 0 in the reference (mechanism.py:310-311), and
// all such blocks tie in its stable order (mechanism.py:317)
constexpr double kProbUnderflow = -745.1332191019412;

// grid (nb, B*H, 2): z = 0 pools Q, z = 1 pools K.  pooled: [2][BH][nb][d].
template <typename T>
__global__ void __launch_bounds__(256) pool_blocks_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                          double* __restrict__ pooled, int64_t L, int d, int block,
                                                          int nb, int64_t BH, int64_t bh0) {
  extern __shared__ double sred[];
  const int64_t bh = bh0 + blockIdx.y;
  const T* src = (blockIdx.z == 0 ? q : k) + bh * L * d;
  const int b = blockIdx.x;
  const int rows = block_size(L, block, b);
  const int64_t r0 = static_cast<int64_t>(b) * block;
  const int chunks = d / 8;
  const int lanes_r = blockDim.x / chunks;
  const int tid = threadIdx.x;
  const int ch = tid % chunks;
  const int rr = tid / chunks;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  if (rr < lanes_r) {
    // four row loads in flight per thread (bf16 sums of <= 128 values are
    // exact in float64, so the order does not matter)
    int r = rr;
    for (; r + 3 * lanes_r < rows; r += 4 * lanes_r) {
      float v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) load8(src + (r0 + r + u * lanes_r) * d + ch * 8, v[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(v[u][i]);
    }
    for (; r < rows; r += lanes_r) {
      float v[8];
      load8(src + (r0 + r) * d + ch * 8, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(v[i]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) sred[rr * d + ch * 8 + i] = acc[i];
  }
  __syncthreads();
  double* dst = pooled + ((static_cast<int64_t>(blockIdx.z) * BH + bh) * nb + b) * d;
  for (int c = tid; c < d; c += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < lanes_r; ++j) s += sred[j * d + c];
    dst[c] = s / static_cast<double>(rows);
  }
}

// The same pooling for bf16 rows of d = 128 and blocks of <= 128 rows: the
// block's rows are one contiguous run of <= 32 KiB, fetched by a single bulk
// copy into shared memory (so the bytes in flight do not depend on register
// occupancy), then summed in float64 from there.  256 threads: column chunk
// c = t % 16 (8 columns), rows t / 16 + 16 i.
__global__ void __launch_bounds__(256) pool_blocks_bulk_kernel(const __nv_bfloat16* __restrict__ q,
                                                               const __nv_bfloat16* __restrict__ k,
                                                               double* __restrict__ pooled, int64_t L, int block,
                                                               int nb, int64_t BH, int64_t bh0) {
  constexpr int D = 128;
  __shared__ __align__(128) uint8_t buf[128 * D * 2];  // the block's rows; then the f64 partial sums
  __shared__ uint64_t bar;
  const int64_t bh = bh0 + blockIdx.y;
  const __nv_bfloat16* src = (blockIdx.z == 0 ? q : k) + bh * L * D;
  const int b = blockIdx.x;
  const int rows = block_size(L, block, b);
  const int tid = threadIdx.x;
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t bytes = static_cast<uint32_t>(rows) * D * 2;
    sm100::mbar_arrive_expect_tx(&bar, bytes);
    sm100::bulk_load_1d(buf, src + static_cast<int64_t>(b) * block * D, bytes, &bar, sm100::policy_evict_first());
  }
  sm100::mbar_wait(&bar, 0);
  const int ch = tid & 15, rr = tid >> 4;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  for (int r = rr; r < rows; r += 16) {
    const uint4 u = *reinterpret_cast<const uint4*>(buf + (r * D + ch * 8) * 2);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      acc[2 * e] += static_cast<double>(f.x);
      acc[2 * e + 1] += static_cast<double>(f.y);
    }
  }
  __syncthreads();  // every row has been read: buf now holds the partial sums
  double* sred = reinterpret_cast<double*>(buf);  // [16 row lanes][128]
#pragma unroll
  for (int i = 0; i < 8; ++i) sred[rr * D + ch * 8 + i] = acc[i];
  __syncthreads();
  if (tid < D) {
    double s = 0.0;
    for (int j = 0; j < 16; ++j) s += sred[j * D + tid];
    pooled[((static_cast<int64_t>(blockIdx.z) * BH + bh) * nb + b) * D + tid] = s / static_cast<double>(rows);
  }
}

// scores[bh, i, j] = dot(pooled_q[bh, i], pooled_k[bh, j]) / sqrt(d), float64.
// 64x64 output tile per CTA, 4x4 per thread, k-chunks of 16 staged in smem.
__global__ void __launch_bounds__(256) block_scores_kernel(const double* __restrict__ pooled, double* __restrict__ scores,
                                                           int nb, int d, int64_t BH, double sqrt_d, int64_t bh0) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int64_t bh = bh0 + blockIdx.z;
  const double* pq = pooled + bh * nb * d;
  const double* pk = pooled + (BH + bh) * nb * d;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < d; k0 += 16) {
    for (int e = tid; e < 64 * 16; e += 256) {
      int r = e / 16, c = e % 16;
      int gi = i0 + r, gj = j0 + r, gc = k0 + c;
      As[c][r] = (gi < nb && gc < d) ? pq[static_cast<int64_t>(gi) * d + gc] : 0.0;
      Bs[c][r] = (gj < nb && gc < d) ? pk[static_cast<int64_t>(gj) * d + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[c][ty + 16 * u];
        b[u] = Bs[c][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  double* out = scores + bh * nb * nb;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int gi = i0 + ty + 16 * u;
    if (gi >= nb) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int gj = j0 + tx + 16 * v;
      if (gj < nb) out[static_cast<int64_t>(gi) * nb + gj] = acc[u][v] / sqrt_d;
    }
  }
}

// The same scores on the FP64 tensor cores (DMMA m8n8k4): 64x64 output tile
// per CTA, four warps of 32x32 (4x4 DMMA tiles each), k-chunks of 32 staged
// in shared memory.  Products and sums are IEEE float64 like the CUDA-core
// kernel (only the summation order differs, ~1 ulp: the top-k margins at
// configs 1-3 are >= 1e-9 relative).
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) block_scores_dmma_kernel(const double* __restrict__ pooled,
                                                                double* __restrict__ scores, int nb, int d,
                                                                int64_t BH, double sqrt_d, int64_t bh0) {
  constexpr int KC = 32;
  __shared__ double As[KC][64 + 1];
  __shared__ double Bs[KC][64 + 1];
  const int64_t bh = bh0 + blockIdx.z;
  const double* pq = pooled + bh * nb * d;
  const double* pk = pooled + (BH + bh) * nb * d;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;  // warp tile origin
  const int g = lane >> 2, t4 = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int k0 = 0; k0 < d; k0 += KC) {
    for (int e = tid; e < 64 * KC; e += 128) {
      const int r = e / KC, c = e % KC;
      const int gi = i0 + r, gj = j0 + r, gc = k0 + c;
      As[c][r] = (gi < nb && gc < d) ? pq[static_cast<int64_t>(gi) * d + gc] : 0.0;
      Bs[c][r] = (gj < nb && gc < d) ? pk[static_cast<int64_t>(gj) * d + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) a[m] = As[kk + t4][wr + 8 * m + g];
#pragma unroll
      for (int n = 0; n < 4; ++n) b[n] = Bs[kk + t4][wc + 8 * n + g];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[m][n], a[m], b[n]);
    }
    __syncthreads();
  }
  double* out = scores + bh * nb * nb;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int gi = i0 + wr + 8 * m + g;
    if (gi >= nb) continue;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gj = j0 + wc + 8 * n + 2 * t4 + e;
        if (gj < nb) out[static_cast<int64_t>(gi) * nb + gj] = acc[m][n][e] / sqrt_d;
      }
  }
}

// The same DMMA tiling with the pooled rows staged row-major by cp.async in
// a 3-stage ring of 16-wide k-chunks (d % 16 == 0), so the loads of chunk
// c + 2 overlap the DMMAs of chunk c.  Row pitch 20 doubles (160 B): the
// 8 rows x 4 k of one fragment load fall into two 128-byte wavefronts, the
// minimum for 256 bytes.  Same products and per-k accumulation order as
// block_scores_dmma_kernel.
namespace sc {
#ifndef ROPESLR_SC_ST
#define ROPESLR_SC_ST 2
#endif
#ifndef ROPESLR_SC_KC
#define ROPESLR_SC_KC 16
#endif
constexpr int KC = ROPESLR_SC_KC, PITCH = KC + 4, ST = ROPESLR_SC_ST, TILE = 64;
constexpr int STAGE_DOUBLES = 2 * TILE * PITCH;  // A then B
__device__ __forceinline__ void cp16(double* dst, const double* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
}  // namespace sc

__global__ void __launch_bounds__(128) block_scores_dmma_pipe_kernel(const double* __restrict__ pooled,
                                                                     double* __restrict__ scores, int nb, int d,
                                                                     int64_t BH, double sqrt_d, int64_t bh0) {
  using namespace sc;
  extern __shared__ __align__(16) double sbuf[];  // ST stages of [A 64 x PITCH | B 64 x PITCH]
  const int64_t bh = bh0 + blockIdx.z;
  const double* pq = pooled + bh * nb * d;
  const double* pk = pooled + (BH + bh) * nb * d;
  const int i0 = blockIdx.y * TILE, j0 = blockIdx.x * TILE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
  const int g = lane >> 2, t4 = lane & 3;
  const int nchunks = d / KC;
  auto load = [&](int c) {
    double* st = sbuf + (c % ST) * STAGE_DOUBLES;
    // 64 rows x KC/2 16-byte pieces per operand
    constexpr int PR = KC / 2, PIECES = 2 * TILE * PR;
#pragma unroll
    for (int it = 0; it < PIECES / 128; ++it) {
      const int e = tid + it * 128;
      const int op = e / (TILE * PR), r = (e / PR) % TILE, piece = e % PR;
      const int grow = (op == 0 ? i0 : j0) + r;
      const bool valid = grow < nb;
      const double* src = (op == 0 ? pq : pk) + static_cast<int64_t>(valid ? grow : 0) * d + c * KC + piece * 2;
      cp16(st + op * TILE * PITCH + r * PITCH + piece * 2, src, valid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int c = 0; c < ST - 1 && c < nchunks; ++c) load(c);
  for (int c = 0; c < nchunks; ++c) {
    if (c + ST - 2 < nchunks - 1)
      asm volatile("cp.async.wait_group %0;" ::"n"(ST - 2) : "memory");
    else
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // chunk c landed for every thread; chunk c - 1's stage is free
    if (c + ST - 1 < nchunks) load(c + ST - 1);
    const double* As = sbuf + (c % ST) * STAGE_DOUBLES;
    const double* Bs = As + TILE * PITCH;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) a[m] = As[(wr + 8 * m + g) * PITCH + kk + t4];
#pragma unroll
      for (int n = 0; n < 4; ++n) b[n] = Bs[(wc + 8 * n + g) * PITCH + kk + t4];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[m][n], a[m], b[n]);
    }
  }
  double* out = scores + bh * nb * nb;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int gi = i0 + wr + 8 * m + g;
    if (gi >= nb) continue;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gj = j0 + wc + 8 * n + 2 * t4 + e;
        if (gj < nb) out[static_cast<int64_t>(gi) * nb + gj] = acc[m][n][e] / sqrt_d;
      }
  }
}

// Order-preserving map double -> uint64, inverted so that an ascending sort
// yields descending scores.  +0 and -0 compare equal in the reference's
// softmax, so -0 is folded onto +0 to keep the lower-index tie rule.
__device__ __forceinline__ uint64_t desc_key(double s) {
  if (s == 0.0) s = 0.0;
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(s));
  uint64_t asc = (u >> 63) ? ~u : (u | (1ull << 63));
  return ~asc;
}

// One CTA per (bh, query block) row.
__global__ void __launch_bounds__(256) select_rows_kernel(const double* __restrict__ scores, int nb, int n2,
                                                          int64_t L, int block, int topk, double keep, int kmax,
                                                          int32_t* __restrict__ idx, int32_t* __restrict__ cnt,
                                                          uint8_t* __restrict__ mask,
                                                          unsigned long long* __restrict__ attended) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* ids = reinterpret_cast<uint32_t*>(keys + n2);
  int* flags = reinterpret_cast<int*>(ids + n2);
  __shared__ int s_nkeep;
  __shared__ double s_red[8];

  const int64_t row = blockIdx.x;  // bh * nb + qb
  const int64_t bh = row / nb;
  const int qb = static_cast<int>(row % nb);
  const double* srow = scores + row * nb;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // row max: scores below max + kProbUnderflow have probability 0 and tie
  __shared__ double s_max;
  {
    double m = -INFINITY;
    for (int i = tid; i < nb; i += blockDim.x) m = fmax(m, srow[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    if (tid == 0) {
      double t = s_red[0];
      for (int w = 1; w < (int)(blockDim.x / 32); ++w) t = fmax(t, s_red[w]);
      s_max = t;
    }
    __syncthreads();
  }
  const double row_max = s_max;
  for (int i = tid; i < n2; i += blockDim.x) {
    if (i < nb) {
      const double v = srow[i];
      keys[i] = desc_key(v - row_max < kProbUnderflow ? -INFINITY : v);
      ids[i] = static_cast<uint32_t>(i);
    } else {
      keys[i] = ~0ull;
      ids[i] = 0xFFFFFFFFu;
    }
  }
  for (int i = tid; i < nb; i += blockDim.x) flags[i] = 0;
  __syncthreads();

  // bitonic sort ascending on (key, id): stable descending order of scores
  for (int kk = 2; kk <= n2; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < n2; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          uint64_t ka = keys[i], kb = keys[ixj];
          uint32_t ia = ids[i], ib = ids[ixj];
          bool a_gt_b = (ka > kb) || (ka == kb && ia > ib);
          bool up = (i & kk) == 0;
          if (a_gt_b == up) {
            keys[i] = kb;
            keys[ixj] = ka;
            ids[i] = ib;
            ids[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  }

  if (topk > 0) {
    if (tid == 0) s_nkeep = topk < nb ? topk : nb;
  } else {
    // cumulative-mass rule on the block softmax (mechanism.py:310-311, 318)
    const double smax = srow[ids[0]];
    double part = 0.0;
    for (int i = tid; i < nb; i += blockDim.x) part += exp(srow[i] - smax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) s_red[warp] = part;
    __syncthreads();
    if (warp == 0) {
      double sum = 0.0;
      for (int w = 0; w < (int)(blockDim.x / 32); ++w) sum += s_red[w];
      double carry = 0.0;
      int found = nb;
      const double target = keep - kMassSlack;
      for (int base = 0; base < nb; base += 32) {
        int i = base + lane;
        double p = (i < nb) ? exp(srow[ids[i]] - smax) / sum : 0.0;
        // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          double t = __shfl_up_sync(0xffffffffu, p, o);
          if (lane >= o) p += t;
        }
        double c = carry + p;
        unsigned bal = __ballot_sync(0xffffffffu, (i < nb) && (c >= target));
        if (bal) {
          found = base + __ffs(bal);  // count = position + 1
          break;
        }
        carry += __shfl_sync(0xffffffffu, p, 31);
      }
      if (lane == 0) s_nkeep = found;
    }
  }
  __syncthreads();
  const int nkeep = s_nkeep;
  for (int i = tid; i < nkeep; i += blockDim.x) flags[ids[i]] = 1;
  __syncthreads();

  if (mask != nullptr) {
    uint8_t* mrow = mask + row * nb;
    for (int i = tid; i < nb; i += blockDim.x) mrow[i] = static_cast<uint8_t>(flags[i]);
  }
  if (warp == 0) {
    int32_t* irow = idx + row * kmax;
    int carry = 0;
    long long ksum = 0;
    for (int base = 0; base < nb; base += 32) {
      int i = base + lane;
      int f = (i < nb) ? flags[i] : 0;
      unsigned bal = __ballot_sync(0xffffffffu, f);
      int pos = carry + __popc(bal & ((1u << lane) - 1u));
      if (f) {
        irow[pos] = i;
        ksum += block_size(L, block, i);
      }
      carry += __popc(bal);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
    if (lane == 0) {
      cnt[row] = nkeep;
      atomicAdd(attended + bh, static_cast<unsigned long long>(ksum * block_size(L, block, qb)));
    }
  }
}

// Top-k rows, one warp per (bh, query block) row, nb <= 32 * NPER.
// MSB-first radix select (8-bit digits) on the order-preserving keys finds
// the k-th best key T; rows keep every key < T and, on exact ties at T, the
// lowest block indices (the stable order of mechanism.py:317).  The keys
// stay in registers; each warp owns a 256-bin histogram in shared memory.
// The radix select and the outputs of one row, from its keys (registers).
template <int NPER>
__device__ __forceinline__ void topk_row(uint64_t (&key)[NPER], int* hist, int lane, int nb, int64_t row, int64_t L, int block, int topk, int kmax, int32_t* __restrict__ idx, int32_t* __restrict__ cnt, uint8_t* __restrict__ mask, unsigned long long* __restrict__ attended) {
  const int64_t bh = row / nb;
  const int qb = static_cast<int>(row % nb);
  int need = topk < nb ? topk : nb;
  uint64_t prefix = 0, pmask = 0;
  bool exact = false;  // the remaining bucket is taken whole
#pragma unroll 1
  for (int shift = 56; shift >= 0; shift -= 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NPER; ++i)
      if ((key[i] & pmask) == prefix && lane + 32 * i < nb) atomicAdd(&hist[(key[i] >> shift) & 255], 1);
    __syncwarp();
    int h8[8];
    int tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      h8[i] = hist[lane * 8 + i];
      tot += h8[i];
    }
    int incl = tot;  // inclusive scan of lane totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int excl = incl - tot;
    // the bucket where the running count first reaches `need`
    const unsigned owner = __ballot_sync(0xffffffffu, excl < need && incl >= need);
    const int src = __ffs(owner) - 1;
    int bucket = 0, before = 0, cnt_b = 0;
    if (lane == src) {
      int run = excl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (run + h8[i] >= need) {
          bucket = lane * 8 + i;
          before = run;
          cnt_b = h8[i];
          break;
        }
        run += h8[i];
      }
    }
    bucket = __shfl_sync(0xffffffffu, bucket, src);
    before = __shfl_sync(0xffffffffu, before, src);
    cnt_b = __shfl_sync(0xffffffffu, cnt_b, src);
    need -= before;
    prefix |= static_cast<uint64_t>(bucket) << shift;
    pmask |= 255ull << shift;
    __syncwarp();
    if (cnt_b == need) {
      exact = true;
      break;
    }
  }
  // selected: masked key below the prefix, or inside the final bucket (whole,
  // or its `need` lowest-index members on exact ties)
  bool sel[NPER];
  int taken = 0;
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const bool valid = lane + 32 * i < nb;
    const uint64_t km = key[i] & pmask;
    bool s = valid && km < prefix;
    const bool tie = valid && km == prefix;
    if (exact) {
      s = s || tie;
    } else {
      const unsigned bal = __ballot_sync(0xffffffffu, tie);
      const int pos = taken + __popc(bal & ((1u << lane) - 1u));
      s = s || (tie && pos < need);
      taken += __popc(bal);
    }
    sel[i] = s;
  }
  int32_t* irow = idx + row * kmax;
  uint8_t* mrow = mask ? mask + row * nb : nullptr;
  int carry = 0;
  long long ksum = 0;
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int c = lane + 32 * i;
    const unsigned bal = __ballot_sync(0xffffffffu, sel[i]);
    if (sel[i]) {
      irow[carry + __popc(bal & ((1u << lane) - 1u))] = c;
      ksum += block_size(L, block, c);
    }
    if (mrow && c < nb) mrow[c] = sel[i] ? 1 : 0;
    carry += __popc(bal);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
  if (lane == 0) {
    cnt[row] = carry;
    atomicAdd(attended + bh, static_cast<unsigned long long>(ksum * block_size(L, block, qb)));
  }
}

// A row spanning more than the float64 exp range: keys of columns whose block
// probability underflows (score more than kProbUnderflow below the row max)
// become the key of -inf, so they tie and go by block index.  Out of line:
// such rows are rare, and the common path keeps its registers.
template <int NPER>
__device__ __noinline__ void topk_row_clamped(const double* srow, double row_max, int* hist, int lane, int nb, int64_t row, int64_t L, int block, int topk, int kmax, int32_t* __restrict__ idx, int32_t* __restrict__ cnt, uint8_t* __restrict__ mask, unsigned long long* __restrict__ attended) {
  uint64_t key[NPER];
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int c = lane + 32 * i;
    const double v = c < nb ? srow[c] : 0.0;
    key[i] = c < nb ? desc_key(v - row_max < kProbUnderflow ? -INFINITY : v) : ~0ull;
  }
  topk_row<NPER>(key, hist, lane, nb, row, L, block, topk, kmax, idx, cnt, mask, attended);
}

template <int NPER>
__global__ void __launch_bounds__(256) select_topk_warp_kernel(const double* __restrict__ scores, int nb,
                                                               int64_t rows, int64_t L, int block, int topk, int kmax,
                                                               int32_t* __restrict__ idx, int32_t* __restrict__ cnt,
                                                               uint8_t* __restrict__ mask,
                                                               unsigned long long* __restrict__ attended) {
  __shared__ int hist_all[8][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (row >= rows) return;
  int* hist = hist_all[warp];
  const double* srow = scores + row * nb;
  // the reference orders blocks by their softmax probability (mechanism.py:
  // 310-317): scores more than kProbUnderflow below the row max have
  // probability 0 and tie (lower block index first), so they key as -inf
  uint64_t key[NPER];
  // the row max and min as ascending keys (~desc_key); invalid columns hold
  // ~0 descending keys = ascending 0, which never wins the max
  uint64_t kmax_key = 0, kmin_key = ~0ull;
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int c = lane + 32 * i;
    key[i] = c < nb ? desc_key(srow[c]) : ~0ull;
    kmax_key = max(kmax_key, ~key[i]);
    if (c < nb) kmin_key = min(kmin_key, ~key[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmax_key = max(kmax_key, __shfl_xor_sync(0xffffffffu, kmax_key, o));
    kmin_key = min(kmin_key, __shfl_xor_sync(0xffffffffu, kmin_key, o));
  }
  // invert the ascending map of desc_key
  auto value_of = [](uint64_t a) {
    return __longlong_as_double(static_cast<long long>((a >> 63) ? (a & ~(1ull << 63)) : ~a));
  };
  const double row_max = value_of(kmax_key);
  // only a row spanning more than the float64 exp range has underflowed probabilities
  if (row_max > -INFINITY && value_of(kmin_key) - row_max < kProbUnderflow) {
    topk_row_clamped<NPER>(srow, row_max, hist, lane, nb, row, L, block, topk, kmax, idx, cnt, mask, attended);
    return;
  }
  topk_row<NPER>(key, hist, lane, nb, row, L, block, topk, kmax, idx, cnt, mask, attended);
}

}  // namespace ropeslr

using namespace ropeslr;

static int next_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

static int check_select(const ropeslr_shape* s, const ropeslr_select_params* sel, int32_t kmax, const int32_t* idx,
                        const int32_t* cnt, const int64_t* attended) {
  if (s == nullptr || sel == nullptr) return ROPESLR_ERR_NULL;
  if (s->B < 1 || s->H < 1 || s->L < 1 || s->block < 1) return ROPESLR_ERR_SHAPE;
  if (s->d < 8 || s->d > 256 || s->d % 8) return ROPESLR_ERR_SHAPE;
  if (s->dtype != ROPESLR_F32 && s->dtype != ROPESLR_BF16) return ROPESLR_ERR_DTYPE;
  if (!idx || !cnt || !attended) return ROPESLR_ERR_NULL;
  const int64_t nb64 = ceil_div(s->L, s->block);
  if (nb64 > 8192) return ROPESLR_ERR_SHAPE;
  const int nb = static_cast<int>(nb64);
  if (sel->topk < 0) return ROPESLR_ERR_VALUE;
  if (sel->topk == 0 && !(sel->keep > 0.0 && sel->keep <= 1.0)) return ROPESLR_ERR_VALUE;
  const int need = sel->topk > 0 ? (sel->topk < nb ? sel->topk : nb) : nb;
  if (kmax < need) return ROPESLR_ERR_SHAPE;
  return ROPESLR_OK;
}

static size_t pooled_bytes(const ropeslr_shape* s) {
  const int64_t nb = ceil_div(s->L, s->block);
  return ((static_cast<size_t>(2 * s->B * s->H * nb * s->d) * sizeof(double) + 255) / 256) * 256;
}

static size_t scores_bytes(const ropeslr_shape* s) {
  const int64_t nb = ceil_div(s->L, s->block);
  return ((static_cast<size_t>(s->B * s->H * nb * nb) * sizeof(double) + 255) / 256) * 256;
}

// Scores of heads [bh0, bh1) from the pooled means.
static int launch_scores(const double* pooled, double* scores, int nb, int d, int64_t BH, int64_t bh0, int64_t bh1,
                         cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(ceil_div(nb, 64)), static_cast<unsigned>(ceil_div(nb, 64)),
            static_cast<unsigned>(bh1 - bh0));
  const double sq = sqrt(static_cast<double>(d));
  // scores = 'f': the CUDA-core kernel, 'd': the unpipelined DMMA kernel (A/B timing)
  const char e = tuning().scores;
  if (e == 'f') {
    block_scores_kernel<<<grid, 256, 0, st>>>(pooled, scores, nb, d, BH, sq, bh0);
  } else if (d % sc::KC == 0 && e != 'd') {
    // opt in above 48 KiB of dynamic shared memory on every call (per-device attribute)
    if (cudaFuncSetAttribute(block_scores_dmma_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             sc::ST * sc::STAGE_DOUBLES * static_cast<int>(sizeof(double))) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    block_scores_dmma_pipe_kernel<<<grid, 128, sc::ST * sc::STAGE_DOUBLES * sizeof(double), st>>>(
        pooled, scores, nb, d, BH, sq, bh0);
  } else {
    block_scores_dmma_kernel<<<grid, 128, 0, st>>>(pooled, scores, nb, d, BH, sq, bh0);
  }
  return launch_status();
}

// Selection of the rows of heads [bh0, bh1).
static int launch_select(const ropeslr_shape* s, const ropeslr_select_params* sel, const double* scores, int32_t* idx,
                         int32_t kmax, int32_t* cnt, uint8_t* mask, int64_t* attended, int64_t bh0, int64_t bh1,
                         cudaStream_t st) {
  const int nb = static_cast<int>(ceil_div(s->L, s->block));
  auto* att = reinterpret_cast<unsigned long long*>(attended);
  const int64_t row0 = bh0 * nb, row1 = bh1 * nb;
  if (sel->topk > 0 && nb <= 1024) {
    const int64_t off = row0, rows = row1 - row0;
    const unsigned grid = static_cast<unsigned>(ceil_div(rows, 8));
#define ROPESLR_SEL_CASE(NPER_)                                                                            \
  select_topk_warp_kernel<NPER_><<<grid, 256, 0, st>>>(scores + off * nb, nb, rows, s->L, s->block, sel->topk, \
                                                        kmax, idx + off * kmax, cnt + off,                    \
                                                        mask ? mask + off * nb : nullptr, att + bh0)
    if (nb <= 128)
      ROPESLR_SEL_CASE(4);
    else if (nb <= 256)
      ROPESLR_SEL_CASE(8);
    else if (nb <= 512)
      ROPESLR_SEL_CASE(16);
    else
      ROPESLR_SEL_CASE(32);
#undef ROPESLR_SEL_CASE
    return launch_status();
  }
  const int n2 = next_pow2(nb);
  size_t sm = static_cast<size_t>(n2) * (sizeof(uint64_t) + sizeof(uint32_t)) + static_cast<size_t>(nb) * sizeof(int);
  static_assert(sizeof(unsigned long long) == sizeof(int64_t), "int64 atomics");
  if (sm > 48 * 1024) {
    if (cudaFuncSetAttribute(select_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm)) != cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
  }
  // select_rows_kernel takes the absolute row from blockIdx.x: offset the pointers of the head range instead
  const int64_t off = row0;
  select_rows_kernel<<<static_cast<unsigned>(row1 - row0), 256, sm, st>>>(
      scores + off * nb, nb, n2, s->L, s->block, sel->topk, sel->keep, kmax, idx + off * kmax, cnt + off,
      mask ? mask + off * nb : nullptr, att + bh0);
  return launch_status();
}

// Scores from the pooled means, then top-k / cumulative-mass selection.
static int select_from_pooled(const ropeslr_shape* s, const ropeslr_select_params* sel, const double* pooled,
                              int32_t* idx, int32_t kmax, int32_t* cnt, uint8_t* mask, int64_t* attended,
                              double* scores, cudaStream_t st) {
  const int64_t BH = s->B * s->H;
  const int d = static_cast<int>(s->d);
  const int nb = static_cast<int>(ceil_div(s->L, s->block));
  if (cudaMemsetAsync(attended, 0, sizeof(int64_t) * BH, st) != cudaSuccess) return ROPESLR_ERR_LAUNCH;
  if (int e = scan_nonfinite(pooled, true, 2 * BH * nb * d, sel->nonfinite, ROPESLR_NONFINITE_QK, st)) return e;
  if (int e = launch_scores(pooled, scores, nb, d, BH, 0, BH, st)) return e;
  return launch_select(s, sel, scores, idx, kmax, cnt, mask, attended, 0, BH, st);
}

static int launch_pool(const ropeslr_shape* s, const void* q, const void* k, double* pooled, int64_t bh0, int64_t bh1,
                       cudaStream_t st) {
  const int64_t BH = s->B * s->H;
  const int d = static_cast<int>(s->d);
  const int nb = static_cast<int>(ceil_div(s->L, s->block));
  dim3 grid(nb, static_cast<unsigned>(bh1 - bh0), 2);
  const int chunks = d / 8;
  const int lanes_r = 256 / chunks;
  size_t sm = static_cast<size_t>(lanes_r) * d * sizeof(double);
  if (s->dtype == ROPESLR_BF16 && d == 128 && s->block <= 128 && aligned16(q) && aligned16(k))
    pool_blocks_bulk_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(q),
                                                   static_cast<const __nv_bfloat16*>(k), pooled, s->L, s->block, nb,
                                                   BH, bh0);
  else if (s->dtype == ROPESLR_BF16)
    pool_blocks_kernel<__nv_bfloat16><<<grid, 256, sm, st>>>(static_cast<const __nv_bfloat16*>(q),
                                                              static_cast<const __nv_bfloat16*>(k), pooled, s->L, d,
                                                              s->block, nb, BH, bh0);
  else
    pool_blocks_kernel<float><<<grid, 256, sm, st>>>(static_cast<const float*>(q), static_cast<const float*>(k),
                                                      pooled, s->L, d, s->block, nb, BH, bh0);
  return launch_status();
}

extern "C" size_t ropeslr_select_workspace_bytes(const ropeslr_shape* s) {
  if (s == nullptr || s->block <= 0) return 0;
  return pooled_bytes(s) + scores_bytes(s);
}

extern "C" size_t ropeslr_select_pooled_workspace_bytes(const ropeslr_shape* s) {
  if (s == nullptr || s->block <= 0) return 0;
  return scores_bytes(s);
}

extern "C" int ropeslr_select_blocks(const ropeslr_shape* s, const ropeslr_select_params* sel, const void* q,
                                     const void* k, int32_t* idx, int32_t kmax, int32_t* cnt, uint8_t* mask,
                                     int64_t* attended, double* scores_out, void* ws, size_t ws_bytes,
                                     void* stream_) {
  int stt = check_select(s, sel, kmax, idx, cnt, attended);
  if (stt) return stt;
  if (!q || !k) return ROPESLR_ERR_NULL;
  if (!aligned16(q) || !aligned16(k)) return ROPESLR_ERR_ALIGN;
  if (ws == nullptr || ws_bytes < ropeslr_select_workspace_bytes(s)) return ROPESLR_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  double* pooled = static_cast<double*>(ws);
  double* scores = scores_out ? scores_out : reinterpret_cast<double*>(static_cast<char*>(ws) + pooled_bytes(s));
  if (int e = launch_pool(s, q, k, pooled, 0, s->B * s->H, st)) return e;
  return select_from_pooled(s, sel, pooled, idx, kmax, cnt, mask, attended, scores, st);
}

extern "C" int ropeslr_select_from_pooled(const ropeslr_shape* s, const ropeslr_select_params* sel,
                                          const double* pooled, int32_t* idx, int32_t kmax, int32_t* cnt,
                                          uint8_t* mask, int64_t* attended, double* scores_out, void* ws,
                                          size_t ws_bytes, void* stream_) {
  int stt = check_select(s, sel, kmax, idx, cnt, attended);
  if (stt) return stt;
  if (!pooled) return ROPESLR_ERR_NULL;
  double* scores = scores_out;
  if (scores == nullptr) {
    if (ws == nullptr || ws_bytes < ropeslr_select_pooled_workspace_bytes(s)) return ROPESLR_ERR_WORKSPACE;
    scores = static_cast<double*>(ws);
  }
  return select_from_pooled(s, sel, pooled, idx, kmax, cnt, mask, attended, scores,
                            static_cast<cudaStream_t>(stream_));
}
