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
#include <algorithm>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cuda_bf16.h>
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
// With img != NULL it also writes the screening path's bf16 hi / lo image
// rows and the row norm (what screen_image_kernel does, without re-reading
// the means).
__global__ void __launch_bounds__(256) pool_blocks_bulk_kernel(const __nv_bfloat16* __restrict__ q,
                                                               const __nv_bfloat16* __restrict__ k,
                                                               double* __restrict__ pooled, int64_t L, int block,
                                                               int nb, int64_t BH, int64_t bh0,
                                                               uint8_t* __restrict__ img, float* __restrict__ norms,
                                                               int ntile) {
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
  __shared__ double nsq[4];
  if (tid < D) {
    double s = 0.0;
    for (int j = 0; j < 16; ++j) s += sred[j * D + tid];
    const double m = s / static_cast<double>(rows);
    pooled[((static_cast<int64_t>(blockIdx.z) * BH + bh) * nb + b) * D + tid] = m;
    if (img != nullptr) {
      constexpr int ATOM = 128 * 128, TILE = 2 * ATOM;
      const __nv_bfloat16 hi = __double2bfloat16(m);
      const __nv_bfloat16 lo = __double2bfloat16(m - static_cast<double>(__bfloat162float(hi)));
      const int atom = tid >> 6, ch = (tid & 63) >> 3, el = tid & 7, rr = b & 127, tile = b >> 7;
      const int64_t off = atom * ATOM + rr * 128 + ((ch ^ (rr & 7)) << 4) + el * 2;
      const int z = blockIdx.z;
      *reinterpret_cast<__nv_bfloat16*>(img + (((z * 2 + 0) * BH + bh) * ntile + tile) * TILE + off) = hi;
      *reinterpret_cast<__nv_bfloat16*>(img + (((z * 2 + 1) * BH + bh) * ntile + tile) * TILE + off) = lo;
      double q2 = m * m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) q2 += __shfl_xor_sync(0xffffffffu, q2, o);
      if ((tid & 31) == 0) nsq[tid >> 5] = q2;
    }
  }
  if (img != nullptr) {
    __syncthreads();
    if (tid == 0)
      norms[(static_cast<int64_t>(blockIdx.z) * BH + bh) * nb + b] =
          __double2float_ru(__dsqrt_ru(nsq[0] + nsq[1] + nsq[2] + nsq[3]));
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

// Cumulative-mass (`keep`) rows, one CTA per (bh, query block) row, nb <=
// 256 * IPT (mechanism.py:310-320, decomposition.py:105-111).  The same
// decisions as select_rows_kernel, from a cheaper sort: the row's scores are
// ordered by the top 24 bits of the float32 rounding of the score (order
// preserving and monotone: sign, exponent, 15 mantissa bits) with a stable
// radix sort (6 passes of 4 bits; the block index rides in the key's low
// bits); runs of equal keys -- float64 scores closer than 2^-15 relative,
// exact duplicates, the underflowed tail -- are then put in the exact order
// (float64 score, then lower block) by an insertion sort per run.  The probabilities exp(s - max) / sum follow in
// that order, their inclusive prefix sums (per-thread sequential, then a
// block scan) give the first position reaching keep - 1e-12; all reductions
// run in a fixed order, so the result is deterministic.
__device__ __forceinline__ uint32_t desc_key32(double s) {
  float f = __double2float_rn(s);  // monotone non-decreasing in s
  if (f == 0.f) f = 0.f;           // -0 -> +0 (the float64 key folds them too)
  const uint32_t u = __float_as_uint(f);
  const uint32_t asc = (u >> 31) ? ~u : (u | 0x80000000u);
  return ~asc;
}

// 128 threads x 8 keys per row: fewer barrier participants than 256 x 4
// (K1 at config 3: 0.98 vs 1.04 ms; 512 x 2: 1.45 ms; 64 x 16 spills).
constexpr int kKeepThreads = 128;

template <int T, int IPT>
__global__ void __launch_bounds__(T, 8) select_keep_kernel(const double* __restrict__ scores, int nb, int64_t L,
                                                          int block, double keep, int kmax,
                                                          int32_t* __restrict__ idx, int32_t* __restrict__ cnt,
                                                          uint8_t* __restrict__ mask,
                                                          unsigned long long* __restrict__ attended) {
  constexpr int N = T * IPT;
  using Sort = cub::BlockRadixSort<uint64_t, T, IPT, cub::NullType, 4>;
  using SortFull = cub::BlockRadixSort<uint64_t, T, IPT, int, 4>;  // long runs: the full float64 key
  using RedD = cub::BlockReduce<double, T>;
  using ScanD = cub::BlockScan<double, T>;
  using RedI = cub::BlockReduce<int, T>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename SortFull::TempStorage sort_full;
    typename RedD::TempStorage redd;
    typename ScanD::TempStorage scan;
    typename RedI::TempStorage redi;
  } tmp;
  __shared__ double s_sc[N];
  __shared__ uint32_t s_key[N];
  __shared__ int s_id[N];
  int* flags = reinterpret_cast<int*>(s_key);  // the float32 keys are dead once the runs are ordered
  __shared__ double s_bc;
  __shared__ int s_nkeep;

  const int64_t row = blockIdx.x;  // bh * nb + qb
  const int64_t bh = row / nb;
  const int qb = static_cast<int>(row % nb);
  const double* srow = scores + row * nb;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  double m = -INFINITY;
  for (int i = tid; i < nb; i += T) {
    const double v = srow[i];
    s_sc[i] = v;
    m = fmax(m, v);
  }
  m = RedD(tmp.redd).Reduce(m, cub::Max());
  if (tid == 0) s_bc = m;
  __syncthreads();
  const double row_max = s_bc;

  // sort keys: float32 score key (blocks below the underflow point tie at
  // -inf), then the block index; blocked arrangement = index order
  uint64_t keys[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = tid * IPT + k;
    if (i < nb) {
      const double v = s_sc[i];
      const uint32_t kk = desc_key32(v - row_max < kProbUnderflow ? -INFINITY : v);
      keys[k] = (static_cast<uint64_t>(kk) << 10) | static_cast<uint64_t>(i);
    } else {
      keys[k] = (1ull << 42) - 1;
    }
  }
  __syncthreads();  // tmp reuse
  Sort(tmp.sort).Sort(keys, 18, 42);  // stable: equal keys stay in block order
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int pos = tid * IPT + k;
    s_key[pos] = static_cast<uint32_t>(keys[k] >> 18);
    s_id[pos] = static_cast<int>(keys[k] & 1023u);
  }
  __syncthreads();
  // exact order inside runs of equal float32 keys: runs whose float64 keys
  // all agree are already in block order; other runs up to 32 long by an
  // insertion sort; a longer one sends the whole row through a radix sort
  // on the full float64 key (16 passes) instead of a quadratic sort
  auto key64 = [&](int i) {
    const double v = s_sc[i];
    return desc_key(v - row_max < kProbUnderflow ? -INFINITY : v);
  };
  int long_run = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int pos = tid * IPT + k;
    if (pos + 1 < nb && s_key[pos + 1] == s_key[pos] && (pos == 0 || s_key[pos - 1] != s_key[pos])) {
      const uint64_t k0 = key64(s_id[pos]);
      int end = pos + 1;
      bool same = true;
      while (end < nb && s_key[end] == s_key[pos]) {
        same = same && key64(s_id[end]) == k0;
        ++end;
      }
      if (same) continue;
      if (end - pos > 32) {
        long_run = 1;
        continue;
      }
      for (int a = pos + 1; a < end; ++a) {
        const int ia = s_id[a];
        const uint64_t ka = key64(ia);
        int b = a - 1;
        while (b >= pos) {
          const int ib = s_id[b];
          const uint64_t kb = key64(ib);
          if (kb < ka || (kb == ka && ib < ia)) break;
          s_id[b + 1] = ib;
          --b;
        }
        s_id[b + 1] = ia;
      }
    }
  }
  if (__syncthreads_or(long_run)) {
    uint64_t kf[IPT];
    int vf[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int i = tid * IPT + k;
      kf[k] = i < nb ? key64(i) : ~0ull;
      vf[k] = i;
    }
    SortFull(tmp.sort_full).Sort(kf, vf);  // stable: equal keys stay in block order
#pragma unroll
    for (int k = 0; k < IPT; ++k) s_id[tid * IPT + k] = vf[k];
  }
  __syncthreads();

  // probabilities in sorted order, their sum, the prefix sums
  double e[IPT];
  double part = 0.0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int pos = tid * IPT + k;
    e[k] = pos < nb ? exp(s_sc[s_id[pos]] - row_max) : 0.0;
    part += e[k];
  }
  const double total = RedD(tmp.redd).Sum(part);
  if (tid == 0) s_bc = total;
  __syncthreads();
  const double sum = s_bc;
  double c[IPT];
  double run = 0.0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    run += e[k] / sum;
    c[k] = run;
  }
  double excl;
  ScanD(tmp.scan).ExclusiveSum(run, excl);
  const double target = keep - kMassSlack;
  int first = nb;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int pos = tid * IPT + k;
    if (pos < nb && excl + c[k] >= target) {
      first = pos;
      break;
    }
  }
  __syncthreads();  // tmp reuse
  first = RedI(tmp.redi).Reduce(first, cub::Min());
  if (tid == 0) s_nkeep = first < nb ? first + 1 : nb;
  __syncthreads();
  const int nkeep = s_nkeep;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int pos = tid * IPT + k;
    if (pos < nb) flags[s_id[pos]] = pos < nkeep ? 1 : 0;
  }
  __syncthreads();

  if (mask != nullptr) {
    uint8_t* mrow = mask + row * nb;
    for (int i = tid; i < nb; i += T) mrow[i] = static_cast<uint8_t>(flags[i]);
  }
  if (warp == 0) {
    int32_t* irow = idx + row * kmax;
    int carry = 0;
    long long ksum = 0;
    for (int base = 0; base < nb; base += 32) {
      const int i = base + lane;
      const int f = (i < nb) ? flags[i] : 0;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      const int pos = carry + __popc(bal & ((1u << lane) - 1u));
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
// The outputs of one row from its selection bits (bit i: column lane +
// 32 i): ascending index list, count, optional mask, attended pairs of the
// head.
template <int NPER>
__device__ __forceinline__ void emit_bits(uint32_t bits, int lane, int nb, int64_t row, int64_t L, int block, int kmax, int32_t* __restrict__ idx, int32_t* __restrict__ cnt, uint8_t* __restrict__ mask, unsigned long long* __restrict__ attended) {
  const int64_t bh = row / nb;
  const int qb = static_cast<int>(row % nb);
  int32_t* irow = idx + row * kmax;
  uint8_t* mrow = mask ? mask + row * nb : nullptr;
  int carry = 0;
  long long ksum = 0;
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int c = lane + 32 * i;
    const bool s = (bits >> i) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, s);
    if (s) {
      irow[carry + __popc(bal & ((1u << lane) - 1u))] = c;
      ksum += block_size(L, block, c);
    }
    if (mrow && c < nb) mrow[c] = s ? 1 : 0;
    carry += __popc(bal);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
  if (lane == 0) {
    cnt[row] = carry;
    atomicAdd(attended + bh, static_cast<unsigned long long>(ksum * block_size(L, block, qb)));
  }
}

template <int NPER>
__device__ __forceinline__ void emit_row(const bool (&sel)[NPER], int lane, int nb, int64_t row, int64_t L, int block, int kmax, int32_t* __restrict__ idx, int32_t* __restrict__ cnt, uint8_t* __restrict__ mask, unsigned long long* __restrict__ attended) {
  uint32_t bits = 0;
#pragma unroll
  for (int i = 0; i < NPER; ++i) bits |= static_cast<uint32_t>(sel[i]) << i;
  emit_bits<NPER>(bits, lane, nb, row, L, block, kmax, idx, cnt, mask, attended);
}

template <int NPER>
__device__ __forceinline__ void topk_row(uint64_t (&key)[NPER], int* hist, int lane, int nb, int64_t row, int64_t L, int block, int topk, int kmax, int32_t* __restrict__ idx, int32_t* __restrict__ cnt, uint8_t* __restrict__ mask, unsigned long long* __restrict__ attended) {
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
  emit_row<NPER>(sel, lane, nb, row, L, block, kmax, idx, cnt, mask, attended);
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


// ---------------------------------------------------------------- screening
// Top-k with d = 128: the decision of mechanism.py:316-320 only depends on
// which blocks score above the k-th, so most of the nb^2 float64 dot
// products never matter.  The path:
//   screen_image_kernel   pooled float64 rows -> bf16 hi/lo splits (x = hi
//                         + lo + r, |r| <= 2^-16 |x|), written as the
//                         128B-swizzled K-major tiles the tensor cores read,
//                         plus an upward-rounded float norm per row (on the
//                         pooling path pool_blocks_bulk_kernel writes them)
//   screen_scores_kernel  s~ = (Qhi Khi^T + Qhi Klo^T + Qlo Khi^T) / sqrt(d)
//                         on tcgen05 (float32 accumulation in TMEM)
//   screen_select_kernel  per row: [lo, hi] around the k-th best s~, t_k,
//                         by counting probes (normal quantile, a Newton step,
//                         interpolation) until the count is exact or hi - lo
//                         <= E; with |s~ - s| <= E for every block of the
//                         row, blocks with s~ > hi + 2E are in, blocks with
//                         s~ < lo - 2E are out, and the few in between get
//                         float64 scores and the exact stable order
//   screen_exact_kernel   the rows the band cannot decide, wholly in float64.
// E = kScreenBound |q_i| max_j |k_j| / sqrt(d).  Derivation (DESIGN.md,
// K1): the dropped split terms are <= 3.1 * 2^-16 sum |q||k|; the float32
// accumulation of 3 d = 384 exact bf16 products, allowing each addition a
// relative error of 2^-22 (twice a truncating adder's), adds <= 383 *
// 2^-22 * 1.02 sum |q||k|; together 1.4e-4 |q||k| (Cauchy-Schwarz), under
// kScreenBound = 2^-12.  Proof that the band decides exactly: the k-th best
// exact score tau lies in [t_k - E, t_k + E], since k blocks have s >= s~ -
// E >= t_k - E and nb - k + 1 blocks have s <= t_k + E; so tau is in
// [lo - E, hi + E], a block with s~ > hi + 2E has s > hi + E >= tau and a
// block with s~ < lo - 2E has s < lo - E <= tau.  Every block with s >= tau
// outside the top set is therefore in the band, where the float64 order
// (ties to the lower block) picks the remaining k - |in|.
// Rows that are non-finite, span more than 700 (the probability underflow
// of mechanism.py:310-311 needs the float64 path) or hold more than
// kScreenBand blocks in the band are decided wholly in float64.
namespace scr {
constexpr int D = 128;
constexpr int ROWS = 128;              // rows of a tile
constexpr int ATOM = ROWS * 128;       // 16 KiB: 128 rows x 64 bf16, 128B-swizzled
constexpr int TILE = 2 * ATOM;         // 128 rows x 128 bf16 (one split)
constexpr double kScreenBound = 1.0 / 4096.0;
constexpr int kScreenBand = 32;
constexpr int EPI_WARPS = 8;
constexpr int SMEM = 1024 + 2 * TILE + 2 * 2 * TILE + EPI_WARPS * 32 * 33 * 4 + 16 * 8;  // 226.1 KiB
}  // namespace scr


// grid (ntile * 16, BH, 2), 256 threads: one warp per pooled row (z = 0: Q,
// 1: K); rows nb .. ntile*128 - 1 are written as zeros.  img:
// [z][hi/lo][BH][ntile][TILE].
__global__ void __launch_bounds__(256) screen_image_kernel(const double* __restrict__ pooled, int nb, int ntile,
                                                           int64_t BH, uint8_t* __restrict__ img,
                                                           float* __restrict__ norms) {
  using namespace scr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int z = blockIdx.z;
  const int64_t bh = blockIdx.y;
  const int r = blockIdx.x * 8 + warp;
  if (r >= ntile * ROWS) return;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  if (r < nb) {
    const double* src = pooled + ((z * BH + bh) * nb + r) * D + lane * 4;
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = src[e];
  }
  __nv_bfloat16 hi[4], lo[4];
  double ss = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    hi[e] = __double2bfloat16(v[e]);
    lo[e] = __double2bfloat16(v[e] - static_cast<double>(__bfloat162float(hi[e])));
    ss = fma(v[e], v[e], ss);
  }
  const int c0 = lane * 4, atom = c0 >> 6, ch = (c0 & 63) >> 3, el = c0 & 7;
  const int rr = r & (ROWS - 1), tile = r / ROWS;
  const int64_t off = static_cast<int64_t>(atom) * ATOM + rr * 128 + ((ch ^ (rr & 7)) << 4) + el * 2;
  uint8_t* base_hi = img + (((z * 2 + 0) * BH + bh) * ntile + tile) * TILE;
  uint8_t* base_lo = img + (((z * 2 + 1) * BH + bh) * ntile + tile) * TILE;
  *reinterpret_cast<uint2*>(base_hi + off) = *reinterpret_cast<const uint2*>(hi);
  *reinterpret_cast<uint2*>(base_lo + off) = *reinterpret_cast<const uint2*>(lo);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0 && r < nb) norms[(z * BH + bh) * nb + r] = __double2float_ru(__dsqrt_ru(ss));
}

// Persistent: grid = min(SMs, items), 384 threads, one CTA per SM; CTA c
// takes a contiguous range of the items (head, row tile, key tile), so the
// 128 Q rows (A operand, hi | lo) are reloaded only when (head, row tile)
// changes.  Warp 0: bulk copies (A when it changes, after the MMAs of the
// previous A; K tiles through a 2-stage ring); warp 1: the MMAs, 3 per
// 16-wide k-step into one of four 128-column TMEM accumulators; warp 3:
// max_j |k_j| of each head it meets; warps 4-11: the epilogue, two warps per
// TMEM lane quarter with 64 columns each (scale, transpose through shared
// memory, coalesced row stores of approx [BH][nb][nbs]).
__global__ void __launch_bounds__(384, 1) screen_scores_kernel(const uint8_t* __restrict__ img,
                                                                const float* __restrict__ norms, int nb, int nbs,
                                                                int ntile, int64_t BH, float scale,
                                                                float* __restrict__ approx,
                                                                float* __restrict__ kmaxn, int* __restrict__ stats) {
  using namespace scr;
  using namespace sm100;
  if (blockIdx.x == 0 && threadIdx.x == 0) stats[0] = 0;  // rows deferred by screen_select_kernel
  extern __shared__ uint8_t scr_smem[];
  uint8_t* sm = scr_smem + ((1024u - (smem_u32(scr_smem) & 1023u)) & 1023u);
  uint8_t* sA = sm;                 // [hi tile | lo tile]
  uint8_t* sB = sm + 2 * TILE;      // 2 stages of [hi tile | lo tile]
  float* sT = reinterpret_cast<float*>(sB + 4 * TILE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sT + EPI_WARPS * 32 * 33);
  uint64_t* afull = bars;
  uint64_t* aempty = bars + 1;
  uint64_t* bfull = bars + 2;   // [2]
  uint64_t* bempty = bars + 4;  // [2]
  uint64_t* tfull = bars + 6;   // [4]
  uint64_t* tempty = bars + 10;  // [4]
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t items = BH * ntile * ntile;
  const int64_t per = (items + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * per;
  const int64_t i1 = items < i0 + per ? items : i0 + per;
  const int nn = i1 > i0 ? static_cast<int>(i1 - i0) : 0;
  // item i: head bh, row tile rt, key tile kt; the A group of an item
  auto group = [&](int64_t it) { return it / ntile; };
  if (threadIdx.x == 0) {
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (warp == 0) {
    if (elect_one()) {
      int na = 0;
      for (int n = 0; n < nn; ++n) {
        const int64_t it = i0 + n, g = group(it);
        const int64_t bh = g / ntile;
        const int kt = static_cast<int>(it % ntile);
        if (n == 0 || g != group(it - 1)) {
          if (na > 0) mbar_wait(aempty, (na - 1) & 1);
          const int rt = static_cast<int>(g % ntile);
          mbar_arrive_expect_tx(afull, 2 * TILE);
          bulk_load_1d(sA, img + ((0 * BH + bh) * ntile + rt) * TILE, TILE, afull, policy_evict_first());
          bulk_load_1d(sA + TILE, img + ((1 * BH + bh) * ntile + rt) * TILE, TILE, afull, policy_evict_first());
          ++na;
        }
        const int s = n & 1;
        if (n >= 2) mbar_wait(&bempty[s], ((n >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&bfull[s], 2 * TILE);
        bulk_load_1d(sB + s * 2 * TILE, img + ((2 * BH + bh) * ntile + kt) * TILE, TILE, &bfull[s],
                     policy_evict_last());
        bulk_load_1d(sB + s * 2 * TILE + TILE, img + ((3 * BH + bh) * ntile + kt) * TILE, TILE, &bfull[s],
                     policy_evict_last());
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16_f32(ROWS, ROWS, false, false);
    const bool leader = elect_one();
    const uint64_t dAh = desc_sw128(smem_u32(sA), 16, 1024), dAl = desc_sw128(smem_u32(sA + TILE), 16, 1024);
    int na = 0;
    for (int n = 0; n < nn; ++n) {
      const int64_t it = i0 + n, g = group(it);
      const int s = n & 1, a = n & 3;
      if (n == 0 || g != group(it - 1)) mbar_wait(afull, (na++) & 1);
      mbar_wait(&bfull[s], (n >> 1) & 1);
      if (n >= 4) mbar_wait(&tempty[a], ((n >> 2) - 1) & 1);
      tc_fence_after();
      if (leader) {
        const uint64_t dBh = desc_sw128(smem_u32(sB + s * 2 * TILE), 16, 1024);
        const uint64_t dBl = desc_sw128(smem_u32(sB + s * 2 * TILE + TILE), 16, 1024);
        const uint32_t acc = tmem + a * ROWS;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ko = ((kk & 3) * 32 + (kk >> 2) * ATOM) >> 4;
          mma_bf16_ss(acc, dAl + ko, dBh + ko, idesc, kk > 0 ? 1u : 0u);
          mma_bf16_ss(acc, dAh + ko, dBl + ko, idesc, 1u);
          mma_bf16_ss(acc, dAh + ko, dBh + ko, idesc, 1u);
        }
        mma_commit(&bempty[s]);
        mma_commit(&tfull[a]);
        // the A of this group is done with after its last item
        if (n + 1 == nn || group(it + 1) != g) mma_commit(aempty);
      }
      __syncwarp();
    }
  } else if (warp == 3) {
    int64_t last_bh = -1;
    for (int n = 0; n < nn; ++n) {
      const int64_t bh = group(i0 + n) / ntile;
      if (bh == last_bh) continue;
      last_bh = bh;
      const float* kn = norms + (BH + bh) * nb;
      float m = 0.f;
      for (int j = lane; j < nb; j += 32) m = fmaxf(m, kn[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) kmaxn[bh] = m;  // every CTA meeting this head writes the same value
    }
  } else if (warp >= 4) {
    const int ew = warp - 4, q4 = warp & 3, half = ew >> 2;
    float* T = sT + ew * 32 * 33;
    for (int n = 0; n < nn; ++n) {
      const int64_t it = i0 + n, g = group(it);
      const int64_t bh = g / ntile;
      const int rt = static_cast<int>(g % ntile), kt = static_cast<int>(it % ntile);
      float* out = approx + bh * nb * static_cast<int64_t>(nbs);
      const int row0 = rt * ROWS + q4 * 32;
      const int rmax = min(32, nb - row0);
      const int a = n & 3;
      mbar_wait(&tfull[a], (n >> 2) & 1);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + a * ROWS + half * 64;
      tmem_ld32(taddr, r0);
      tmem_ld32(taddr + 32, r1);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
#pragma unroll
      for (int gg = 0; gg < 2; ++gg) {
#pragma unroll
        for (int j = 0; j < 32; ++j) T[lane * 33 + j] = __uint_as_float(gg ? r1[j] : r0[j]) * scale;
        __syncwarp();
        const int col = kt * ROWS + half * 64 + gg * 32 + lane;
        if (col < nb)
          for (int rr = 0; rr < rmax; ++rr) out[static_cast<int64_t>(row0 + rr) * nbs + col] = T[rr * 33 + lane];
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

struct ScreenArgs {
  const float* approx;
  const double* pooled;
  const float* norms;
  const float* kmaxn;
  int* full_count;  // rows decided wholly in float64 ...
  int* full_list;   // ... and which
  int* diag;        // per row: band size | bisection steps << 16 (-1: deferred)
  int nb;
  int64_t BH, rows, L;
  int block, topk, kmax;
  double sqrt_d, inv_sqrt_d;
  int nbs;  // row stride of approx (floats)
  int32_t* idx;
  int32_t* cnt;
  uint8_t* mask;
  unsigned long long* attended;
};

// One warp per row: a bracket [lo, hi] of the k-th best approximate score,
// the band, float64 scores of the band, the exact decision.  Rows that
// cannot be decided this way go to a list for screen_exact_kernel.  Lane l
// loads float4 j of its row at 32 j + l (coalesced; the approx rows are
// padded to 32 NPER floats), so value b is column 128 (b / 4) + 4 l + b % 4;
// the band is compacted by one prefix sum over the lanes (any order), the
// selection is regrouped into 32-column words (one per lane) for the
// ascending index list.
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <int NPER>
__device__ __forceinline__ void screen_one_row(const ScreenArgs& a, int64_t row, int lane, int* listA) {
  using namespace scr;
  const int nb = a.nb;
  const int64_t bh = row / nb;
  // value b of a lane: column 128 (b / 4) + 4 lane + b % 4 (coalesced float4 loads)
  auto col = [&](int b) { return 128 * (b >> 2) + 4 * lane + (b & 3); };
  // every load of the row up front: its approximate scores, its Q mean
  // (4 columns per lane, for the float64 scores of the band), its bound
  const float4* arow = reinterpret_cast<const float4*>(a.approx + row * (32 * NPER)) + lane;
  float v[NPER];
#pragma unroll
  for (int j = 0; j < NPER / 4; ++j) {
    const float4 t = arow[32 * j];
    v[4 * j] = t.x;
    v[4 * j + 1] = t.y;
    v[4 * j + 2] = t.z;
    v[4 * j + 3] = t.w;
  }
  const double2 q01 = reinterpret_cast<const double2*>(a.pooled + row * D)[lane * 2];
  const double2 q23 = reinterpret_cast<const double2*>(a.pooled + row * D)[lane * 2 + 1];
  const float qn = a.norms[row], kn = a.kmaxn[bh];
  float vmax = -INFINITY, vmin = INFINITY, vsum = 0.f, vsq = 0.f;
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    // padding is NaN: ignored by fmaxf / fminf, above nothing, in no band
    if (col(i) >= nb) v[i] = __int_as_float(0x7fffffff);
    const float u = col(i) < nb ? v[i] : 0.f;
    vmax = fmaxf(vmax, v[i]);
    vmin = fminf(vmin, v[i]);
    vsum += u;  // a NaN / inf score anywhere makes this non-finite
    vsq = fmaf(u, u, vsq);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
    vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
    vsq += __shfl_xor_sync(0xffffffffu, vsq, o);
  }
  const bool bad = !isfinite(vsum) || !isfinite(vsq);
  const int need = a.topk < nb ? a.topk : nb;
  const double E = kScreenBound * static_cast<double>(qn) * static_cast<double>(kn) * a.inv_sqrt_d * (1.0 + 1e-6) +
                   1e-300;
  uint32_t bits = 0;
  if (need < nb) {
    auto defer = [&]() {
      if (lane == 0) {
        a.full_list[atomicAdd(a.full_count, 1)] = static_cast<int>(row);
        a.diag[row] = -1;
      }
    };
    if (bad || !(E < 1e300) || static_cast<double>(vmax) - static_cast<double>(vmin) > 700.0) {
      defer();
      return;
    }
    // count(v > x): the sign of x - v (exact: x - v is 0 only for x == v,
    // and never -0 for x != -0), one FADD and one shifted add per value; the
    // NaN padding gives a positive NaN
    auto count_gt = [&](float x) {
      x += 0.f;  // -0 -> +0
      unsigned c = 0;
#pragma unroll
      for (int i = 0; i < NPER; ++i) c += __float_as_uint(__fsub_rn(x, v[i])) >> 31;
      return static_cast<int>(__reduce_add_sync(0xffffffffu, c));
    };
    // Bracket t_k, the need-th best approximate score: count(v >= lo) >=
    // need and count(v > hi) < need, until count(v > lo) == need exactly
    // (then t_k = min{v > lo}) or hi - lo <= E.  Probes: the normal quantile
    // of the row's mean and spread, one Newton step with the normal density
    // there, then interpolation of the count inside the bracket.  The probes
    // only steer; the bracket is kept by the exact counts.
    float lo = vmin, hi = vmax;
    int clo = nb, chi = 0;
    bool lo_exact = false;
    int it = 0;
    const float mean = vsum / nb, sd = sqrtf(fmaxf(vsq / nb - mean * mean, 0.f));
    const float z = 1.41421356f * erfinvf(1.f - 2.f * (static_cast<float>(need) - 0.5f) / static_cast<float>(nb));
    const float dens = static_cast<float>(nb) * 0.39894228f * __expf(-0.5f * z * z) / fmaxf(sd, 1e-30f);
    float x = mean + z * sd;
    int c = 0;
    for (; it < 48 && static_cast<double>(hi) - static_cast<double>(lo) > E; ++it) {
      const float w = hi - lo;
      if (it == 1) {
        x = x + (static_cast<float>(c - need) + 0.5f) / dens;
      } else if (it > 1) {
        const float f = (static_cast<float>(clo - need) + 0.5f) / static_cast<float>(clo - chi);
        x = lo + fminf(fmaxf(f, 0.125f), 0.875f) * w;
      }
      x = fminf(fmaxf(x, lo + w * (1.f / 64.f)), hi - w * (1.f / 64.f));
      if (!(x > lo && x < hi)) break;
      c = count_gt(x);
      if (c >= need) {
        lo = x;
        clo = c;
        if (c == need) {
          lo_exact = true;
          break;
        }
      } else {
        hi = x;
        chi = c;
      }
    }
    if (lo_exact) {
      float m = INFINITY;
#pragma unroll
      for (int i = 0; i < NPER; ++i) m = fminf(m, __fsub_rn(v[i], lo) > 0.f ? v[i] : INFINITY);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
      lo = hi = m;
    }
    // tau (the k-th best float64 score) lies in [lo - E, hi + E]: in above
    // hi + 2E, out below lo - 2E (thresholds rounded outward to float)
    const float hiB = __double2float_ru(static_cast<double>(hi) + 2.0 * E);
    const float loB = __double2float_rd(static_cast<double>(lo) - 2.0 * E);
    uint32_t abits = 0;
#pragma unroll
    for (int i = 0; i < NPER; ++i) {
      const bool inD = v[i] > hiB;
      bits |= static_cast<uint32_t>(inD) << i;
      abits |= static_cast<uint32_t>(!inD && v[i] >= loB) << i;
    }
    const int nD = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(__popc(bits))));
    const int myA = __popc(abits);
    int incl = myA;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int nA = __shfl_sync(0xffffffffu, incl, 31);
    if (nA > kScreenBand) {
      defer();
      return;
    }
    if (lane == 0) a.diag[row] = nA | (it << 16);
    {
      int p = incl - myA;
      for (uint32_t m = abits; m; m &= m - 1) listA[p++] = col(__ffs(m) - 1);
    }
    __syncwarp();
    const double* kbase = a.pooled + (a.BH + bh) * nb * D;
    // the band's K means into L1 at once (lane: one 128-byte line of one
    // entry, four entries per pass), so the dot products below do not pay
    // one L2 round trip per pair
    for (int b0 = 0; b0 < nA; b0 += 4)
      if (b0 + (lane >> 3) < nA) prefetch_l1(kbase + static_cast<int64_t>(listA[b0 + (lane >> 3)]) * D + (lane & 7) * 16);
    // float64 scores of the band (warp dot products, two K rows in flight);
    // lane b keeps band entry b
    const int cb = lane < nA ? listA[lane] : 0;
    double pm = 0.0;
    for (int b = 0; b < nA; b += 2) {
      const int j0 = listA[b], j1 = listA[b + 1 < nA ? b + 1 : b];
      const double2* k0 = reinterpret_cast<const double2*>(kbase + static_cast<int64_t>(j0) * D) + lane * 2;
      const double2* k1 = reinterpret_cast<const double2*>(kbase + static_cast<int64_t>(j1) * D) + lane * 2;
      const double2 a0 = k0[0], a1 = k0[1], b0 = k1[0], b1 = k1[1];
      double p0 = q01.x * a0.x, p1 = q01.x * b0.x;
      p0 = fma(q01.y, a0.y, p0);
      p1 = fma(q01.y, b0.y, p1);
      p0 = fma(q23.x, a1.x, p0);
      p1 = fma(q23.x, b1.x, p1);
      p0 = fma(q23.y, a1.y, p0);
      p1 = fma(q23.y, b1.y, p1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, o);
        p1 += __shfl_xor_sync(0xffffffffu, p1, o);
      }
      if (lane == b) pm = p0;
      if (lane == b + 1) pm = p1;
    }
    const uint64_t key = lane < nA ? desc_key(pm / a.sqrt_d) : ~0ull;
    // the band's best need - nD by (float64 score, then lower block)
    int rank = 0;
    for (int y = 0; y < nA; ++y) {
      const uint64_t ky = __shfl_sync(0xffffffffu, key, y);
      const int cy = __shfl_sync(0xffffffffu, cb, y);
      rank += (ky < key) || (ky == key && cy < cb);
    }
    const uint32_t won = __ballot_sync(0xffffffffu, lane < nA && rank < need - nD);
    {
      int p = incl - myA;
      for (uint32_t m = abits; m; m &= m - 1, ++p)
        if ((won >> p) & 1u) bits |= 1u << (__ffs(m) - 1);
    }
  } else {
#pragma unroll
    for (int i = 0; i < NPER; ++i) bits |= static_cast<uint32_t>(col(i) < nb) << i;
  }
  // the selection as 32-column words, lane w holding columns [32 w, 32 w +
  // 32): nibble j of lane l is columns 128 j + 4 l .. + 3, i.e. word 4 j +
  // l / 8, bits 4 (l % 8) ..; OR them across each 8-lane group, then lane w
  // takes word w from group w % 4 of nibble w / 4
  uint32_t word = 0;
#pragma unroll
  for (int j = 0; j < NPER / 4; ++j) {
    uint32_t x = ((bits >> (4 * j)) & 15u) << (4 * (lane & 7));
    x |= __shfl_xor_sync(0xffffffffu, x, 1);
    x |= __shfl_xor_sync(0xffffffffu, x, 2);
    x |= __shfl_xor_sync(0xffffffffu, x, 4);
    const uint32_t y = __shfl_sync(0xffffffffu, x, 8 * (lane & 3));
    if ((lane >> 2) == j) word = y;
  }
  // outputs: ascending index list (lane-major = column order), count,
  // mask, attended pairs
  const int mine = __popc(word);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  int32_t* irow = a.idx + row * a.kmax + (incl - mine);
  for (uint32_t m = word; m; m &= m - 1) *irow++ = 32 * lane + __ffs(m) - 1;
  if (a.mask != nullptr) {
    uint8_t* mrow = a.mask + row * nb;
    for (int i = 0; i < 32 && 32 * lane + i < nb; ++i) mrow[32 * lane + i] = (word >> i) & 1u;
  }
  // every selected block has `block` keys except a selected ragged last one
  const int last = nb - 1;
  const bool last_sel = __any_sync(0xffffffffu, last / 32 == lane && ((word >> (last % 32)) & 1u));
  if (lane == 0) {
    const int qb = static_cast<int>(row % nb);
    const long long ksum = static_cast<long long>(need) * a.block -
                           (last_sel ? static_cast<long long>(nb) * a.block - a.L : 0);
    a.cnt[row] = need;
    atomicAdd(a.attended + bh, static_cast<unsigned long long>(ksum * block_size(a.L, a.block, qb)));
  }
}

// Persistent warps over the rows; each warp prefetches its next row's
// approximate scores and Q mean into L1 before deciding the current one.
template <int NPER>
__global__ void __launch_bounds__(256, NPER >= 32 ? 3 : 4) screen_select_kernel(const ScreenArgs a) {
  __shared__ int listA[8][scr::kScreenBand];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * 8;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp; row < a.rows; row += stride) {
    const int64_t next = row + stride;
    if (next < a.rows) {
      if (lane < NPER) prefetch_l1(a.approx + next * (32 * NPER) + lane * 32);
      if (lane < 8) prefetch_l1(a.pooled + next * scr::D + lane * 16);
    }
    screen_one_row<NPER>(a, row, lane, listA[warp]);
    __syncwarp();
  }
}

// The listed rows, decided wholly in float64: every score (lane = column,
// the 128 products in order, Q row from shared memory), the probability-
// underflow clamp of mechanism.py:310-317 and topk_row.  A grid-stride loop
// over the list; the count is read once.
template <int NPER>
__global__ void __launch_bounds__(256) screen_exact_kernel(const ScreenArgs a) {
  using namespace scr;
  __shared__ int hist_all[8][256];
  __shared__ double qs_all[8][D];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = *a.full_count;
  const int nb = a.nb;
  for (int w = blockIdx.x * 8 + warp; w < n; w += gridDim.x * 8) {
    const int64_t row = a.full_list[w];
    const int64_t bh = row / nb;
    const double* qrow = a.pooled + row * D;
    const double* kbase = a.pooled + (a.BH + bh) * nb * D;
    double* qs = qs_all[warp];
#pragma unroll
    for (int e = 0; e < 4; ++e) qs[lane * 4 + e] = qrow[lane * 4 + e];
    __syncwarp();
    uint64_t key[NPER];
    uint64_t amax = 0, amin = ~0ull;  // ascending keys of the row max / min
#pragma unroll
    for (int i = 0; i < NPER; ++i) {
      const int c = lane + 32 * i;
      key[i] = ~0ull;
      if (c < nb) {
        const double2* kr = reinterpret_cast<const double2*>(kbase + static_cast<int64_t>(c) * D);
        double p = 0.0;
#pragma unroll 8
        for (int e = 0; e < D / 2; ++e) {
          const double2 kk = kr[e];
          p = fma(qs[2 * e], kk.x, p);
          p = fma(qs[2 * e + 1], kk.y, p);
        }
        key[i] = desc_key(p / a.sqrt_d);
        amax = max(amax, ~key[i]);
        amin = min(amin, ~key[i]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      amin = min(amin, __shfl_xor_sync(0xffffffffu, amin, o));
    }
    auto value_of = [](uint64_t asc) {
      return __longlong_as_double(static_cast<long long>((asc >> 63) ? (asc & ~(1ull << 63)) : ~asc));
    };
    const double row_max = value_of(amax);
    if (row_max > -INFINITY && value_of(amin) - row_max < kProbUnderflow) {
#pragma unroll
      for (int i = 0; i < NPER; ++i)
        if (lane + 32 * i < nb && value_of(~key[i]) - row_max < kProbUnderflow) key[i] = desc_key(-INFINITY);
    }
    topk_row<NPER>(key, hist_all[warp], lane, nb, row, a.L, a.block, a.topk, a.kmax, a.idx, a.cnt, a.mask,
                   a.attended);
    __syncwarp();
  }
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

// The screening path's state inside the scores area (select.cu, K1 screening).
struct ScreenLayout {
  size_t approx, img, norms, kmaxn, stats, list, diag, total;
};

// Values per lane of screen_select_kernel, and the approx row stride 32 * that.
static int screen_nper(int64_t nb) { return nb <= 128 ? 4 : nb <= 256 ? 8 : nb <= 512 ? 16 : 32; }

static ScreenLayout screen_layout(int64_t BH, int64_t nb) {
  const int64_t ntile = ceil_div(nb, scr::ROWS);
  const int64_t nbs = 32 * screen_nper(nb);
  ScreenLayout y{};
  size_t off = 0;
  auto take = [&off](size_t b) {
    const size_t o = off;
    off += (b + 255) / 256 * 256;
    return o;
  };
  y.approx = take(static_cast<size_t>(BH * nb * nbs) * sizeof(float));
  y.img = take(static_cast<size_t>(4 * BH * ntile) * scr::TILE);
  y.norms = take(static_cast<size_t>(2 * BH * nb) * sizeof(float));
  y.kmaxn = take(static_cast<size_t>(BH) * sizeof(float));
  y.stats = take(16);
  y.list = take(static_cast<size_t>(BH * nb) * sizeof(int));
  y.diag = take(static_cast<size_t>(BH * nb) * sizeof(int));
  y.total = off;
  return y;
}

static bool screen_eligible(const ropeslr_shape* s, int32_t topk) {
  const int64_t nb = ceil_div(s->L, s->block);
  return tuning().screen && topk > 0 && s->d == scr::D && nb <= 1024;
}

static size_t scores_bytes(const ropeslr_shape* s) {
  const int64_t nb = ceil_div(s->L, s->block);
  const size_t f64 = ((static_cast<size_t>(s->B * s->H * nb * nb) * sizeof(double) + 255) / 256) * 256;
  const size_t scr_bytes = s->d == scr::D ? screen_layout(s->B * s->H, nb).total : 0;
  return f64 > scr_bytes ? f64 : scr_bytes;
}

// Top-k of every row through the screening kernels (area: the scores area).
static int launch_screen(const ropeslr_shape* s, const ropeslr_select_params* sel, const double* pooled,
                         int32_t* idx, int32_t kmax, int32_t* cnt, uint8_t* mask, int64_t* attended, uint8_t* area,
                         bool have_img, cudaStream_t st) {
  const int64_t BH = s->B * s->H;
  const int nb = static_cast<int>(ceil_div(s->L, s->block));
  const int ntile = static_cast<int>(ceil_div(nb, scr::ROWS));
  const int nbs = 32 * screen_nper(nb);
  const ScreenLayout y = screen_layout(BH, nb);
  float* approx = reinterpret_cast<float*>(area + y.approx);
  uint8_t* img = area + y.img;
  float* norms = reinterpret_cast<float*>(area + y.norms);
  float* kmaxn = reinterpret_cast<float*>(area + y.kmaxn);
  int* stats = reinterpret_cast<int*>(area + y.stats);
  if (!have_img)
    screen_image_kernel<<<dim3(static_cast<unsigned>(ntile * 16), static_cast<unsigned>(BH), 2), 256, 0, st>>>(
        pooled, nb, ntile, BH, img, norms);
  if (cudaFuncSetAttribute(screen_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, scr::SMEM) !=
      cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  const int64_t items = BH * ntile * static_cast<int64_t>(ntile);
  const unsigned grid_s = static_cast<unsigned>(std::min<int64_t>(items, num_sms()));
  screen_scores_kernel<<<grid_s, 128 + 32 * scr::EPI_WARPS, scr::SMEM, st>>>(
      img, norms, nb, nbs, ntile, BH, static_cast<float>(1.0 / sqrt(static_cast<double>(scr::D))), approx, kmaxn,
      stats);
  ScreenArgs a{};
  a.approx = approx;
  a.pooled = pooled;
  a.norms = norms;
  a.kmaxn = kmaxn;
  a.full_count = stats;
  a.full_list = reinterpret_cast<int*>(area + y.list);
  a.diag = reinterpret_cast<int*>(area + y.diag);
  a.nb = nb;
  a.BH = BH;
  a.rows = BH * nb;
  a.L = s->L;
  a.block = s->block;
  a.topk = sel->topk;
  a.kmax = kmax;
  a.sqrt_d = sqrt(static_cast<double>(scr::D));
  a.inv_sqrt_d = 1.0 / a.sqrt_d;
  a.nbs = nbs;
  a.idx = idx;
  a.cnt = cnt;
  a.mask = mask;
  a.attended = reinterpret_cast<unsigned long long*>(attended);
  // the selection: persistent warps, as many CTAs of 8 as fit per SM (3 for
  // NPER 32: 78 registers, no spills; 4 below); the exact pass: enough warps
  // for a list of every row
  const unsigned grid_x = static_cast<unsigned>(std::min<int64_t>(ceil_div(a.rows, 8), 4 * num_sms()));
#define ROPESLR_SCREEN_CASE(NPER_)                                                                        \
  do {                                                                                                    \
    const unsigned grid = static_cast<unsigned>(                                                          \
        std::min<int64_t>(ceil_div(a.rows, 8), ((NPER_) >= 32 ? 3 : 4) * static_cast<int64_t>(num_sms()))); \
    screen_select_kernel<NPER_><<<grid, 256, 0, st>>>(a);                                                 \
    screen_exact_kernel<NPER_><<<grid_x, 256, 0, st>>>(a);                                                \
  } while (0)
  if (nb <= 128)
    ROPESLR_SCREEN_CASE(4);
  else if (nb <= 256)
    ROPESLR_SCREEN_CASE(8);
  else if (nb <= 512)
    ROPESLR_SCREEN_CASE(16);
  else
    ROPESLR_SCREEN_CASE(32);
#undef ROPESLR_SCREEN_CASE
  return launch_status();
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
  if (sel->topk <= 0 && nb <= 1024 && !tuning().keep_bitonic) {
    const int64_t off = row0;
    const unsigned grid = static_cast<unsigned>(row1 - row0);
    constexpr int KT = kKeepThreads;
    if (nb <= KT * 2)
      select_keep_kernel<KT, 2><<<grid, KT, 0, st>>>(scores + off * nb, nb, s->L, s->block, sel->keep, kmax,
                                                     idx + off * kmax, cnt + off, mask ? mask + off * nb : nullptr,
                                                     att + bh0);
    else
      select_keep_kernel<KT, 1024 / KT><<<grid, KT, 0, st>>>(scores + off * nb, nb, s->L, s->block, sel->keep,
                                                             kmax, idx + off * kmax, cnt + off,
                                                             mask ? mask + off * nb : nullptr, att + bh0);
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
// scores_out: the caller's float64 scores (then every pair is scored in
// float64), else NULL; area: the workspace's scores area.
static int select_from_pooled(const ropeslr_shape* s, const ropeslr_select_params* sel, const double* pooled,
                              int32_t* idx, int32_t kmax, int32_t* cnt, uint8_t* mask, int64_t* attended,
                              double* scores_out, uint8_t* area, cudaStream_t st, bool have_img = false) {
  const int64_t BH = s->B * s->H;
  const int d = static_cast<int>(s->d);
  const int nb = static_cast<int>(ceil_div(s->L, s->block));
  if (cudaMemsetAsync(attended, 0, sizeof(int64_t) * BH, st) != cudaSuccess) return ROPESLR_ERR_LAUNCH;
  if (int e = scan_nonfinite(pooled, true, 2 * BH * nb * d, sel->nonfinite, ROPESLR_NONFINITE_QK, st)) return e;
  if (scores_out == nullptr && screen_eligible(s, sel->topk))
    return launch_screen(s, sel, pooled, idx, kmax, cnt, mask, attended, area, have_img, st);
  double* scores = scores_out ? scores_out : reinterpret_cast<double*>(area);
  if (int e = launch_scores(pooled, scores, nb, d, BH, 0, BH, st)) return e;
  return launch_select(s, sel, scores, idx, kmax, cnt, mask, attended, 0, BH, st);
}

static int launch_pool(const ropeslr_shape* s, const void* q, const void* k, double* pooled, int64_t bh0, int64_t bh1,
                       cudaStream_t st, uint8_t* img = nullptr, float* norms = nullptr, bool* wrote_img = nullptr) {
  const int64_t BH = s->B * s->H;
  const int d = static_cast<int>(s->d);
  const int nb = static_cast<int>(ceil_div(s->L, s->block));
  dim3 grid(nb, static_cast<unsigned>(bh1 - bh0), 2);
  const int chunks = d / 8;
  const int lanes_r = 256 / chunks;
  size_t sm = static_cast<size_t>(lanes_r) * d * sizeof(double);
  const bool bulk = s->dtype == ROPESLR_BF16 && d == 128 && s->block <= 128 && aligned16(q) && aligned16(k);
  if (wrote_img != nullptr) *wrote_img = bulk && img != nullptr;
  if (bulk)
    pool_blocks_bulk_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(q),
                                                   static_cast<const __nv_bfloat16*>(k), pooled, s->L, s->block, nb,
                                                   BH, bh0, img, norms, static_cast<int>(ceil_div(nb, 128)));
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
  uint8_t* area = static_cast<uint8_t*>(ws) + pooled_bytes(s);
  // the screening path's image rows and norms come from the pooling kernel
  uint8_t* img = nullptr;
  float* norms = nullptr;
  if (scores_out == nullptr && screen_eligible(s, sel->topk)) {
    const ScreenLayout y = screen_layout(s->B * s->H, ceil_div(s->L, s->block));
    img = area + y.img;
    norms = reinterpret_cast<float*>(area + y.norms);
  }
  bool have_img = false;
  if (int e = launch_pool(s, q, k, pooled, 0, s->B * s->H, st, img, norms, &have_img)) return e;
  return select_from_pooled(s, sel, pooled, idx, kmax, cnt, mask, attended, scores_out, area, st, have_img);
}

extern "C" int ropeslr_select_from_pooled(const ropeslr_shape* s, const ropeslr_select_params* sel,
                                          const double* pooled, int32_t* idx, int32_t kmax, int32_t* cnt,
                                          uint8_t* mask, int64_t* attended, double* scores_out, void* ws,
                                          size_t ws_bytes, void* stream_) {
  int stt = check_select(s, sel, kmax, idx, cnt, attended);
  if (stt) return stt;
  if (!pooled) return ROPESLR_ERR_NULL;
  if (scores_out == nullptr && (ws == nullptr || ws_bytes < ropeslr_select_pooled_workspace_bytes(s)))
    return ROPESLR_ERR_WORKSPACE;
  return select_from_pooled(s, sel, pooled, idx, kmax, cnt, mask, attended, scores_out, static_cast<uint8_t*>(ws),
                            static_cast<cudaStream_t>(stream_));
}

extern "C" int ropeslr_select_screen_offsets(const ropeslr_shape* s, int32_t topk, size_t* approx_offset,
                                             size_t* stats_offset, size_t* diag_offset) {
  if (s == nullptr || approx_offset == nullptr || stats_offset == nullptr) return ROPESLR_ERR_NULL;
  if (s->block < 1 || s->L < 1 || s->B < 1 || s->H < 1) return ROPESLR_ERR_SHAPE;
  if (!screen_eligible(s, topk)) return ROPESLR_ERR_VALUE;
  const ScreenLayout y = screen_layout(s->B * s->H, ceil_div(s->L, s->block));
  *approx_offset = y.approx;
  *stats_offset = y.stats;
  if (diag_offset != nullptr) *diag_offset = y.diag;
  return ROPESLR_OK;
}
