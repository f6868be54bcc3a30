// Fused 3D RoPE + block pooling: the step before K1 selection (SURVEY.md
// section 8f, "next" #1).  Un-rotated Q and K [B, H, L, d] go in; rotated Q
// and K (same dtype) and the float64 block means of the *rotated, cast*
// values (what K1 pools, mechanism.py:306-308) come out, from one HBM pass
// instead of a rotation pass plus a pooling pass.
//
// The rotation restates rope3d.rotate_rows (rope3d.py:102-143) exactly as
// the package's torch path computes it (paper_2605_20659_b200/rope3d.py):
// angle = coord_axis * base^(-2(m-1)/d_axis) in float64, cos / sin in
// float64, (e, o) -> (c*e - s*o, s*e + c*o) with each product and sum
// rounded separately (no FMA contraction), then cast to the storage dtype
// the way torch does (float64 -> float32 -> bfloat16).  The cos / sin
// values depend only on (axis coordinate, pair), so they are tabulated per
// axis ([n_axis, d_axis / 2]) by rope_tables_kernel.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace ropeslr {
namespace rp {

constexpr int kMaxPairs = 128;  // d <= 256

struct Tables {
  const double* cs;  // [rows, 2] interleaved (cos, sin); row = base of the pair's axis + coordinate
  int pair_axis[kMaxPairs];   // axis of pair j (0 t, 1 x, 2 y)
  int pair_col[kMaxPairs];    // m - 1 within the axis
  int axis_half[3];           // d_axis / 2
  int axis_row0[3];           // first table row of each axis (rows of axis a: n_a * d_a/2 entries)
};

// entries: axis a, coordinate c, pair m -> (cos, sin) of c * theta_{a,m}
__global__ void rope_tables_kernel(double* cs, const double* thetas, int n_t, int n_x, int n_y, int h_t, int h_x,
                                   int h_y) {
  const int total = n_t * h_t + n_x * h_x + n_y * h_y;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    int a, r = e, coord, m;
    if (r < n_t * h_t) {
      a = 0;
      coord = r / h_t;
      m = r % h_t;
    } else if ((r -= n_t * h_t) < n_x * h_x) {
      a = 1;
      coord = r / h_x;
      m = r % h_x;
    } else {
      r -= n_x * h_x;
      a = 2;
      coord = r / h_y;
      m = r % h_y;
    }
    const int off = a == 0 ? 0 : (a == 1 ? h_t : h_t + h_x);
    const double ang = static_cast<double>(coord) * thetas[off + m];
    cs[2 * e] = cos(ang);
    cs[2 * e + 1] = sin(ang);
  }
}

template <typename T>
__device__ __forceinline__ T cast_out(double v);
template <>
__device__ __forceinline__ float cast_out<float>(double v) {
  return __double2float_rn(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 cast_out<__nv_bfloat16>(double v) {
  return __float2bfloat16_rn(__double2float_rn(v));  // torch: float64 -> float -> bfloat16
}

// grid (nb, B*H, 2): z = 0 Q, z = 1 K; 256 threads; each thread owns 8
// consecutive columns (4 pairs) of the rows r = rr, rr + lanes_r, ...
// BULK (bf16, d = 128, block <= 128): the block's rows, one contiguous run of
// <= 32 KiB, arrive by a single bulk copy into shared memory first, so the
// loads in flight do not hang on one row load per thread at a time; the
// staging buffer then holds the f64 partial sums.
template <typename T, bool BULK>
__global__ void __launch_bounds__(256) rope_pool_kernel(const T* __restrict__ q_in, const T* __restrict__ k_in,
                                                        T* __restrict__ q_out, T* __restrict__ k_out,
                                                        double* __restrict__ pooled, const Tables tab, int64_t L,
                                                        int d, int block, int nb, int64_t BH, int grid_h,
                                                        int grid_w) {
  extern __shared__ double sred_dyn[];
  __shared__ __align__(128) uint8_t stage[BULK ? 128 * 128 * 2 : 16];
  __shared__ uint64_t bar;
  const int64_t bh = blockIdx.y;
  const T* src = (blockIdx.z == 0 ? q_in : k_in) + bh * L * d;
  T* dst = (blockIdx.z == 0 ? q_out : k_out) + bh * L * d;
  const int b = blockIdx.x;
  const int rows = block_size(L, block, b);
  const int64_t r0 = static_cast<int64_t>(b) * block;
  if (BULK) {
    if (threadIdx.x == 0) {
      sm100::mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = static_cast<uint32_t>(rows) * d * sizeof(T);
      sm100::mbar_arrive_expect_tx(&bar, bytes);
      sm100::bulk_load_1d(stage, src + r0 * d, bytes, &bar, sm100::policy_evict_first());
    }
    sm100::mbar_wait(&bar, 0);
  }
  double* sred = BULK ? reinterpret_cast<double*>(stage) : sred_dyn;
  const int chunks = d / 8;
  const int lanes_r = blockDim.x / chunks;
  const int tid = threadIdx.x;
  const int ch = tid % chunks;
  const int rr = tid / chunks;
  const int64_t frame = static_cast<int64_t>(grid_h) * grid_w;
  int ax[4], col[4], half[4], row0[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = ch * 4 + u;
    ax[u] = tab.pair_axis[j];
    col[u] = tab.pair_col[j];
    half[u] = tab.axis_half[ax[u]];
    row0[u] = tab.axis_row0[ax[u]];
  }
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  if (rr < lanes_r) {
    // grid coordinates of the first row, then stepped by lanes_r tokens
    // (L < 2^31: 32-bit index arithmetic)
    int p0 = static_cast<int>(r0 + rr);
    int ct = p0 / static_cast<int>(frame);
    int rem = p0 - ct * static_cast<int>(frame);
    int cx = rem / grid_w;
    int cy = rem - cx * grid_w;
    const int step_x = lanes_r / grid_w, step_y = lanes_r % grid_w;
    for (int r = rr; r < rows; r += lanes_r) {
      const int64_t pos = r0 + r;
      float v[8];
      if (BULK)
        load8(reinterpret_cast<const T*>(stage) + static_cast<int64_t>(r) * d + ch * 8, v);
      else
        load8(src + pos * d + ch * 8, v);
      double out[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int coord = ax[u] == 0 ? ct : (ax[u] == 1 ? cx : cy);
        const double2 csv = *reinterpret_cast<const double2*>(tab.cs + 2 * (row0[u] + coord * half[u] + col[u]));
        const double e = v[2 * u], o = v[2 * u + 1];
        out[2 * u] = __dsub_rn(__dmul_rn(csv.x, e), __dmul_rn(csv.y, o));
        out[2 * u + 1] = __dadd_rn(__dmul_rn(csv.y, e), __dmul_rn(csv.x, o));
      }
      T ov[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        ov[i] = cast_out<T>(out[i]);
        acc[i] += static_cast<double>(to_f(ov[i]));  // pool the values K2 will see
      }
      if (sizeof(T) == 2) {
        *reinterpret_cast<uint4*>(dst + pos * d + ch * 8) = *reinterpret_cast<const uint4*>(ov);
      } else {
        *reinterpret_cast<float4*>(dst + pos * d + ch * 8) = *reinterpret_cast<const float4*>(ov);
        *reinterpret_cast<float4*>(dst + pos * d + ch * 8 + 4) = *reinterpret_cast<const float4*>(ov + 4);
      }
      // advance (t, x, y) by lanes_r tokens
      cy += step_y;
      cx += step_x;
      if (cy >= grid_w) {
        cy -= grid_w;
        ++cx;
      }
      while (cx >= grid_h) {
        cx -= grid_h;
        ++ct;
      }
    }
  }
  if (BULK) __syncthreads();  // every staged row has been read
  if (rr < lanes_r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) sred[rr * d + ch * 8 + i] = acc[i];
  }
  __syncthreads();
  double* pdst = pooled + ((static_cast<int64_t>(blockIdx.z) * BH + bh) * nb + b) * d;
  for (int c = tid; c < d; c += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < lanes_r; ++j) s += sred[j * d + c];
    pdst[c] = s / static_cast<double>(rows);
  }
}

// ---------------------------------------------------------------------------
// bf16, d = 128, block <= 128: the block's two 64-column halves arrive by TMA
// (128-byte swizzle) and leave by TMA store from the same buffer, rotated in
// place.  Thread mapping: warp w, lane l works on 16-byte chunk
// ch = 2w + (l >> 4) (columns 8ch .. 8ch + 7, pairs 4ch .. 4ch + 3) of rows
// j + 16k, j = l & 15 -- the (row lane, chunk) split of K1's pooling
// (select.cu pool_blocks_bulk_kernel), so the float64 sums run in the same
// order and the means are bit-identical to K1's.  Within a half-warp the
// rows are 16 consecutive tokens: the swizzled chunks of 8 consecutive rows
// hit 8 different bank groups, and the (cos, sin) entries of a y-axis pair
// for 16 consecutive tokens are 16 consecutive table entries (the table is
// coordinate-minor: [axis][pair][coordinate]); t- and x-axis entries are
// nearly always one broadcast.
struct TablesT {
  const double2* cs;          // [rows] (cos, sin); row = axis_row0 + m * axis_n + coordinate
  int pair_axis[kMaxPairs];
  int pair_col[kMaxPairs];
  int axis_n[3];
  int axis_row0[3];
};

__global__ void rope_tables_t_kernel(double2* cs, const double* thetas, int n_t, int n_x, int n_y, int h_t, int h_x,
                                     int h_y) {
  const int total = n_t * h_t + n_x * h_x + n_y * h_y;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    int r = e, n, off;
    if (r < n_t * h_t) {
      n = n_t;
      off = 0;
    } else if ((r -= n_t * h_t) < n_x * h_x) {
      n = n_x;
      off = h_t;
    } else {
      r -= n_x * h_x;
      n = n_y;
      off = h_t + h_x;
    }
    const int m = r / n, coord = r % n;
    const double ang = static_cast<double>(coord) * thetas[off + m];
    cs[e] = make_double2(cos(ang), sin(ang));
  }
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(sm100::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

constexpr int kHalfBytes = 128 * 128;  // one 64-column half of a <= 128-row block
constexpr int kTmaSmem = 1024 + 2 * kHalfBytes + 16 * 128 * 8 + 16;

__global__ void __launch_bounds__(256) rope_pool_tma_kernel(const __grid_constant__ CUtensorMap m_qin,
                                                            const __grid_constant__ CUtensorMap m_kin,
                                                            const __grid_constant__ CUtensorMap m_qout,
                                                            const __grid_constant__ CUtensorMap m_kout,
                                                            double* __restrict__ pooled, const TablesT tab, int64_t L,
                                                            int block, int nb, int64_t BH, int grid_h, int grid_w) {
  constexpr int D = 128;
  extern __shared__ uint8_t dsm[];  // kTmaSmem bytes: two swizzled halves, the f64 partials, the barrier
  uint8_t* stage = dsm + ((1024u - (sm100::smem_u32(dsm) & 1023u)) & 1023u);  // 1024-aligned for the swizzle
  double* sred = reinterpret_cast<double*>(stage + 2 * kHalfBytes);
  uint64_t& bar = *reinterpret_cast<uint64_t*>(sred + 16 * D);
  const int bh = blockIdx.y, b = blockIdx.x;
  const CUtensorMap* min = blockIdx.z == 0 ? &m_qin : &m_kin;
  const CUtensorMap* mout = blockIdx.z == 0 ? &m_qout : &m_kout;
  const int rows = block_size(L, block, b);
  const int r0 = b * block;  // L < 2^31
  const int tid = threadIdx.x;
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    sm100::mbar_arrive_expect_tx(&bar, 2u * block * 128u);  // full boxes (rows past L are zero-filled)
    sm100::tma_load_3d(stage, min, &bar, 0, r0, bh);
    sm100::tma_load_3d(stage + kHalfBytes, min, &bar, 64, r0, bh);
  }
  const int lane = tid & 31;
  const int j = lane & 15;
  const int ch = 2 * (tid >> 5) + (lane >> 4);
  uint8_t* half = stage + (ch >> 3) * kHalfBytes;
  const int c16 = ch & 7;
  int ax[4], tb[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int p = ch * 4 + u;
    ax[u] = tab.pair_axis[p];
    tb[u] = tab.axis_row0[ax[u]] + tab.pair_col[p] * tab.axis_n[ax[u]];
  }
  const int frame = grid_h * grid_w;
  int pos = r0 + j;
  int ct = pos / frame;
  int rem = pos - ct * frame;
  int cx = rem / grid_w;
  int cy = rem - cx * grid_w;
  const int step_x = 16 / grid_w, step_y = 16 % grid_w;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  sm100::mbar_wait(&bar, 0);
  for (int r = j; r < rows; r += 16) {
    uint4* cell = reinterpret_cast<uint4*>(half + r * 128 + ((c16 ^ (r & 7)) << 4));
    const uint4 raw = *cell;
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
    uint32_t packed[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int coord = ax[u] == 0 ? ct : (ax[u] == 1 ? cx : cy);
      const double2 csv = __ldg(tab.cs + tb[u] + coord);
      const float2 eo = __bfloat1622float2(h2[u]);
      const double e = eo.x, o = eo.y;
      const double y0 = __dsub_rn(__dmul_rn(csv.x, e), __dmul_rn(csv.y, o));
      const double y1 = __dadd_rn(__dmul_rn(csv.y, e), __dmul_rn(csv.x, o));
      const __nv_bfloat162 ob = __floats2bfloat162_rn(__double2float_rn(y0), __double2float_rn(y1));
      const float2 of = __bfloat1622float2(ob);
      acc[2 * u] += static_cast<double>(of.x);  // pool the values K2 will see
      acc[2 * u + 1] += static_cast<double>(of.y);
      packed[u] = *reinterpret_cast<const uint32_t*>(&ob);
    }
    *cell = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    cy += step_y;
    cx += step_x;
    if (cy >= grid_w) {
      cy -= grid_w;
      ++cx;
    }
    while (cx >= grid_h) {
      cx -= grid_h;
      ++ct;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sred[j * D + ch * 8 + i] = acc[i];
  sm100::fence_proxy_async_smem();  // the rotated rows -> the TMA store
  __syncthreads();
  if (tid == 0) {
    tma_store_3d(mout, stage, 0, r0, bh);
    tma_store_3d(mout, stage + kHalfBytes, 64, r0, bh);
  }
  if (tid < D) {
    double sum = 0.0;
    for (int q = 0; q < 16; ++q) sum += sred[q * D + tid];
    pooled[((static_cast<int64_t>(blockIdx.z) * BH + bh) * nb + b) * D + tid] = sum / static_cast<double>(rows);
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // stage stays valid until read
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

// [BH, L, 128] bf16 as a 3-D tensor, box [64 columns, block rows, 1], 128-byte swizzle.
bool make_map(CUtensorMap* m, const void* base, int64_t BH, int64_t L, int block) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[3] = {128, static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(BH)};
  cuuint64_t strides[2] = {256, static_cast<cuuint64_t>(L) * 256};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(block), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int table_rows(const ropeslr_rope_args* r) {
  return r->grid_t * (r->d_t / 2) + r->grid_h * (r->d_x / 2) + r->grid_w * (r->d_y / 2);
}

}  // namespace rp
}  // namespace ropeslr

using namespace ropeslr;

// ROPESLR_ROPE_TMA=0 selects the row-bulk-copy kernel (rope_pool_kernel) for A/B runs.
static bool rp_tma_disabled() { return !tuning().rope_tma; }

extern "C" size_t ropeslr_rope_pool_workspace_bytes(const ropeslr_rope_args* r) {
  if (!r) return 0;
  const size_t half = static_cast<size_t>(r->d_t + r->d_x + r->d_y) / 2;
  return (static_cast<size_t>(rp::table_rows(r)) * 2 + half) * sizeof(double) + 256;
}

extern "C" int ropeslr_rope_pool(const ropeslr_shape* s, const ropeslr_rope_args* r, const void* q_in,
                                 const void* k_in, void* q_out, void* k_out, double* pooled, void* ws,
                                 size_t ws_bytes, void* stream) {
  if (!s || !r) return ROPESLR_ERR_NULL;
  if (s->B < 1 || s->H < 1 || s->L < 1 || s->block < 1) return ROPESLR_ERR_SHAPE;
  if (s->d < 8 || s->d > 2 * rp::kMaxPairs || s->d % 8) return ROPESLR_ERR_SHAPE;
  if (s->dtype != ROPESLR_F32 && s->dtype != ROPESLR_BF16) return ROPESLR_ERR_DTYPE;
  if (r->d_t < 0 || r->d_x < 0 || r->d_y < 0 || (r->d_t | r->d_x | r->d_y) & 1) return ROPESLR_ERR_VALUE;
  if (r->d_t + r->d_x + r->d_y != s->d) return ROPESLR_ERR_SHAPE;
  if (r->grid_t < 1 || r->grid_h < 1 || r->grid_w < 1) return ROPESLR_ERR_SHAPE;
  if (static_cast<int64_t>(r->grid_t) * r->grid_h * r->grid_w != s->L) return ROPESLR_ERR_SHAPE;
  if (!(r->base > 0.0) || !isfinite(r->base)) return ROPESLR_ERR_VALUE;
  if (!q_in || !k_in || !q_out || !k_out || !pooled) return ROPESLR_ERR_NULL;
  if (!aligned16(q_in) || !aligned16(k_in) || !aligned16(q_out) || !aligned16(k_out)) return ROPESLR_ERR_ALIGN;
  if (!ws || ws_bytes < ropeslr_rope_pool_workspace_bytes(r)) return ROPESLR_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  // theta_{a,m} = base^(-2(m-1)/d_a) on the host (C pow, as Python's ** does)
  const int ht = r->d_t / 2, hx = r->d_x / 2, hy = r->d_y / 2;
  double thetas[rp::kMaxPairs];
  rp::Tables tab;
  int j = 0;
  const int dims[3] = {r->d_t, r->d_x, r->d_y};
  const int halves[3] = {ht, hx, hy};
  const int ns[3] = {r->grid_t, r->grid_h, r->grid_w};
  int row0 = 0;
  for (int a = 0; a < 3; ++a) {
    tab.axis_half[a] = halves[a];
    tab.axis_row0[a] = row0;
    row0 += ns[a] * halves[a];
    for (int m = 0; m < halves[a]; ++m, ++j) {
      thetas[j] = pow(r->base, -2.0 * m / dims[a]);
      tab.pair_axis[j] = a;
      tab.pair_col[j] = m;
    }
  }
  double* cs = static_cast<double*>(ws);
  double* dthetas = cs + 2 * static_cast<size_t>(rp::table_rows(r));
  if (cudaMemcpyAsync(dthetas, thetas, sizeof(double) * j, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return ROPESLR_ERR_LAUNCH;
  const bool tma_path = s->dtype == ROPESLR_BF16 && s->d == 128 && s->block <= 128 && s->block % 8 == 0 &&
                        !rp_tma_disabled();
  if (tma_path)
    rp::rope_tables_t_kernel<<<static_cast<unsigned>(ceil_div(rp::table_rows(r), 256)), 256, 0, st>>>(
        reinterpret_cast<double2*>(cs), dthetas, r->grid_t, r->grid_h, r->grid_w, ht, hx, hy);
  else
    rp::rope_tables_kernel<<<static_cast<unsigned>(ceil_div(rp::table_rows(r), 256)), 256, 0, st>>>(
        cs, dthetas, r->grid_t, r->grid_h, r->grid_w, ht, hx, hy);
  if (launch_status()) return ROPESLR_ERR_LAUNCH;
  tab.cs = cs;
  const int64_t BH = s->B * s->H;
  const int d = static_cast<int>(s->d);
  const int nb = static_cast<int>(ceil_div(s->L, s->block));
  dim3 grid(nb, static_cast<unsigned>(BH), 2);
  const int lanes_r = 256 / (d / 8);
  const size_t sm = static_cast<size_t>(lanes_r) * d * sizeof(double);
  if (tma_path) {
    rp::TablesT tt;
    tt.cs = reinterpret_cast<const double2*>(cs);
    for (int p = 0; p < j; ++p) {
      tt.pair_axis[p] = tab.pair_axis[p];
      tt.pair_col[p] = tab.pair_col[p];
    }
    for (int a = 0; a < 3; ++a) {
      tt.axis_n[a] = ns[a];
      tt.axis_row0[a] = tab.axis_row0[a];
    }
    CUtensorMap mqi, mki, mqo, mko;
    if (!rp::make_map(&mqi, q_in, BH, s->L, s->block) || !rp::make_map(&mki, k_in, BH, s->L, s->block) ||
        !rp::make_map(&mqo, q_out, BH, s->L, s->block) || !rp::make_map(&mko, k_out, BH, s->L, s->block))
      return ROPESLR_ERR_LAUNCH;
    // opt in above 48 KiB on every call: the attribute is per device
    if (cudaFuncSetAttribute(rp::rope_pool_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rp::kTmaSmem) !=
        cudaSuccess)
      return ROPESLR_ERR_LAUNCH;
    rp::rope_pool_tma_kernel<<<grid, 256, rp::kTmaSmem, st>>>(mqi, mki, mqo, mko, pooled, tt, s->L, s->block, nb, BH, r->grid_h,
                                                   r->grid_w);
  } else if (s->dtype == ROPESLR_BF16 && d == 128 && s->block <= 128)
    rp::rope_pool_kernel<__nv_bfloat16, true><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(q_in), static_cast<const __nv_bfloat16*>(k_in),
        static_cast<__nv_bfloat16*>(q_out), static_cast<__nv_bfloat16*>(k_out), pooled, tab, s->L, d, s->block, nb,
        BH, r->grid_h, r->grid_w);
  else if (s->dtype == ROPESLR_BF16)
    rp::rope_pool_kernel<__nv_bfloat16, false><<<grid, 256, sm, st>>>(
        static_cast<const __nv_bfloat16*>(q_in), static_cast<const __nv_bfloat16*>(k_in),
        static_cast<__nv_bfloat16*>(q_out), static_cast<__nv_bfloat16*>(k_out), pooled, tab, s->L, d, s->block, nb,
        BH, r->grid_h, r->grid_w);
  else
    rp::rope_pool_kernel<float, false><<<grid, 256, sm, st>>>(static_cast<const float*>(q_in), static_cast<const float*>(k_in),
                                                       static_cast<float*>(q_out), static_cast<float*>(k_out), pooled,
                                                       tab, s->L, d, s->block, nb, BH, r->grid_h, r->grid_w);
  return launch_status();
}
