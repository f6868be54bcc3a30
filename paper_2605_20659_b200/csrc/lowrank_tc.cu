// K3 on the tensor cores: the low-rank compensator + gate logits for bf16
// inputs with d = 128 (the BASELINE configs).
//
// Algebra (exact in real arithmetic, mechanism.py:429-447):
//   x_hat_h W_A[h] = X_h W_A[h] + sum_axis (alpha * P_axis[coord])_h W_A[h]
// so the 3D PE injection collapses into three tiny per-head tables
// Z_axis[h] = (alpha * P_axis)_h W_A[h]  ([T|Hg|Wg, r], computed once per call
// by lowrank_fold_kernel), and likewise the gate logit
//   x_hat . w_g = X . w_g + sum_axis G_axis[h][coord].
// The hot kernel therefore reads X exactly once, never materialises x_hat,
// and the gate's X . w_g rides GEMM1 as two extra output columns (w_g split
// into bf16 hi + lo, so the product keeps ~16 mantissa bits).
//
// Main kernel: 8 warps x 16 tokens per CTA, loop over local heads;
// mma.sync m16n8k16 bf16 -> fp32:
//   GEMM1 [16 x 128] x [128 x (r + 16)]  -> +Z tables -> sigmoid -> bf16
//   GEMM2 [16 x r]   x [r x 128]         -> sigmoid -> RMSNorm * rms_lowrank
// The C fragments of GEMM1 feed GEMM2's A fragments directly (registers).
// HBM traffic: X in (2 B/elt) + y_lr out (2 B/elt); the weights stay in L2/smem.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace ropeslr {
namespace lr {

constexpr int D = 128;
constexpr int kWarps = 8;
constexpr int kTokTile = 16 * kWarps;  // tokens per CTA
constexpr int XP = D * 2 + 16;         // padded smem pitch (bytes) of a 128-wide bf16 row

struct FoldArgs {
  const float* w_a;   // [H, d, r]
  const float* w_b;   // [H, r, d]
  const float* alpha; // [D_total]
  const float* w_g;   // [D_total]
  const float *pe_t, *pe_x, *pe_y;  // [n, D_total]
  int64_t d_model, head_offset;
  int H, r, T, Hg, Wg, use_pe;
  // outputs (workspace)
  __nv_bfloat16* waT;  // [H, r + 16, d]   rows r, r+1: w_g hi / lo
  __nv_bfloat16* wbT;  // [H, d, r]
  float* Z;            // [H, T + Hg + Wg, r]
  float* G;            // [H, T + Hg + Wg]
};

// grid (T + Hg + Wg + 1, H): the last x-block transposes the weights.
__global__ void __launch_bounds__(128) lowrank_fold_kernel(FoldArgs a) {
  const int h = blockIdx.y;
  const int r = a.r;
  const int NA = r + 16;
  const int64_t gc0 = (a.head_offset + h) * D;
  const int nrows = a.T + a.Hg + a.Wg;
  if (blockIdx.x == nrows) {
    const float* wa = a.w_a + static_cast<int64_t>(h) * D * r;
    const float* wb = a.w_b + static_cast<int64_t>(h) * r * D;
    __nv_bfloat16* waT = a.waT + static_cast<int64_t>(h) * NA * D;
    __nv_bfloat16* wbT = a.wbT + static_cast<int64_t>(h) * D * r;
    for (int e = threadIdx.x; e < NA * D; e += blockDim.x) {
      const int n = e / D, k = e % D;
      float v = 0.f;
      if (n < r) {
        v = wa[k * r + n];
      } else if (n == r) {
        v = __bfloat162float(__float2bfloat16_rn(a.w_g[gc0 + k]));
      } else if (n == r + 1) {
        const float hi = __bfloat162float(__float2bfloat16_rn(a.w_g[gc0 + k]));
        v = a.w_g[gc0 + k] - hi;
      }
      waT[e] = __float2bfloat16_rn(v);
    }
    for (int e = threadIdx.x; e < D * r; e += blockDim.x) {
      const int n = e / r, k = e % r;
      wbT[e] = __float2bfloat16_rn(wb[k * D + n]);
    }
    return;
  }
  if (!a.use_pe) return;
  __shared__ float v[D];
  __shared__ float red[4];
  const int i = blockIdx.x;
  const float* tab = i < a.T ? a.pe_t + static_cast<int64_t>(i) * a.d_model
                             : (i < a.T + a.Hg ? a.pe_x + static_cast<int64_t>(i - a.T) * a.d_model
                                               : a.pe_y + static_cast<int64_t>(i - a.T - a.Hg) * a.d_model);
  const int j = threadIdx.x;  // blockDim == D
  const float pv = a.alpha[gc0 + j] * tab[gc0 + j];
  v[j] = pv;
  float gp = pv * a.w_g[gc0 + j];
  gp = warp_sum(gp);
  if ((j & 31) == 0) red[j >> 5] = gp;
  __syncthreads();
  if (j < r) {
    const float* wa = a.w_a + static_cast<int64_t>(h) * D * r;
    float z = 0.f;
    for (int k = 0; k < D; ++k) z = fmaf(v[k], wa[k * r + j], z);
    a.Z[(static_cast<int64_t>(h) * nrows + i) * r + j] = z;
  }
  if (j == 0) a.G[static_cast<int64_t>(h) * nrows + i] = (red[0] + red[1]) + (red[2] + red[3]);
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float sig(float x) { return 1.f / (1.f + __expf(-x)); }

struct MainArgs {
  const __nv_bfloat16* x;  // [B, L, row_stride], local head 0 at column 0
  int64_t x_row_stride;
  int64_t L;
  int H, Hg, Wg, T, use_pe;
  const __nv_bfloat16* waT;
  const __nv_bfloat16* wbT;
  const float* Z;
  const float* G;
  const float* rms_lr;
  float eps;
  __nv_bfloat16* y_lr;  // [B, L, H, d]
  float* o_lr;          // [B, H, L, d] or null
  float* g_part;        // [B, H, L] per-head gate partials (reduced by gate_reduce_kernel)
};

// grid (ceil(L / 128), H, B), block 256: one (token tile, head) per CTA.
// R = rank (multiple of 16, <= 128).
template <int R>
__global__ void __launch_bounds__(kWarps * 32) lowrank_tc_kernel(MainArgs a) {
  constexpr int NA = R + 16;        // GEMM1 output columns (rank + gate hi/lo + pad)
  constexpr int WAP = D * 2 + 16;   // waT row pitch (bytes)
  constexpr int WBP = R * 2 + 16;   // wbT row pitch (bytes)
  extern __shared__ __align__(16) uint8_t sm[];
  uint8_t* sWa = sm;                          // [NA][WAP]
  uint8_t* sWb = sWa + NA * WAP;              // [D][WBP]
  uint8_t* sX = sWb + D * WBP;                // [kTokTile][XP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t b = blockIdx.z;
  const int h = blockIdx.y;
  const int64_t tok0 = static_cast<int64_t>(blockIdx.x) * kTokTile;
  const int nrows = a.T + a.Hg + a.Wg;
  // this thread's two token rows (g, g + 8) of the warp's 16-token slab
  int64_t tk[2];
  int ct[2], cx[2], cy[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    tk[i] = tok0 + warp * 16 + g + 8 * i;
    const int64_t tt = tk[i] < a.L ? tk[i] : a.L - 1;
    const int64_t hw = static_cast<int64_t>(a.Hg) * a.Wg;
    ct[i] = static_cast<int>(tt / hw);
    cx[i] = static_cast<int>((tt % hw) / a.Wg);
    cy[i] = static_cast<int>(tt % a.Wg);
  }
  float gacc[2] = {0.f, 0.f};
  {
  const uint32_t sWa_u = static_cast<uint32_t>(__cvta_generic_to_shared(sWa));
  const uint32_t sWb_u = static_cast<uint32_t>(__cvta_generic_to_shared(sWb));
  const uint32_t sX_u = static_cast<uint32_t>(__cvta_generic_to_shared(sX)) + warp * 16 * XP;

    {
      const uint4* wa = reinterpret_cast<const uint4*>(a.waT + static_cast<int64_t>(h) * NA * D);
      for (int e = tid; e < NA * D / 8; e += blockDim.x) {
        const int n = e / (D / 8), c = e % (D / 8);
        *reinterpret_cast<uint4*>(sWa + n * WAP + c * 16) = wa[e];
      }
      const uint4* wb = reinterpret_cast<const uint4*>(a.wbT + static_cast<int64_t>(h) * D * R);
      for (int e = tid; e < D * R / 8; e += blockDim.x) {
        const int n = e / (R / 8), c = e % (R / 8);
        *reinterpret_cast<uint4*>(sWb + n * WBP + c * 16) = wb[e];
      }
      // X slab of this warp: 16 rows x 256 B, 16-byte loads
      for (int e = lane; e < 16 * 16; e += 32) {
        const int row = e >> 4, c = e & 15;
        const int64_t tok = tok0 + warp * 16 + row;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (tok < a.L)
          v = __ldcs(reinterpret_cast<const uint4*>(a.x + (b * a.L + tok) * a.x_row_stride +
                                                    static_cast<int64_t>(h) * D) + c);
        *reinterpret_cast<uint4*>(sX + (warp * 16 + row) * XP + c * 16) = v;
      }
    }
    __syncthreads();

    // ---- GEMM1: z1 = X_h W_A[h] (+ gate hi/lo columns)
    float c1[NA / 8][4];
#pragma unroll
    for (int n = 0; n < NA / 8; ++n) c1[n][0] = c1[n][1] = c1[n][2] = c1[n][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      uint32_t a0, a1, a2, a3;
      ldmatrix_x4(sX_u + (lane & 15) * XP + (ks * 16 + (lane >> 4) * 8) * 2, a0, a1, a2, a3);
#pragma unroll
      for (int n = 0; n < NA / 8; n += 2) {
        uint32_t b0, b1, b2, b3;
        const int nrow = n * 8 + (lane & 7) + ((lane >> 4) << 3);
        ldmatrix_x4(sWa_u + nrow * WAP + (ks * 16 + ((lane >> 3) & 1) * 8) * 2, b0, b1, b2, b3);
        mma16816(c1[n], a0, a1, a2, a3, b0, b1);
        mma16816(c1[n + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // gate partial: columns R (hi) and R + 1 (lo) live in n-tile R/8, cols 0..1 (t4 == 0)
    {
      const float* Gh = a.G + static_cast<int64_t>(h) * nrows;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        float v = (t4 == 0) ? (c1[R / 8][2 * i] + c1[R / 8][2 * i + 1]) : 0.f;
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (a.use_pe) v += Gh[ct[i]] + Gh[a.T + cx[i]] + Gh[a.T + a.Hg + cy[i]];
        gacc[i] += v;
      }
    }
    // + PE fold, sigmoid, repack as GEMM2 A fragments
    uint32_t ha[R / 16][4];
    {
      const float* Zh = a.Z + static_cast<int64_t>(h) * nrows * R;
#pragma unroll
      for (int n = 0; n < R / 8; ++n) {
        const int col = n * 8 + 2 * t4;
        float v[4] = {c1[n][0], c1[n][1], c1[n][2], c1[n][3]};
        if (a.use_pe) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const float2 zt = *reinterpret_cast<const float2*>(Zh + static_cast<int64_t>(ct[i]) * R + col);
            const float2 zx = *reinterpret_cast<const float2*>(Zh + static_cast<int64_t>(a.T + cx[i]) * R + col);
            const float2 zy = *reinterpret_cast<const float2*>(Zh + static_cast<int64_t>(a.T + a.Hg + cy[i]) * R + col);
            v[2 * i] += (zt.x + zx.x) + zy.x;
            v[2 * i + 1] += (zt.y + zx.y) + zy.y;
          }
        }
        const uint32_t lo = pack_bf16(sig(v[0]), sig(v[1]));  // row g
        const uint32_t hi = pack_bf16(sig(v[2]), sig(v[3]));  // row g + 8
        const int ks = n >> 1;
        if ((n & 1) == 0) {
          ha[ks][0] = lo;
          ha[ks][1] = hi;
        } else {
          ha[ks][2] = lo;
          ha[ks][3] = hi;
        }
      }
    }
    // ---- GEMM2: z2 = h1 W_B[h]
    float c2[D / 8][4];
#pragma unroll
    for (int n = 0; n < D / 8; ++n) c2[n][0] = c2[n][1] = c2[n][2] = c2[n][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < R / 16; ++ks) {
#pragma unroll
      for (int n = 0; n < D / 8; n += 2) {
        uint32_t b0, b1, b2, b3;
        const int nrow = n * 8 + (lane & 7) + ((lane >> 4) << 3);
        ldmatrix_x4(sWb_u + nrow * WBP + (ks * 16 + ((lane >> 3) & 1) * 8) * 2, b0, b1, b2, b3);
        mma16816(c2[n], ha[ks][0], ha[ks][1], ha[ks][2], ha[ks][3], b0, b1);
        mma16816(c2[n + 1], ha[ks][0], ha[ks][1], ha[ks][2], ha[ks][3], b2, b3);
      }
    }
    // ---- sigmoid, RMSNorm over the 128 columns of each row, store
    float ss[2] = {0.f, 0.f};
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float o = sig(c2[n][e]);
        c2[n][e] = o;
        ss[e >> 1] = fmaf(o, o, ss[e >> 1]);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      ss[i] += __shfl_xor_sync(0xffffffffu, ss[i], 1);
      ss[i] += __shfl_xor_sync(0xffffffffu, ss[i], 2);
      ss[i] = 1.f / sqrtf(ss[i] / static_cast<float>(D) + a.eps);
    }
    // stage the bf16 tile in this warp's X slab (its X rows are consumed), then 16-byte stores
    __syncwarp();
    uint8_t* slab = sX + warp * 16 * XP;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int col = n * 8 + 2 * t4;
      const float2 w = *reinterpret_cast<const float2*>(a.rms_lr + col);
      *reinterpret_cast<uint32_t*>(slab + g * XP + col * 2) = pack_bf16(c2[n][0] * ss[0] * w.x, c2[n][1] * ss[0] * w.y);
      *reinterpret_cast<uint32_t*>(slab + (g + 8) * XP + col * 2) =
          pack_bf16(c2[n][2] * ss[1] * w.x, c2[n][3] * ss[1] * w.y);
      if (a.o_lr) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int64_t tok = tk[i];
          if (tok < a.L)
            *reinterpret_cast<float2*>(a.o_lr + ((b * a.H + h) * a.L + tok) * D + col) =
                make_float2(c2[n][2 * i], c2[n][2 * i + 1]);
        }
      }
    }
    __syncwarp();
    for (int e = lane; e < 16 * 16; e += 32) {
      const int row = e >> 4, c = e & 15;
      const int64_t tok = tok0 + warp * 16 + row;
      if (tok < a.L)
        __stcs(reinterpret_cast<uint4*>(a.y_lr + ((b * a.L + tok) * a.H + h) * D) + c,
               *reinterpret_cast<const uint4*>(slab + row * XP + c * 16));
    }
  }
  if (t4 == 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      if (tk[i] < a.L) a.g_part[(b * a.H + h) * a.L + tk[i]] = gacc[i];
  }
}

// g_logit[b, l] = sum_h g_part[b, h, l] in fixed head order (deterministic).
__global__ void gate_reduce_kernel(const float* __restrict__ g_part, int H, int64_t L, int64_t BL,
                                   float* __restrict__ g_logit) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= BL) return;
  const int64_t b = e / L, l = e % L;
  const float* src = g_part + b * H * L + l;
  float s = 0.f;
  for (int h = 0; h < H; ++h) s += src[static_cast<int64_t>(h) * L];
  g_logit[e] = s;
}

}  // namespace lr

size_t lowrank_tc_workspace_bytes(int64_t B, int64_t H, int64_t L, int r, int T, int Hg, int Wg) {
  const size_t nrows = static_cast<size_t>(T + Hg + Wg);
  size_t wa = static_cast<size_t>(H) * (r + 16) * lr::D * 2;
  size_t wb = static_cast<size_t>(H) * lr::D * r * 2;
  size_t z = static_cast<size_t>(H) * nrows * r * 4;
  size_t gg = static_cast<size_t>(H) * nrows * 4;
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  return up(wa) + up(wb) + up(z) + up(gg) + up(static_cast<size_t>(B * H * L) * 4);
}

bool lowrank_tc_eligible(const ropeslr_shape* s, int r) {
  return s->dtype == ROPESLR_BF16 && s->d == lr::D && r % 16 == 0 && r >= 16 && r <= 128;
}

int launch_lowrank_tc(const ropeslr_shape* s, const ropeslr_token_args* t, const float* w_a, const float* w_b,
                      int r, const float* rms_lowrank, float eps, void* y_lr, float* o_lr, float* g_logit, void* ws,
                      cudaStream_t st) {
  using namespace lr;
  const int H = static_cast<int>(s->H);
  const int nrows = t->grid_t + t->grid_h + t->grid_w;
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
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
  f.r = r;
  f.T = t->grid_t;
  f.Hg = t->grid_h;
  f.Wg = t->grid_w;
  f.use_pe = t->use_pe;
  f.waT = reinterpret_cast<__nv_bfloat16*>(p);
  p += up(static_cast<size_t>(H) * (r + 16) * D * 2);
  f.wbT = reinterpret_cast<__nv_bfloat16*>(p);
  p += up(static_cast<size_t>(H) * D * r * 2);
  f.Z = reinterpret_cast<float*>(p);
  p += up(static_cast<size_t>(H) * nrows * r * 4);
  f.G = reinterpret_cast<float*>(p);
  p += up(static_cast<size_t>(H) * nrows * 4);
  float* g_part = reinterpret_cast<float*>(p);
  lowrank_fold_kernel<<<dim3(nrows + 1, H), 128, 0, st>>>(f);
  if (launch_status()) return ROPESLR_ERR_LAUNCH;

  MainArgs m;
  m.x = static_cast<const __nv_bfloat16*>(t->x);
  m.x_row_stride = t->x_row_stride;
  m.L = s->L;
  m.H = H;
  m.Hg = t->grid_h;
  m.Wg = t->grid_w;
  m.T = t->grid_t;
  m.use_pe = t->use_pe;
  m.waT = f.waT;
  m.wbT = f.wbT;
  m.Z = f.Z;
  m.G = f.G;
  m.rms_lr = rms_lowrank;
  m.eps = eps;
  m.y_lr = static_cast<__nv_bfloat16*>(y_lr);
  m.o_lr = o_lr;
  m.g_part = g_part;
  dim3 grid(static_cast<unsigned>(ceil_div(s->L, kTokTile)), static_cast<unsigned>(H), static_cast<unsigned>(s->B));
#define ROPESLR_LR_CASE(R_)                                                                                   \
  case R_: {                                                                                                  \
    const size_t sm = static_cast<size_t>(R_ + 16) * (D * 2 + 16) + static_cast<size_t>(D) * (R_ * 2 + 16) + \
                      static_cast<size_t>(kTokTile) * XP;                                                     \
    auto kfn = lowrank_tc_kernel<R_>;                                                                         \
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)) !=       \
        cudaSuccess)                                                                                          \
      return ROPESLR_ERR_LAUNCH;                                                                              \
    kfn<<<grid, kWarps * 32, sm, st>>>(m);                                                                    \
    break;                                                                                                    \
  }
  switch (r) {
    ROPESLR_LR_CASE(16)
    ROPESLR_LR_CASE(32)
    ROPESLR_LR_CASE(64)
    ROPESLR_LR_CASE(128)
    default:
      return ROPESLR_ERR_SHAPE;
  }
#undef ROPESLR_LR_CASE
  if (launch_status()) return ROPESLR_ERR_LAUNCH;
  if (g_logit != nullptr) {
    const int64_t BL = s->B * s->L;
    gate_reduce_kernel<<<static_cast<unsigned>(ceil_div(BL, 256)), 256, 0, st>>>(g_part, H, s->L, BL, g_logit);
  }
  return launch_status();
}

}  // namespace ropeslr
