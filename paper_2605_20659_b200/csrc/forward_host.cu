// Whole RoPeSLR forward from host buffers, pipelined over PCIe.
//
// The reference's forward (mechanism.py:491-512) takes NumPy arrays in host
// memory.  This entry point accepts the same (host Q/K/V/X, host output),
// and hides the host<->device copies behind the kernels:
//
//   copy-in stream   params, X (all local columns), then Q/K/V head chunk by
//                    head chunk, an event after each chunk
//   caller's stream  K3 (compensator + gate) as soon as X is resident, the
//                    gate hook (head-parallel all-reduce), then per chunk:
//                    K1 selection and the fused K2/K4 attention writing the
//                    chunk's columns of the [B, L, H, d] output
//   copy-out stream  each finished chunk's output columns back to the host
//                    (2D copies), overlapping the next chunk's H2D and math
//
// Chunking needs the tcgen05 attention path (bf16, d = 128, block 64/128),
// whose epilogue can write a head slice of a wider output row; other shapes
// run as one chunk.  Everything is stream-ordered on the caller's stream.
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace ropeslr {

int attend_fused_tc_strided(const ropeslr_shape* s, const void* q, const void* k, const void* v, const int32_t* idx,
                            int32_t kmax, const int32_t* cnt, const void* y_lr, const float* g_logit, float b_g,
                            const float* rms_sparse, float eps, void* out, int out_H, int out_h0, void* ws,
                            size_t ws_bytes, cudaStream_t stream);
bool attend_tc_eligible(const ropeslr_shape* s);

namespace {

constexpr size_t kAlign = 256;
size_t up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

size_t elem_bytes(const ropeslr_shape& s) { return s.dtype == ROPESLR_BF16 ? 2 : 4; }

int64_t kmax_of(const ropeslr_host_forward* a, int64_t nb) {
  return a->sel.topk > 0 ? (a->sel.topk < nb ? a->sel.topk : nb) : nb;
}

bool chunkable(const ropeslr_host_forward* a) {
  return attend_tc_eligible(&a->shape);
}

int chunk_heads(const ropeslr_host_forward* a) {
  const int H = static_cast<int>(a->shape.H);
  if (!chunkable(a)) return H;
  if (a->chunk_heads > 0) return a->chunk_heads < H ? a->chunk_heads : H;
  const size_t qkv = static_cast<size_t>(a->shape.B * a->shape.H * a->shape.L * a->shape.d) * elem_bytes(a->shape);
  if (qkv < (64u << 20)) return H;  // small: one chunk
  const int c = static_cast<int>(ceil_div(H, 12));
  return c < 1 ? 1 : c;
}

// Head chunks: Hc heads each, except that the last Hc heads go one per chunk,
// so the compute and the output copy left after the final input copy are
// one head's worth.
struct Chunk {
  int64_t h0, hc;
};

Chunk chunk_at(int64_t H, int Hc, int c) {
  const int64_t tail = Hc > 1 && H > Hc ? Hc : 0;
  const int64_t n1 = ceil_div(H - tail, Hc);
  if (c < n1) {
    const int64_t h0 = static_cast<int64_t>(c) * Hc;
    return {h0, (H - tail - h0) < Hc ? (H - tail - h0) : Hc};
  }
  return {H - tail + (c - n1), 1};
}

int chunk_count(int64_t H, int Hc) {
  const int64_t tail = Hc > 1 && H > Hc ? Hc : 0;
  return static_cast<int>(ceil_div(H - tail, Hc) + tail);
}

// Workspace carve-up (offsets only; base may be null for sizing).
struct Plan {
  int Hc, nchunks;
  int64_t nb, kmax;
  size_t q, k, v, x, y_lr, out, g, lr_ws, lr_ws_bytes, sel_ws, sel_ws_bytes, idx, cnt, att, osp, osp_bytes;
  size_t w_a, w_b, rms_sp, rms_lr, alpha, w_g, pe_t, pe_x, pe_y, total;
};

Plan make_plan(const ropeslr_host_forward* a) {
  Plan p{};
  const ropeslr_shape& s = a->shape;
  const size_t es = elem_bytes(s);
  p.Hc = chunk_heads(a);
  p.nchunks = chunk_count(s.H, p.Hc);
  p.nb = ceil_div(s.L, s.block);
  p.kmax = kmax_of(a, p.nb);
  const size_t act = static_cast<size_t>(s.B * s.H * s.L * s.d) * es;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += up(bytes);
    return o;
  };
  p.q = take(act);
  p.k = take(act);
  p.v = take(act);
  p.x = take(act);
  p.y_lr = take(act);
  p.out = take(act);
  p.g = take(static_cast<size_t>(s.B * s.L) * 4);
  ropeslr_shape sh = s;
  p.lr_ws_bytes = ropeslr_lowrank_workspace_bytes(&sh, &a->tok, a->rank);
  p.lr_ws = take(p.lr_ws_bytes);
  ropeslr_shape sc = s;
  sc.H = p.Hc;
  p.sel_ws_bytes = ropeslr_select_workspace_bytes(&sc);
  p.sel_ws = take(p.sel_ws_bytes);
  p.idx = take(static_cast<size_t>(s.B * p.Hc * p.nb * p.kmax) * 4);
  p.cnt = take(static_cast<size_t>(s.B * p.Hc * p.nb) * 4);
  p.att = take(static_cast<size_t>(p.nchunks) * s.B * p.Hc * 8);
  // K2 scratch (the CUDA-core path's o_sparse, or the tcgen05 path's unit
  // schedule and key-block norms); chunks run in stream order and share it
  p.osp_bytes = ropeslr_attend_workspace_bytes(p.nchunks == 1 ? &sh : &sc, ROPESLR_IMPL_AUTO);
  p.osp = take(p.osp_bytes);
  const size_t D = static_cast<size_t>(a->tok.d_model);
  p.w_a = take(static_cast<size_t>(s.H * s.d * a->rank) * 4);
  p.w_b = take(static_cast<size_t>(s.H * s.d * a->rank) * 4);
  p.rms_sp = take(static_cast<size_t>(s.d) * 4);
  p.rms_lr = take(static_cast<size_t>(s.d) * 4);
  p.alpha = take(D * 4);
  p.w_g = take(D * 4);
  p.pe_t = take(static_cast<size_t>(a->tok.grid_t) * D * 4);
  p.pe_x = take(static_cast<size_t>(a->tok.grid_h) * D * 4);
  p.pe_y = take(static_cast<size_t>(a->tok.grid_w) * D * 4);
  p.total = off;
  return p;
}

bool is_device_ptr(const void* ptr) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Device copy of a parameter: used in place when already on the device,
// otherwise staged into the workspace on the copy stream.
template <typename T>
int stage(const T* src, size_t bytes, uint8_t* base, size_t off, cudaStream_t st, const T** dst) {
  if (src == nullptr) {
    *dst = nullptr;
    return ROPESLR_OK;
  }
  if (is_device_ptr(src)) {
    *dst = src;
    return ROPESLR_OK;
  }
  if (cudaMemcpyAsync(base + off, src, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) return ROPESLR_ERR_LAUNCH;
  *dst = reinterpret_cast<const T*>(base + off);
  return ROPESLR_OK;
}

int check(const ropeslr_host_forward* a) {
  if (!a) return ROPESLR_ERR_NULL;
  const ropeslr_shape& s = a->shape;
  if (s.B < 1 || s.H < 1 || s.L < 1 || s.d < 8 || s.block < 1) return ROPESLR_ERR_SHAPE;
  if (s.dtype != ROPESLR_F32 && s.dtype != ROPESLR_BF16) return ROPESLR_ERR_DTYPE;
  if (!a->q || !a->k || !a->v || !a->tok.x || !a->out || !a->w_a || !a->w_b || !a->rms_sparse || !a->rms_lowrank ||
      !a->tok.w_g)
    return ROPESLR_ERR_NULL;
  if (a->tok.use_pe && (!a->tok.pe_t || !a->tok.pe_x || !a->tok.pe_y || !a->tok.alpha)) return ROPESLR_ERR_NULL;
  if (a->out_row_stride < s.H * s.d || a->tok.x_row_stride < s.H * s.d) return ROPESLR_ERR_SHAPE;
  if (a->rank < 1) return ROPESLR_ERR_SHAPE;
  if (a->chunk_heads < 0) return ROPESLR_ERR_VALUE;
  return ROPESLR_OK;
}

struct Streams {
  cudaStream_t in = nullptr, out = nullptr;
  std::vector<cudaEvent_t> events;
  ~Streams() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);  // deferred until complete
    if (in) cudaStreamDestroy(in);
    if (out) cudaStreamDestroy(out);
  }
  cudaEvent_t event() {
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    events.push_back(e);
    return e;
  }
};

}  // namespace
}  // namespace ropeslr

using namespace ropeslr;

extern "C" size_t ropeslr_forward_host_workspace_bytes(const ropeslr_host_forward* a) {
  if (check(a) != ROPESLR_OK) return 0;
  return make_plan(a).total;
}

#define ROPESLR_TRY_CUDA(expr)                   \
  do {                                           \
    if ((expr) != cudaSuccess) return ROPESLR_ERR_LAUNCH; \
  } while (0)
#define ROPESLR_TRY(expr)        \
  do {                           \
    int st_ = (expr);            \
    if (st_ != ROPESLR_OK) return st_; \
  } while (0)

extern "C" int ropeslr_forward_host(const ropeslr_host_forward* a, void* workspace, size_t ws_bytes, void* stream) {
  ROPESLR_TRY(check(a));
  const Plan p = make_plan(a);
  if (!workspace || ws_bytes < p.total) return ROPESLR_ERR_WORKSPACE;
  const ropeslr_shape& s = a->shape;
  const size_t es = elem_bytes(s);
  const int64_t B = s.B, H = s.H, L = s.L, d = s.d;
  uint8_t* base = static_cast<uint8_t*>(workspace);
  cudaStream_t S = static_cast<cudaStream_t>(stream);

  Streams ss;
  ROPESLR_TRY_CUDA(cudaStreamCreateWithFlags(&ss.in, cudaStreamNonBlocking));
  ROPESLR_TRY_CUDA(cudaStreamCreateWithFlags(&ss.out, cudaStreamNonBlocking));
  // the workspace may still be in use by earlier work on the caller's stream
  cudaEvent_t ev_start = ss.event();
  if (!ev_start) return ROPESLR_ERR_LAUNCH;
  ROPESLR_TRY_CUDA(cudaEventRecord(ev_start, S));
  ROPESLR_TRY_CUDA(cudaStreamWaitEvent(ss.in, ev_start, 0));
  ROPESLR_TRY_CUDA(cudaStreamWaitEvent(ss.out, ev_start, 0));

  // ---- copy-in: parameters, X, then Q/K/V per head chunk
  const size_t D = static_cast<size_t>(a->tok.d_model);
  const float *w_a, *w_b, *rms_sp, *rms_lr, *alpha, *w_g, *pe_t, *pe_x, *pe_y;
  ROPESLR_TRY(stage(a->w_a, static_cast<size_t>(H * d * a->rank) * 4, base, p.w_a, ss.in, &w_a));
  ROPESLR_TRY(stage(a->w_b, static_cast<size_t>(H * d * a->rank) * 4, base, p.w_b, ss.in, &w_b));
  ROPESLR_TRY(stage(a->rms_sparse, static_cast<size_t>(d) * 4, base, p.rms_sp, ss.in, &rms_sp));
  ROPESLR_TRY(stage(a->rms_lowrank, static_cast<size_t>(d) * 4, base, p.rms_lr, ss.in, &rms_lr));
  ROPESLR_TRY(stage(a->tok.alpha, D * 4, base, p.alpha, ss.in, &alpha));
  ROPESLR_TRY(stage(a->tok.w_g, D * 4, base, p.w_g, ss.in, &w_g));
  const bool pe = a->tok.use_pe != 0;
  ROPESLR_TRY(stage(pe ? a->tok.pe_t : nullptr, a->tok.grid_t * D * 4, base, p.pe_t, ss.in, &pe_t));
  ROPESLR_TRY(stage(pe ? a->tok.pe_x : nullptr, a->tok.grid_h * D * 4, base, p.pe_x, ss.in, &pe_x));
  ROPESLR_TRY(stage(pe ? a->tok.pe_y : nullptr, a->tok.grid_w * D * 4, base, p.pe_y, ss.in, &pe_y));
  uint8_t* dx = base + p.x;
  ROPESLR_TRY_CUDA(cudaMemcpy2DAsync(dx, static_cast<size_t>(H * d) * es, a->tok.x,
                                     static_cast<size_t>(a->tok.x_row_stride) * es, static_cast<size_t>(H * d) * es,
                                     static_cast<size_t>(B * L), cudaMemcpyHostToDevice, ss.in));
  cudaEvent_t ev_x = ss.event();
  if (!ev_x) return ROPESLR_ERR_LAUNCH;
  ROPESLR_TRY_CUDA(cudaEventRecord(ev_x, ss.in));

  // device Q/K/V are chunk-major: chunk c is a dense [B, Hc_c, L, d] tensor
  const size_t head_bytes = static_cast<size_t>(L * d) * es;
  std::vector<cudaEvent_t> ev_in(p.nchunks);
  const uint8_t* hsrc[3] = {static_cast<const uint8_t*>(a->q), static_cast<const uint8_t*>(a->k),
                            static_cast<const uint8_t*>(a->v)};
  const size_t doff[3] = {p.q, p.k, p.v};
  for (int c = 0; c < p.nchunks; ++c) {
    const Chunk ck = chunk_at(H, p.Hc, c);
    const int64_t h0 = ck.h0, hc = ck.hc;
    for (int t = 0; t < 3; ++t) {
      uint8_t* dst = base + doff[t] + static_cast<size_t>(B * h0) * head_bytes;
      ROPESLR_TRY_CUDA(cudaMemcpy2DAsync(dst, hc * head_bytes, hsrc[t] + h0 * head_bytes, H * head_bytes,
                                         hc * head_bytes, static_cast<size_t>(B), cudaMemcpyHostToDevice, ss.in));
    }
    ev_in[c] = ss.event();
    if (!ev_in[c]) return ROPESLR_ERR_LAUNCH;
    ROPESLR_TRY_CUDA(cudaEventRecord(ev_in[c], ss.in));
  }

  // ---- compute: K3 on all local heads once X (and the parameters) landed
  ROPESLR_TRY_CUDA(cudaStreamWaitEvent(S, ev_x, 0));
  ropeslr_token_args tok = a->tok;
  tok.x = dx;
  tok.x_row_stride = H * d;
  tok.pe_t = pe_t;
  tok.pe_x = pe_x;
  tok.pe_y = pe_y;
  tok.alpha = alpha;
  tok.w_g = w_g;
  void* y_lr = base + p.y_lr;
  float* g_logit = reinterpret_cast<float*>(base + p.g);
  ROPESLR_TRY(ropeslr_lowrank_branch(&s, &tok, w_a, w_b, a->rank, rms_lr, a->eps, y_lr, nullptr, g_logit,
                                     base + p.lr_ws, p.lr_ws_bytes, S));
  if (a->gate_hook) a->gate_hook(g_logit, B * L, S, a->gate_hook_user);

  uint8_t* dout = base + p.out;
  int32_t* idx = reinterpret_cast<int32_t*>(base + p.idx);
  int32_t* cnt = reinterpret_cast<int32_t*>(base + p.cnt);
  for (int c = 0; c < p.nchunks; ++c) {
    const Chunk ck = chunk_at(H, p.Hc, c);
    const int64_t h0 = ck.h0, hc = ck.hc;
    ropeslr_shape sc = s;
    sc.H = hc;
    const size_t coff = static_cast<size_t>(B * h0) * head_bytes;
    const void* q = base + p.q + coff;
    const void* k = base + p.k + coff;
    const void* v = base + p.v + coff;
    int64_t* att = reinterpret_cast<int64_t*>(base + p.att) + static_cast<int64_t>(c) * B * p.Hc;
    ROPESLR_TRY_CUDA(cudaStreamWaitEvent(S, ev_in[c], 0));
    ROPESLR_TRY(ropeslr_select_blocks(&sc, &a->sel, q, k, idx, static_cast<int32_t>(p.kmax), cnt, nullptr, att,
                                      nullptr, base + p.sel_ws, p.sel_ws_bytes, S));
    if (p.nchunks == 1) {
      ROPESLR_TRY(ropeslr_attend_fused(&sc, q, k, v, idx, static_cast<int32_t>(p.kmax), cnt, nullptr, y_lr, g_logit,
                                       a->b_g, rms_sp, a->eps, dout, sc.dtype, nullptr, ROPESLR_IMPL_AUTO, base + p.osp,
                                       p.osp_bytes, S));
    } else {
      ROPESLR_TRY(attend_fused_tc_strided(&sc, q, k, v, idx, static_cast<int32_t>(p.kmax), cnt, y_lr, g_logit,
                                          a->b_g, rms_sp, a->eps, dout, static_cast<int>(H), static_cast<int>(h0),
                                          base + p.osp, p.osp_bytes, S));
    }
    cudaEvent_t ev_done = ss.event();
    if (!ev_done) return ROPESLR_ERR_LAUNCH;
    ROPESLR_TRY_CUDA(cudaEventRecord(ev_done, S));
    // ---- copy-out of this chunk's output columns (and attended counts)
    ROPESLR_TRY_CUDA(cudaStreamWaitEvent(ss.out, ev_done, 0));
    const size_t row_bytes = static_cast<size_t>(H * d) * es;
    ROPESLR_TRY_CUDA(cudaMemcpy2DAsync(static_cast<uint8_t*>(a->out) + static_cast<size_t>(h0 * d) * es,
                                       static_cast<size_t>(a->out_row_stride) * es,
                                       dout + static_cast<size_t>(h0 * d) * es, row_bytes,
                                       static_cast<size_t>(hc * d) * es, static_cast<size_t>(B * L),
                                       cudaMemcpyDeviceToHost, ss.out));
    if (a->attended)
      ROPESLR_TRY_CUDA(cudaMemcpy2DAsync(a->attended + h0, static_cast<size_t>(H) * 8, att,
                                         static_cast<size_t>(hc) * 8, static_cast<size_t>(hc) * 8,
                                         static_cast<size_t>(B), cudaMemcpyDeviceToHost, ss.out));
  }
  cudaEvent_t ev_end = ss.event();
  if (!ev_end) return ROPESLR_ERR_LAUNCH;
  ROPESLR_TRY_CUDA(cudaEventRecord(ev_end, ss.out));
  ROPESLR_TRY_CUDA(cudaStreamWaitEvent(S, ev_end, 0));
  return launch_status();
}
