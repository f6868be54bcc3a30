/*
 * ropeslr_b200.h -- C ABI of the B200-native RoPeSLR attention forward.
 *
 * The reference (arxiv 2605.20659, /root/reference/pkg/src/ropeslr) is a pure
 * Python/NumPy package with no FFI; its "plugin API" is the Python function
 * set of mechanism.py.  Each entry point below replaces one of those
 * functions (cited as mechanism.py:LINE) and is what a ctypes / cffi binding
 * on the reference side would bind.  The Python package
 * paper_2605_20659_b200 binds exactly these symbols.
 *
 * Conventions
 *   - Plain pointers to device memory, sizes in elements, caller-allocated
 *     outputs, stream-ordered (the `stream` argument is a cudaStream_t, 0 is
 *     the legacy default stream).  No hidden allocation: scratch comes from a
 *     caller-provided workspace whose size the *_workspace_bytes queries give.
 *   - Layouts (row-major, innermost last):
 *       Q, K, V          [B, H, L, d]   post-RoPE, dtype = shape.dtype
 *       X                [B, L, *]      token rows; the local heads' columns
 *                                       start at x_col_offset with row stride
 *                                       x_row_stride (elements)
 *       out, y_lr        [B, L, H, d]   == the reference's (L, d_model) rows
 *       o_sparse, o_lr   [B, H, L, d]   float32 debug/intermediate outputs
 *       g_logit          [B, L]         float32, x_hat . w_g over the local
 *                                       columns (no bias, no sigmoid)
 *       idx              [B, H, nb, kmax] int32, selected key blocks in
 *                                       ascending block order
 *       cnt              [B, H, nb]     int32 selected count per query block
 *       mask             [B, H, nb, nb] uint8 (the reference's `selected`)
 *       attended         [B, H]         int64 attended (query, key) pairs
 *     with nb = ceil(L / block) flat blocks, the last one ragged.
 *   - Parameters are float32: w_a [H,d,r], w_b [H,r,d], alpha/w_g [D_total],
 *     rms_sparse/rms_lowrank [d], per-axis PE tables [T|Hg|Wg, D_total].
 *   - Errors: a negative ropeslr_status; nothing is launched on error.  The
 *     Python layer maps every nonzero status to ValueError, mirroring the
 *     reference's ValueError on bad shapes/ranges (mechanism.py:230-233,
 *     266-270, 282-283, 297-300).
 *   - Threading: no global mutable state apart from a per-device attribute
 *     cache; calls on different streams may run concurrently.
 */
#ifndef ROPESLR_B200_H
#define ROPESLR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ROPESLR_ABI_VERSION 3

typedef enum ropeslr_status {
  ROPESLR_OK = 0,
  ROPESLR_ERR_SHAPE = -1,      /* inconsistent or unsupported sizes */
  ROPESLR_ERR_DTYPE = -2,      /* unsupported dtype code */
  ROPESLR_ERR_ALIGN = -3,      /* pointer not 16-byte aligned (32 bytes for out / y_lr on the tcgen05 paths) */
  ROPESLR_ERR_DIVIS = -4,      /* 3D block does not divide the grid */
  ROPESLR_ERR_LAUNCH = -5,     /* CUDA launch / runtime error */
  ROPESLR_ERR_VALUE = -6,      /* out-of-range scalar (keep, eps, topk, ...) */
  ROPESLR_ERR_WORKSPACE = -7,  /* workspace missing or too small */
  ROPESLR_ERR_ARCH = -8,       /* device is not sm_100 */
  ROPESLR_ERR_NULL = -9        /* required pointer is NULL */
} ropeslr_status;

typedef enum ropeslr_dtype { ROPESLR_F32 = 0, ROPESLR_BF16 = 1 } ropeslr_dtype;
typedef enum ropeslr_compensator { ROPESLR_LOWRANK = 0, ROPESLR_LINEAR = 1 } ropeslr_compensator;
/* Sparse-attention implementation: AUTO picks the tcgen05/TMEM kernel for
 * bf16 with d == 128 and block in {64, 128}, the CUDA-core kernel otherwise. */
typedef enum ropeslr_impl { ROPESLR_IMPL_AUTO = 0, ROPESLR_IMPL_SIMT = 1, ROPESLR_IMPL_TCGEN05 = 2 } ropeslr_impl;

typedef struct ropeslr_shape {
  int64_t B;      /* batch */
  int64_t H;      /* heads handled by this call (the local head slice) */
  int64_t L;      /* real tokens; no padding */
  int64_t d;      /* head dim */
  int32_t block;  /* flat block size in tokens (query blocks == key blocks) */
  int32_t dtype;  /* ropeslr_dtype of Q/K/V/X/out/y_lr */
  /* Query-block range [qb_begin, qb_end) of this call; 0, 0 = every block.
   * Honoured by the sparse attention (ropeslr_attend_fused, ropeslr_sparse_
   * attention; tcgen05 path): only the units (head, query block) of the range
   * run and only their output rows are written, the tensors keeping their
   * full-length layouts (a rank that shares a head with another rank computes
   * its half of the query blocks).  The other entry points ignore it. */
  int32_t qb_begin;
  int32_t qb_end;
} ropeslr_shape;

/* Selection rule.  topk > 0: keep the k best blocks (BASELINE configs);
 * topk == 0: the reference's cumulative-mass rule, smallest prefix of the
 * stable descending block-softmax order whose mass reaches keep - 1e-12
 * (mechanism.py:316-320, decomposition.py:105-111). */
typedef struct ropeslr_select_params {
  int32_t topk;
  double keep;
  /* Nullable device word.  The reference rejects non-finite inputs
   * (linalg.py:17-20 via as_matrix, mechanism.py:494): when set, the
   * selection ORs in ROPESLR_NONFINITE_QK (stream-ordered) if a Q or K value
   * is NaN or infinite.  Detected on the float64 block means, which any
   * non-finite member makes non-finite (a bf16/f32 sum cannot overflow f64). */
  uint32_t* nonfinite;
} ropeslr_select_params;

#define ROPESLR_NONFINITE_QK 1u
#define ROPESLR_NONFINITE_X 2u

/* Token-side inputs of the compensator / gate (mechanism.py:426-447). */
typedef struct ropeslr_token_args {
  const void* x;           /* X at [b=0, l=0, first local column] */
  int64_t x_row_stride;    /* elements between consecutive tokens */
  int64_t head_offset;     /* global index of local head 0 (for PE/alpha/w_g columns) */
  int64_t d_model;         /* D_total = columns of alpha / w_g / PE tables */
  int32_t grid_t, grid_h, grid_w;  /* 3D latent grid, grid_t*grid_h*grid_w == L */
  int32_t use_pe;          /* x_hat = x + alpha * PE when nonzero */
  const float* pe_t;       /* [grid_t, D_total] */
  const float* pe_x;       /* [grid_h, D_total] */
  const float* pe_y;       /* [grid_w, D_total] */
  const float* alpha;      /* [D_total] */
  const float* w_g;        /* [D_total] */
  /* Nullable device word: ORs in ROPESLR_NONFINITE_X when an X value of the
   * local columns is NaN or infinite (detected on the gate logits, whose
   * sums every value enters; needs g_logit). */
  uint32_t* nonfinite;
  /* Grid index of X's row 0.  Nonzero only for ropeslr_gate_logits on a
   * sequence shard (rows [token_offset, token_offset + L) of the grid, for
   * the PE coordinates); every other entry point requires 0 and L = the grid. */
  int64_t token_offset;
} ropeslr_token_args;

/* ---------------------------------------------------------------- misc */
int ropeslr_abi_version(void);
const char* ropeslr_status_string(int status);
/* The CUDA runtime's message for the last error behind a ROPESLR_ERR_LAUNCH
 * on the calling thread ("no error" if none). */
const char* ropeslr_last_cuda_error(void);
/* ROPESLR_OK when `device` is an sm_100 part the kernels were built for. */
int ropeslr_device_check(int device);
/* Number of flat blocks: ceil(L / block). */
int64_t ropeslr_num_blocks(int64_t L, int32_t block);
/* Kernel-variant switches for A/B tests and benchmarks, process-wide,
 * initialised once from the ROPESLR_* environment:
 *   "k2_online"     1: the running-max K2 kernel instead of the fixed-exponent one
 *   "pair64"        0: unpaired block-64 K/V tiles
 *   "pairs64"       0: block-64 units of one query block (default 1: units
 *                   of two adjacent query blocks over the union of their
 *                   selections, each row masking what its block did not select)
 *   "schedule"      0: no longest-first unit schedule under the keep rule
 *   "kv_evict_last" 0: no L2 evict-last hint on K/V tiles
 *   "scores"        'f' / 'd': CUDA-core / unpipelined DMMA block scores
 *   "rope_tma"      0: the row-bulk-copy RoPE pre-pass
 *   "linear_simt"   1: the CUDA-core linear compensator
 *   "screen"        0: K1 top-k from float64 scores of every block pair
 *                   (default 1: float32-grade tensor-core screening, float64
 *                   only where the decision can depend on it)
 *   "keep_bitonic"  1: keep-rule rows by the round-1 bitonic sort per row
 *                   (default 0: radix sort on float32 keys, exact order
 *                   restored inside runs of equal keys)
 * Not synchronised with calls in flight on other threads.  Unknown name:
 * ROPESLR_ERR_VALUE.  ropeslr_get_option returns the current value. */
int ropeslr_set_option(const char* name, int value);
int ropeslr_get_option(const char* name);

/* ------------------------------------------------ K1: block selection
 * Replaces the routing half of block_sparse_attention (mechanism.py:305-320,
 * 326): fp64 mean-pooling of Q and K per block, fp64 scores / sqrt(d),
 * stable descending order (ties to the lower block index), top-k or
 * cumulative-mass count, ascending index list.  `mask` and `scores`
 * ([B,H,nb,nb] float64) may be NULL.  kmax must be >= min(topk, nb) in top-k
 * mode and >= nb in keep mode.
 *
 * Top-k with d = 128 and `scores` NULL takes the screening path: float32-
 * grade scores on the tensor cores with a proven per-row error bound E, then
 * float64 scores only for the blocks within 2E of the k-th (the result is
 * the float64 selection, K1). */
size_t ropeslr_select_workspace_bytes(const ropeslr_shape* shape);
int ropeslr_select_blocks(const ropeslr_shape* shape, const ropeslr_select_params* sel,
                          const void* q, const void* k,
                          int32_t* idx, int32_t kmax, int32_t* cnt, uint8_t* mask,
                          int64_t* attended, double* scores,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Selection from precomputed float64 block means pooled [2, B*H, nb, d]
 * (Q means, then K means; e.g. from ropeslr_rope_pool): the scores and
 * selection stages of ropeslr_select_blocks.  `scores` may be NULL, then
 * the workspace holds them. */
size_t ropeslr_select_pooled_workspace_bytes(const ropeslr_shape* shape);
int ropeslr_select_from_pooled(const ropeslr_shape* shape, const ropeslr_select_params* sel, const double* pooled,
                               int32_t* idx, int32_t kmax, int32_t* cnt, uint8_t* mask, int64_t* attended,
                               double* scores, void* workspace, size_t workspace_bytes, void* stream);

/* Where the screening path keeps its state inside the `scores` area of the
 * selection workspace (the workspace of ropeslr_select_from_pooled, or the
 * select workspace past the pooled means, ropeslr_select_pooled_workspace_
 * bytes): the float32 approximate scores [B*H, nb, nbs] at *approx_offset
 * (row stride nbs: the first of 128, 256, 512, 1024 that is >= nb),
 * at *stats_offset an int32 count of rows decided wholly in float64 (rows
 * whose band held more than 32 blocks, or non-finite / very wide rows), and
 * at *diag_offset (may be NULL) an int32 per row: band size | bisection
 * steps << 16, or -1 for a row decided wholly in float64.  For tests and
 * measurement.  Returns ROPESLR_ERR_VALUE when this shape does not take the
 * screening path. */
int ropeslr_select_screen_offsets(const ropeslr_shape* shape, int32_t topk, size_t* approx_offset,
                                  size_t* stats_offset, size_t* diag_offset);

/* ------------------------------- fused 3D RoPE + block pooling (pre-pass)
 * The caller-side rotation of the reference (rope3d.rotate_rows,
 * rope3d.py:102-143) fused with K1's pooling (mechanism.py:306-308): reads
 * un-rotated Q/K [B,H,L,d], writes the rotated Q/K (same dtype; float64
 * math, cast float64 -> float32 -> storage dtype like torch) and the float64
 * block means of the rotated, cast values, pooled [2, B*H, nb, d].  Pairs
 * (2j, 2j+1) in [t | x | y] order, angle = coord * base^(-2(m-1)/d_axis). */
typedef struct ropeslr_rope_args {
  int32_t d_t, d_x, d_y;            /* per-axis head-dim split, even, sum = d */
  int32_t grid_t, grid_h, grid_w;   /* 3D latent grid, product = L */
  double base;                      /* frequency base (10000) */
} ropeslr_rope_args;

size_t ropeslr_rope_pool_workspace_bytes(const ropeslr_rope_args* rope);
int ropeslr_rope_pool(const ropeslr_shape* shape, const ropeslr_rope_args* rope, const void* q_in, const void* k_in,
                      void* q_out, void* k_out, double* pooled, void* workspace, size_t workspace_bytes,
                      void* stream);

/* ------------------------------------ K2: block-sparse softmax attention
 * Replaces the exact-attention half of block_sparse_attention
 * (mechanism.py:321-326): each query block attends, with an exact softmax,
 * to the tokens of its selected key blocks.  Writes the un-normalised-branch
 * output o_sparse [B,H,L,d] float32.  `row_perm` (nullable, [L] int32) maps
 * the flat position of a query row to its token index (3D tiles, see
 * DESIGN.md); outputs are written at the token index. */
int ropeslr_sparse_attention(const ropeslr_shape* shape, const void* q, const void* k, const void* v,
                             const int32_t* idx, int32_t kmax, const int32_t* cnt,
                             const int32_t* row_perm, float* o_sparse, int32_t impl, void* stream);

/* -------------------------------------- K3: compensators and the gate
 * Low-rank compensator (mechanism.py:225-235, 441-446) with PE injection
 * (mechanism.py:212-218, 429-432), then RMSNorm (mechanism.py:238-246) with
 * rms_lowrank: y_lr = RMS(sigmoid(sigmoid(x_hat_h W_A[h]) W_B[h])) * rms_lowrank.
 * Optionally fuses the gate logits over the local columns (g_logit, nullable)
 * and writes the raw compensator output o_lr (nullable, float32 [B,H,L,d]).
 * bf16 with d == 128 runs on the tensor cores: the PE injection is folded
 * into per-axis [T|Hg|Wg, rank] tables ((alpha*P_axis)_h W_A[h]) built in the
 * workspace, so X is read once and x_hat is never materialised. */
size_t ropeslr_lowrank_workspace_bytes(const ropeslr_shape* shape, const ropeslr_token_args* tok,
                                       int32_t rank);
int ropeslr_lowrank_branch(const ropeslr_shape* shape, const ropeslr_token_args* tok,
                           const float* w_a, const float* w_b, int32_t rank,
                           const float* rms_lowrank, float eps,
                           void* y_lr, float* o_lr, float* g_logit,
                           void* workspace, size_t workspace_bytes, void* stream);

/* The same branch with its parameter-only tables built once: the W_A^T /
 * W_B^T operand images and the per-axis PE folds Z_axis = (alpha P_axis)_h
 * W_A and G_axis (what ropeslr_lowrank_branch rebuilds on every call).  They
 * depend on w_a, w_b, alpha, w_g, the PE tables, the grid and the head slice
 * only.  tcgen05 path only (bf16, d = 128, rank 16/32/48/64); _bytes
 * returns 0 otherwise.  The folded call's workspace holds the gate partials,
 * B*H*L floats (ropeslr_lowrank_workspace_bytes suffices). */
size_t ropeslr_lowrank_tables_bytes(const ropeslr_shape* shape, const ropeslr_token_args* tok, int32_t rank);
int ropeslr_lowrank_tables(const ropeslr_shape* shape, const ropeslr_token_args* tok, const float* w_a,
                           const float* w_b, int32_t rank, void* tables, size_t tables_bytes, void* stream);
int ropeslr_lowrank_branch_folded(const ropeslr_shape* shape, const ropeslr_token_args* tok, int32_t rank,
                                  const void* tables, size_t tables_bytes, const float* rms_lowrank, float eps,
                                  void* y_lr, float* o_lr, float* g_logit, void* workspace, size_t workspace_bytes,
                                  void* stream);

/* Gate logits alone: g_logit[b,l] = sum over the local columns of
 * x_hat[b,l,c] * w_g[c] (mechanism.py:249-255, 434; bias and sigmoid are
 * applied in the fused epilogue so that head-sharded ranks can all-reduce
 * the partial logits first).  With tok->token_offset the rows are the grid
 * tokens [token_offset, token_offset + L): a sequence shard's own gate over
 * all columns (ulysses.py). */
int ropeslr_gate_logits(const ropeslr_shape* shape, const ropeslr_token_args* tok,
                        float* g_logit, void* stream);

/* Linear-attention compensator (mechanism.py:33-36, 350-362): from the
 * caller's projections q_lin/k_lin/v_lin [B,H,L,d] (x_hat @ w_{q,k,v}[h], no
 * RoPE): phi = elu + 1, state S = phi(k)^T v (d x d) and z = sum phi(k),
 * reduced over L in fixed order (deterministic), then
 * o = phi(q) S / max(phi(q).z, 1e-8) and y_lr = RMS(o) * rms_lowrank. */
size_t ropeslr_linear_workspace_bytes(const ropeslr_shape* shape);
int ropeslr_linear_branch(const ropeslr_shape* shape, const void* q_lin, const void* k_lin,
                          const void* v_lin, const float* rms_lowrank, float eps,
                          void* y_lr, float* o_lr, void* workspace, size_t workspace_bytes,
                          void* stream);

/* Linear compensator with the PE injection in the kernels (bf16, d = 128;
 * csrc/linear_umma.cu).  The caller supplies the frozen projections of the
 * PLAIN token features, q_lin/k_lin/v_lin = x W_{q,k,v}[h] ([B,H,L,d] bf16,
 * no PE, no RoPE).  x_hat W = x W + (alpha * PE) W, and the second term is
 * parameter-only and axis-separable: ropeslr_linear_tables folds it into
 * per-axis tables T_axis = (alpha * P_axis) W_z[h] ([n_axis, d] per local
 * head and z in {q, k, v}, bf16) plus the gate's per-axis scalars
 * G_axis = (alpha * P_axis) . w_g over the local columns (float32), from
 * w_q/w_k/w_v float32 [H, D_total, d] (the local heads' backbone weights).
 * Cache the tables while the parameters do not change.  Then
 * ropeslr_linear_branch_pe runs the tcgen05 state pass (phi(K)^T V and
 * sum phi(K), fixed-order reduction), the apply pass (phi(Q) S / max(phi(Q) z,
 * 1e-8), RMSNorm * rms_lowrank -> y_lr, o_lr nullable) and the gate logits
 * (x . w_g + G rows; g_logit nullable).  `state` (nullable) receives S and z
 * as float32 [B*H, d, 144] (column 128 = z).  Both return ROPESLR_ERR_SHAPE
 * for shapes outside the path (then pass x_hat projections to
 * ropeslr_linear_branch). */
size_t ropeslr_linear_tables_bytes(const ropeslr_shape* shape, const ropeslr_token_args* tok);
int ropeslr_linear_tables(const ropeslr_shape* shape, const ropeslr_token_args* tok, const float* w_q,
                          const float* w_k, const float* w_v, void* tables, size_t tables_bytes, void* stream);
size_t ropeslr_linear_pe_workspace_bytes(const ropeslr_shape* shape, const ropeslr_token_args* tok);
int ropeslr_linear_branch_pe(const ropeslr_shape* shape, const ropeslr_token_args* tok, const void* q_lin,
                             const void* k_lin, const void* v_lin, const void* tables, const float* rms_lowrank,
                             float eps, void* y_lr, float* o_lr, float* g_logit, float* state, void* workspace,
                             size_t workspace_bytes, void* stream);

/* ------------------------------------------------ K4: fused epilogue
 * out = RMS(o_sparse) * rms_sparse + sigmoid(g_logit + b_g) * y_lr
 * (mechanism.py:437-451).  Standalone form used after the CUDA-core
 * attention kernel; the tcgen05 kernel fuses it (ropeslr_attend_fused). */
int ropeslr_fuse_output(const ropeslr_shape* shape, const float* o_sparse, const void* y_lr,
                        const float* g_logit, float b_g, const float* rms_sparse, float eps,
                        void* out, void* stream);

/* K2 + K4 in one launch where the tcgen05 path applies (else K2 then K4):
 * attention, normalisation by the softmax denominator, RMSNorm, gated
 * combination with y_lr and the store of out, in out_dtype: shape.dtype, or
 * ROPESLR_F32 for a float32 output from bf16 inputs (the fused result before
 * any bf16 rounding; [B,L,H,d] float32).  o_sparse (nullable)
 * additionally receives the raw sparse-branch output.  On the tcgen05 path
 * y_lr and out must be 32-byte aligned (256-bit row accesses), else
 * ROPESLR_ERR_ALIGN.  Workspace: the CUDA-core path keeps o_sparse there when
 * o_sparse is NULL.  The tcgen05 path keeps there, as int32:
 *   [0, NU)          a longest-first schedule of the NU = B*H*nb
 *                    (head, query block) units (`keep` rule only; top-k rows
 *                    are balanced by construction; ROPESLR_SCHEDULE=0 turns
 *                    it off),
 *   [NU, 2 NU)       per-unit flags of the fixed-exponent kernel,
 *   [2 NU]           the number of units whose exponent reference failed and
 *                    that the running-max kernel recomputed (the fallback
 *                    count; readable after the call),
 *   [2 NU + 1, ...)  their list,
 * and, for block 64 from the next 256-byte boundary, the query-block pairs'
 * union lists (pairs64 option): NP = B*H*ceil(nb/2) counts (int32), NP*nb
 * block indices (int32), NP*nb selection bytes; the schedule area then holds
 * the pairs' longest-first order.
 * Without a workspace the tcgen05 path runs the running-max kernel alone. */
int ropeslr_attend_fused(const ropeslr_shape* shape, const void* q, const void* k, const void* v,
                         const int32_t* idx, int32_t kmax, const int32_t* cnt,
                         const int32_t* row_perm, const void* y_lr, const float* g_logit, float b_g,
                         const float* rms_sparse, float eps, void* out, int32_t out_dtype, float* o_sparse,
                         int32_t impl, void* workspace, size_t workspace_bytes, void* stream);
size_t ropeslr_attend_workspace_bytes(const ropeslr_shape* shape, int32_t impl);

/* ------------------------------------- whole forward from HOST buffers
 * The reference's calling convention (NumPy arrays in host memory,
 * mechanism.py:491-512) for the low-rank compensator: copies X, then Q/K/V
 * in head chunks, to the device on an internal copy stream, runs K3 once X
 * is resident and K1 + K2/K4 per chunk as each chunk lands, and copies each
 * chunk's output columns back on a second copy stream, so PCIe traffic in
 * both directions overlaps the kernels.  Device scratch (activations,
 * routing, staged parameters) comes from `workspace`.  Parameter pointers may
 * be host or device memory.  Stream-ordered on `stream`: the host outputs
 * are valid once `stream` has been synchronised.  Host activation buffers
 * should be pinned (pageable memory works, without the overlap). */
typedef struct ropeslr_host_forward {
  ropeslr_shape shape;            /* H = heads of this call; dtype of q/k/v/x/out */
  ropeslr_select_params sel;
  const void* q;                  /* host [B, H, L, d] post-RoPE */
  const void* k;
  const void* v;
  ropeslr_token_args tok;         /* tok.x: host X rows (x_row_stride elements apart) */
  const float* w_a;               /* [H, d, r] */
  const float* w_b;               /* [H, r, d] */
  int32_t rank;
  const float* rms_sparse;        /* [d] */
  const float* rms_lowrank;       /* [d] */
  float b_g;
  float eps;
  void* out;                      /* host [B, L, *]: this call's heads from column 0 */
  int64_t out_row_stride;         /* elements between consecutive output rows */
  int64_t* attended;              /* host [B, H] attended pairs, nullable */
  int32_t chunk_heads;            /* heads per pipeline chunk; 0 = automatic */
  /* Called once, on the calling thread, after the gate logits [B, L]
   * (float32, device) have been enqueued on `stream` and before any use:
   * head-parallel ranks enqueue their all-reduce here.  Nullable. */
  void (*gate_hook)(float* g_logit, int64_t n, void* stream, void* user);
  void* gate_hook_user;
} ropeslr_host_forward;

size_t ropeslr_forward_host_workspace_bytes(const ropeslr_host_forward* args);
int ropeslr_forward_host(const ropeslr_host_forward* args, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------- caller helper: segmented row copy (ulysses.py)
 * The pack and unpack around the sequence <-> head all-to-alls of BASELINE
 * config 4, one launch each.  segs: DEVICE array of nseg segments, row0
 * ascending; segment k copies its `rows` rows (row_bytes each, a multiple of
 * 16, pointers and strides 16-byte aligned) from src to dst and covers the
 * launch's global rows [row0, row0 + rows); total_rows = the sum. */
typedef struct ropeslr_row_segment {
  const void* src;
  void* dst;
  int64_t src_stride;  /* bytes between rows */
  int64_t dst_stride;
  int64_t rows;
  int64_t row0;
  int32_t row_bytes;
  int32_t pad;
} ropeslr_row_segment;
int ropeslr_copy_rows(const ropeslr_row_segment* segs, int32_t nseg, int64_t total_rows, void* stream);

/* ------------------------- caller helpers: the config-4 DiT block (dit.py)
 * Fused token-wise ops around the op, bf16 rows of D columns (D % 8 == 0,
 * D <= 2048), fp32 math, one launch each instead of PyTorch's 5-8:
 *   ln_modulate:    y = LayerNorm(x) * (1 + scale) + shift   (scale, shift [D] fp32)
 *   rms_heads:      RMSNorm(x) * weight (weight NULL: no norm), written
 *                   head-major [H, N, D/H] when head_major, else [N, D]
 *   gated_residual: x += bf16(y * gate)                      (gate [D] fp32) */
int ropeslr_dit_ln_modulate(const void* x, const float* shift, const float* scale, float eps, int64_t N, int32_t D,
                            void* y, void* stream);
/* bf16(LayerNorm(x) * weight + bias) (an affine LayerNorm; float32 weight / bias [D]). */
int ropeslr_dit_ln_affine(const void* x, const float* weight, const float* bias, float eps, int64_t N, int32_t D,
                          void* y, void* stream);
int ropeslr_dit_rms_heads(const void* x, const void* weight, float eps, int64_t N, int32_t D, int32_t H,
                          int32_t head_major, void* out, void* stream);
/* rms_heads from rows x_row_stride elements apart (a column slice of a wider
 * row: the Q / K / V parts of one fused projection). */
int ropeslr_dit_rms_heads_strided(const void* x, int64_t x_row_stride, const void* weight, float eps, int64_t N,
                                  int32_t D, int32_t H, int32_t head_major, void* out, void* stream);
int ropeslr_dit_gated_residual(void* x, const void* y, const float* gate, int64_t N, int32_t D, void* stream);
/* out = x + bf16(y * gate), out of place (out may alias x). */
int ropeslr_dit_gated_add(const void* x, const void* y, const float* gate, int64_t N, int32_t D, void* out,
                          void* stream);
/* y [B, L, H, dh] = x [B, H, L, dh] (bf16, dh % 8 == 0): the attention
 * output back to token-major rows for the output projection. */
int ropeslr_dit_heads_to_tokens(const void* x, int64_t B, int32_t H, int64_t L, int32_t dh, void* y, void* stream);

/* ------------------------- Stage-I training (training.py; mechanism.py:426-488, 519-614)
 * The per-row chains of the fused forward / backward around the float32
 * GEMMs, on head-major float32 rows [H, L, d] (d in {32, 64, 128}):
 *   pre:      xh = x + alpha_h * pe (pe NULL: no PE), gpart[h, l] = xh . w_g_h,
 *             g[l] = sigmoid(sum_h gpart + b_g)
 *   rows:     z2 (= H1 W_B) in, d z2 out in place; dgpart[h, l] = d loss / d g
 *             per row; red[blocks][2][d] partial d rms_sparse / d rms_lowrank;
 *             loss_part[blocks] = partial sum of diff^2 (float64);
 *             gscale = 2 / (H * L * d * samples)
 *   gate_bwd: dzg[l] = (sum_h dgpart) g (1 - g); bg_part[ceil(L/256)] its sums
 *   dsig:     t *= h1 * (1 - h1)  (n floats, 16-byte aligned)
 *   xgrad:    red[H][blocks][2][d] partial d alpha (needs pe; dxh = d xh) / d w_g
 *   reduce:   out[o][j][c] += sum over parts, in part order (deterministic)
 * *_blocks give the partial counts (grid sizes) of rows / xgrad. */
int ropeslr_stage1_supported(int64_t d);
int ropeslr_stage1_rows_blocks(int64_t H, int64_t L);
int ropeslr_stage1_xgrad_blocks(int64_t H, int64_t L);
int ropeslr_stage1_pre(int64_t H, int64_t L, int64_t d, const float* x, const float* pe, const float* alpha,
                       const float* w_g, float b_g, float* xh, float* gpart, float* g, void* stream);
/* The same with b_g read from device memory (float64), for a training step
 * captured once in a CUDA graph and replayed while b_g changes. */
int ropeslr_stage1_pre_dev(int64_t H, int64_t L, int64_t d, const float* x, const float* pe, const float* alpha,
                           const float* w_g, const double* b_g, float* xh, float* gpart, float* g, void* stream);
int ropeslr_stage1_rows(int64_t H, int64_t L, int64_t d, float* z2, const float* o_sp, const float* target,
                        const float* g, const float* rms_sp, const float* rms_lr, float eps, float gscale,
                        float* dgpart, float* red, double* loss_part, void* stream);
int ropeslr_stage1_gate_bwd(int64_t H, int64_t L, const float* dgpart, const float* g, float* dzg, double* bg_part,
                            void* stream);
int ropeslr_stage1_dsig(float* t, const float* h1, int64_t n, void* stream);
int ropeslr_stage1_xgrad(int64_t H, int64_t L, int64_t d, const float* dxh, const float* xh, const float* pe,
                         const float* dzg, const float* w_g, float* red, void* stream);
int ropeslr_stage1_reduce(const float* parts, int32_t outer, int32_t nparts, int32_t groups, int32_t width, float* out,
                          void* stream);

/* The step's float32 GEMMs on the tcgen05 tensor cores, float32-grade (each
 * operand split into bf16 hi + lo, three MMAs per product; csrc/stage1_gemm.cu):
 *   gemm_rows: C[h] = epi(A[h] B[h]), A [H, L, K], B [H, K, N] ([H, N, K] when
 *              b_trans), C [H, L, N], K, N in {64, 128}; epi 0 none,
 *              1 sigmoid, 2 times aux (1 - aux) with aux [H, L, N];
 *   gemm_gram: out[h] (+)= A[h]^T B[h] summed over L, A [H, L, 128],
 *              B [H, L, N], N in {64, 128}; out [H, 128, N], or [H, N, 128]
 *              when transpose; fixed-order reduction over token chunks. */
int ropeslr_stage1_gemm_rows(int64_t H, int64_t L, int32_t K, int32_t N, const float* A, const float* B,
                             int32_t b_trans, int32_t epi, const float* aux, float* C, void* stream);
size_t ropeslr_stage1_gram_workspace_bytes(int64_t H, int64_t L, int32_t N);
int ropeslr_stage1_gemm_gram(int64_t H, int64_t L, int32_t N, const float* A, const float* B, float* out,
                             int32_t transpose, int32_t accumulate, void* workspace, size_t workspace_bytes,
                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ROPESLR_B200_H */
