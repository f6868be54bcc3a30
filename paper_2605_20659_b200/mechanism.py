"""Host-side mirror of the reference's ``mechanism`` API over the B200 kernels.

Same names, dataclasses and error behaviour as
``/root/reference/pkg/src/ropeslr/mechanism.py``; every compute step runs in
``libropeslr_b200.so`` (include/ropeslr_b200.h).  Differences from the
reference signature, all at the drop-in boundary:

* the op consumes already-projected, RoPE-rotated Q/K/V ``[B, H, L, d]`` plus
  the token features X ``[B, L, H*d]`` (the frozen projections and the
  rotation are the caller's step; ``forward_from_x`` performs them on the
  device for callers that hold the reference's ``(x, backbone)`` pair);
* tensors are batched over B and all heads at once (the reference loops
  over heads, mechanism.py:498-499, 439-452);
* ``SparseSettings`` adds a fixed ``topk`` rule next to the cumulative-mass
  ``keep`` rule, and accepts a flat token block (ragged last block) next to
  the reference's 3D tiles;
* the 3D absolute PE is given as three per-axis tables; ``PETables.sinusoidal``
  reproduces the reference's ``build_pe3d`` exactly.

Bad shapes, ranges and dtypes raise ``ValueError`` like the reference.
"""

from __future__ import annotations

import math
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence, Tuple, Union

import numpy as np
import torch

from . import _lib
from .rope3d import AXES, GridShape, RopeConfig, rotate_rows

RMS_EPS = 1e-6  # mechanism.py:24

BlockSpec = Union[int, Tuple[int, int, int]]


# ---------------------------------------------------------------------------
# settings and parameters


@dataclass(frozen=True)
class SparseSettings:
    """Block partition and selection rule (mechanism.py:258-270).

    block: flat token count (contiguous blocks, ragged last block) or a 3D
        tile ``(b_t, b_x, b_y)`` that must divide the grid (mechanism.py:280-287).
    keep:  cumulative block-softmax mass kept per query block, in (0, 1]
        (used when ``topk == 0``; the reference rule).
    topk:  when > 0, keep exactly min(topk, n_blocks) key blocks per query block.
    """

    block: BlockSpec
    keep: float = 1.0
    topk: int = 0

    def __post_init__(self):
        if isinstance(self.block, (tuple, list)):
            if len(self.block) != 3 or min(self.block) < 1:
                raise ValueError(f"block dims must be three positive counts, got {self.block}")
            object.__setattr__(self, "block", tuple(int(b) for b in self.block))
        elif int(self.block) < 1:
            raise ValueError(f"block must be a positive token count, got {self.block}")
        if int(self.topk) < 0:
            raise ValueError(f"topk must be non-negative, got {self.topk}")
        if int(self.topk) == 0 and not (0.0 < self.keep <= 1.0):
            raise ValueError(f"keep must lie in (0, 1], got {self.keep}")

    @property
    def block_tokens(self) -> int:
        b = self.block
        return int(b[0] * b[1] * b[2]) if isinstance(b, tuple) else int(b)

    @staticmethod
    def topk_for_sparsity(n_blocks: int, sparsity: float) -> int:
        """k = floor((1 - S) * nb + 1/2), at least one block."""
        if not (0.0 <= sparsity < 1.0):
            raise ValueError(f"sparsity must lie in [0, 1), got {sparsity}")
        return max(1, int(math.floor((1.0 - sparsity) * n_blocks + 0.5)))

    @classmethod
    def for_sparsity(cls, block: int, L: int, sparsity: float) -> "SparseSettings":
        nb = -(-L // block)
        return cls(block=block, topk=cls.topk_for_sparsity(nb, sparsity))


@dataclass(frozen=True)
class ForwardSettings:
    """mechanism.py:387-396."""

    sparse: SparseSettings
    compensator: str = "lowrank"  # "lowrank" or "linear"
    use_pe: bool = True
    rms_eps: float = RMS_EPS

    def __post_init__(self):
        if self.compensator not in ("lowrank", "linear"):
            raise ValueError(f"unknown compensator {self.compensator!r}")
        if not (self.rms_eps > 0.0):
            raise ValueError("eps must be positive")


@dataclass
class MechanismParams:
    """The new parameter set (mechanism.py:100-133), float32 device tensors."""

    w_a: torch.Tensor  # (H, d_h, r)
    w_b: torch.Tensor  # (H, r, d_h)
    alpha: torch.Tensor  # (d_model,)
    w_g: torch.Tensor  # (d_model,)
    b_g: float
    rms_sparse: torch.Tensor  # (d_h,)
    rms_lowrank: torch.Tensor  # (d_h,)

    @property
    def n_heads(self) -> int:
        return self.w_a.shape[0]

    @property
    def d_h(self) -> int:
        return self.w_a.shape[1]

    @property
    def rank(self) -> int:
        return self.w_a.shape[2]

    @property
    def d_model(self) -> int:
        return self.alpha.shape[0]

    def to(self, device) -> "MechanismParams":
        f = lambda t: torch.as_tensor(t, dtype=torch.float32).to(device).contiguous()  # noqa: E731
        return MechanismParams(w_a=f(self.w_a), w_b=f(self.w_b), alpha=f(self.alpha), w_g=f(self.w_g),
                               b_g=float(self.b_g), rms_sparse=f(self.rms_sparse), rms_lowrank=f(self.rms_lowrank))

    @classmethod
    def from_arrays(cls, device="cuda", **arrays) -> "MechanismParams":
        """From a key -> array map (the reference's save_params npz layout,
        mechanism.py:163-176)."""
        return cls(w_a=arrays["w_a"], w_b=arrays["w_b"], alpha=arrays["alpha"], w_g=arrays["w_g"],
                   b_g=float(arrays["b_g"]), rms_sparse=arrays["rms_sparse"],
                   rms_lowrank=arrays["rms_lowrank"]).to(device)

    def heads(self, start: int, stop: int) -> "MechanismParams":
        """The per-head slice owned by a head-parallel rank (alpha/w_g stay global)."""
        return MechanismParams(w_a=self.w_a[start:stop].contiguous(), w_b=self.w_b[start:stop].contiguous(),
                               alpha=self.alpha, w_g=self.w_g, b_g=self.b_g, rms_sparse=self.rms_sparse,
                               rms_lowrank=self.rms_lowrank)


def init_params(n_heads: int, d_h: int, rank: int, seed: int, device="cuda") -> MechanismParams:
    """Same draws as the reference init (mechanism.py:136-152)."""
    if min(n_heads, d_h, rank) < 1:
        raise ValueError("head count, head dim and rank must be positive")
    rng = np.random.default_rng(seed)
    d_model = n_heads * d_h
    return MechanismParams.from_arrays(
        device=device,
        w_a=rng.standard_normal((n_heads, d_h, rank)) / math.sqrt(d_h),
        w_b=rng.standard_normal((n_heads, rank, d_h)) / math.sqrt(rank),
        alpha=np.full(d_model, 0.1), w_g=np.zeros(d_model), b_g=-2.0,
        rms_sparse=np.ones(d_h), rms_lowrank=np.ones(d_h))


@dataclass(frozen=True)
class PETables:
    """Learnable 3D absolute PE as per-axis tables: PE[p] = P_t[t] + P_x[x] + P_y[y]."""

    pe_t: torch.Tensor  # (T, d_model) float32
    pe_x: torch.Tensor  # (H_grid, d_model)
    pe_y: torch.Tensor  # (W_grid, d_model)

    @classmethod
    def sinusoidal(cls, grid: GridShape, d_model: int, cfg: RopeConfig, device="cuda") -> "PETables":
        """Per-axis decomposition of build_pe3d (mechanism.py:183-209): the
        model width is split across axes in proportion to the rotary split and
        each axis block interleaves (sin, cos)(theta_m * coord)."""
        d_h = cfg.d_h
        if d_model % d_h != 0:
            raise ValueError(f"d_model={d_model} is not a multiple of the head dim {d_h}")
        sizes = grid.as_tuple()
        tabs = []
        col = 0
        for ai, axis in enumerate(AXES):
            numer = d_model * cfg.axis_dim(axis)
            if numer % d_h != 0:
                raise ValueError(f"axis block width {numer}/{d_h} is not an integer")
            width = numer // d_h
            if width % 2 != 0:
                raise ValueError(f"axis block width {width} must be even")
            tab = np.zeros((sizes[ai], d_model))
            c = np.arange(sizes[ai], dtype=np.float64)
            for m in range(1, width // 2 + 1):
                theta = cfg.base ** (-2.0 * (m - 1) / width)
                tab[:, col] = np.sin(theta * c)
                tab[:, col + 1] = np.cos(theta * c)
                col += 2
            tabs.append(torch.as_tensor(tab, dtype=torch.float32, device=device))
        return cls(*tabs)

    def dense(self, grid: GridShape) -> torch.Tensor:
        """(L, d_model) float32 table (debug / caller-side use only)."""
        c = grid.coords(self.pe_t.device)
        return self.pe_t[c[:, 0]] + self.pe_x[c[:, 1]] + self.pe_y[c[:, 2]]


@dataclass(frozen=True)
class Backbone:
    """Frozen per-head projections (mechanism.py:47-66), device tensors (H, d_model, d_h)."""

    w_q: torch.Tensor
    w_k: torch.Tensor
    w_v: torch.Tensor

    @property
    def n_heads(self) -> int:
        return self.w_q.shape[0]

    @property
    def d_model(self) -> int:
        return self.w_q.shape[1]

    @property
    def d_h(self) -> int:
        return self.w_q.shape[2]


# ---------------------------------------------------------------------------
# results


@dataclass(frozen=True)
class Selection:
    idx: torch.Tensor        # [B, H, nb, kmax] int32, ascending block ids
    cnt: torch.Tensor        # [B, H, nb] int32
    mask: Optional[torch.Tensor]  # [B, H, nb, nb] bool
    attended: torch.Tensor   # [B, H] int64
    scores: Optional[torch.Tensor]  # [B, H, nb, nb] float64
    kmax: int
    block: int
    perm: Optional[torch.Tensor]  # [L] int32 flat position -> token (3D tiles)


@dataclass(frozen=True)
class BlockSparseResult:
    """mechanism.py:273-277, batched: output [B,H,L,d] float32, selected
    [B,H,nb,nb] bool, sparsity [B,H] = 1 - attended / L^2."""

    output: torch.Tensor
    selected: torch.Tensor
    sparsity: torch.Tensor
    selection: Selection = field(repr=False, default=None)


@dataclass(frozen=True)
class ForwardTrace:
    """mechanism.py:399-408 (batched).  output [B, L, H*d] in the input dtype;
    o_sparse / o_lowrank [B, H, L, d] float32; g [B, L] float32."""

    output: torch.Tensor
    o_sparse: Optional[torch.Tensor]
    o_lowrank: Optional[torch.Tensor]
    g: torch.Tensor
    sparsity: torch.Tensor
    selected: Optional[torch.Tensor]
    attended: torch.Tensor


# ---------------------------------------------------------------------------
# helpers


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.BF16
    if t.dtype == torch.float32:
        return _lib.F32
    raise ValueError(f"unsupported dtype {t.dtype}; expected bfloat16 or float32")


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _check_qkv(*ts: torch.Tensor):
    q = ts[0]
    if q.dim() != 4:
        raise ValueError(f"expected [B, H, L, d] tensors, got shape {tuple(q.shape)}")
    for t in ts:
        if t.shape != q.shape:
            raise ValueError(f"Q/K/V shapes differ: {tuple(t.shape)} vs {tuple(q.shape)}")
        if t.dtype != q.dtype:
            raise ValueError("Q/K/V dtypes differ")
        if not t.is_cuda or t.device != q.device:
            raise ValueError("Q/K/V must be CUDA tensors on one device")
    _dtype_code(q)


def _shape(q: torch.Tensor, block: int) -> _lib.Shape:
    B, H, L, d = q.shape
    return _lib.Shape(B, H, L, d, block, _dtype_code(q))


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def block_layout(L: int, settings: SparseSettings, grid: Optional[GridShape], device) -> Tuple[int, Optional[torch.Tensor]]:
    """(tokens per block, permutation or None).  3D tiles are served by
    permuting tokens tile-major (stable, so block ids keep the reference's
    numbering, mechanism.py:280-287) and running flat blocks."""
    if not isinstance(settings.block, tuple):
        return settings.block, None
    if grid is None:
        raise ValueError("a 3D block needs the grid shape")
    if grid.size != L:
        raise ValueError(f"grid size {grid.size} != sequence length {L}")
    b_t, b_x, b_y = settings.block
    if grid.t % b_t or grid.h % b_x or grid.w % b_y:
        raise ValueError(f"block dims {settings.block} do not divide grid {(grid.t, grid.h, grid.w)}")
    n_x, n_y = grid.h // b_x, grid.w // b_y
    c = grid.coords(device)
    ids = (c[:, 0] // b_t) * (n_x * n_y) + (c[:, 1] // b_x) * n_y + (c[:, 2] // b_y)
    perm = torch.sort(ids, stable=True).indices.to(torch.int32)
    if bool(torch.all(perm == torch.arange(L, device=device, dtype=torch.int32))):
        perm = None
    return b_t * b_x * b_y, perm


# ---------------------------------------------------------------------------
# K1: selection


def select_blocks(q: torch.Tensor, k: torch.Tensor, settings: SparseSettings, grid: Optional[GridShape] = None,
                  *, want_mask: bool = True, want_scores: bool = False, _layout=None,
                  pooled: Optional[torch.Tensor] = None, nonfinite: Optional[torch.Tensor] = None) -> Selection:
    """Block routing of block_sparse_attention (mechanism.py:305-320).
    ``pooled`` ([2, B*H, nb, d] float64 block means, e.g. from ``rope_pool``)
    skips the pooling stage."""
    _check_qkv(q, k)
    B, H, L, d = q.shape
    block, perm = _layout if _layout is not None else block_layout(L, settings, grid, q.device)
    if perm is not None and _layout is None:
        q = q.index_select(2, perm.long())
        k = k.index_select(2, perm.long())
    q, k = q.contiguous(), k.contiguous()
    nb = -(-L // block)
    kmax = min(int(settings.topk), nb) if settings.topk > 0 else nb
    dev = q.device
    idx = torch.empty((B, H, nb, kmax), dtype=torch.int32, device=dev)
    cnt = torch.empty((B, H, nb), dtype=torch.int32, device=dev)
    mask = torch.empty((B, H, nb, nb), dtype=torch.uint8, device=dev) if want_mask else None
    attended = torch.empty((B, H), dtype=torch.int64, device=dev)
    scores = torch.empty((B, H, nb, nb), dtype=torch.float64, device=dev) if want_scores else None
    shp = _shape(q, block)
    sel = _lib.SelectParams(int(settings.topk), float(settings.keep), _ptr(nonfinite))
    if pooled is not None:
        if pooled.shape != (2, B * H, nb, d) or pooled.dtype != torch.float64 or not pooled.is_contiguous():
            raise ValueError(f"pooled must be contiguous float64 [2, {B * H}, {nb}, {d}]")
        ws = _workspace(_lib.lib().ropeslr_select_pooled_workspace_bytes(ctypes_ref(shp)), dev)
        _lib.call("ropeslr_select_from_pooled", ctypes_ref(shp), ctypes_ref(sel), pooled.data_ptr(), idx.data_ptr(),
                  kmax, cnt.data_ptr(), _ptr(mask), attended.data_ptr(), _ptr(scores), ws.data_ptr(), ws.numel(),
                  _stream(dev))
    else:
        ws = _workspace(_lib.lib().ropeslr_select_workspace_bytes(ctypes_ref(shp)), dev)
        _lib.call("ropeslr_select_blocks", ctypes_ref(shp), ctypes_ref(sel), q.data_ptr(), k.data_ptr(),
                  idx.data_ptr(), kmax, cnt.data_ptr(), _ptr(mask), attended.data_ptr(), _ptr(scores), ws.data_ptr(),
                  ws.numel(), _stream(dev))
    return Selection(idx=idx, cnt=cnt, mask=None if mask is None else mask.bool(), attended=attended,
                     scores=scores, kmax=kmax, block=block, perm=perm)


def ctypes_ref(obj):
    import ctypes

    return ctypes.byref(obj)


def rope_pool(q: torch.Tensor, k: torch.Tensor, grid: GridShape, cfg: RopeConfig, block: int):
    """Fused 3D RoPE + block pooling (the pre-pass of K1): un-rotated Q/K
    [B, H, L, d] -> rotated Q/K (same dtype; rope3d.py:102-143, computed like
    ``rope3d.rotate_rows`` then cast) and the float64 block means of the
    rotated values, [2, B*H, nb, d] (mechanism.py:306-308), in one pass."""
    _check_qkv(q, k)
    B, H, L, d = q.shape
    if grid.size != L:
        raise ValueError(f"grid size {grid.size} != sequence length {L}")
    if cfg.d_h != d:
        raise ValueError(f"rotary split {cfg.split} does not sum to the head dim {d}")
    if isinstance(block, tuple) or int(block) < 1:
        raise ValueError("rope_pool takes a flat token block")
    q, k = q.contiguous(), k.contiguous()
    nb = -(-L // int(block))
    q_out, k_out = torch.empty_like(q), torch.empty_like(k)
    pooled = torch.empty((2, B * H, nb, d), dtype=torch.float64, device=q.device)
    shp = _shape(q, int(block))
    ra = _lib.RopeArgs(cfg.d_t, cfg.d_x, cfg.d_y, grid.t, grid.h, grid.w, float(cfg.base))
    ws = _workspace(_lib.lib().ropeslr_rope_pool_workspace_bytes(ctypes_ref(ra)), q.device)
    _lib.call("ropeslr_rope_pool", ctypes_ref(shp), ctypes_ref(ra), q.data_ptr(), k.data_ptr(), q_out.data_ptr(),
              k_out.data_ptr(), pooled.data_ptr(), ws.data_ptr(), ws.numel(), _stream(q.device))
    return q_out, k_out, pooled


# ---------------------------------------------------------------------------
# K2: sparse branch


def block_sparse_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, settings: SparseSettings,
                           grid: Optional[GridShape] = None, *, impl: str = "auto",
                           want_mask: bool = True) -> BlockSparseResult:
    """Sparse branch of every head (mechanism.py:290-328) on post-RoPE Q/K/V
    [B, H, L, d]: block routing, then exact softmax attention over the
    selected key blocks.  Returns float32 outputs [B, H, L, d]."""
    _check_qkv(q, k, v)
    B, H, L, d = q.shape
    layout = block_layout(L, settings, grid, q.device)
    block, perm = layout
    if perm is not None:
        pl = perm.long()
        q, k, v = q.index_select(2, pl), k.index_select(2, pl), v.index_select(2, pl)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    sel = select_blocks(q, k, settings, want_mask=want_mask, _layout=layout)
    out = torch.empty((B, H, L, d), dtype=torch.float32, device=q.device)
    shp = _shape(q, block)
    _lib.call("ropeslr_sparse_attention", ctypes_ref(shp), q.data_ptr(), k.data_ptr(), v.data_ptr(),
              sel.idx.data_ptr(), sel.kmax, sel.cnt.data_ptr(), _ptr(perm), out.data_ptr(), _lib.IMPL[impl],
              _stream(q.device))
    sparsity = 1.0 - sel.attended.to(torch.float64) / float(L) ** 2
    return BlockSparseResult(output=out, selected=sel.mask, sparsity=sparsity, selection=sel)


# ---------------------------------------------------------------------------
# K3: compensators and gate


def _token_args(x: torch.Tensor, grid: GridShape, params: MechanismParams, pe: Optional[PETables], use_pe: bool,
                head_offset: int, H_local: int, d: int, nonfinite: Optional[torch.Tensor] = None,
                check_grid: bool = True) -> _lib.TokenArgs:
    if x.dim() != 3:
        raise ValueError(f"expected X of shape [B, L, H*d], got {tuple(x.shape)}")
    B, L, W = x.shape
    if W != H_local * d:
        raise ValueError(f"X has {W} columns, expected {H_local * d}")
    if x.stride(2) != 1 or (B > 1 and x.stride(0) != L * x.stride(1)):
        raise ValueError("X rows must be unit-stride with batch stride L * row stride")
    if check_grid and grid.size != L:
        raise ValueError(f"grid size {grid.size} != sequence length {L}")
    if params.d_model < (head_offset + H_local) * d:
        raise ValueError("alpha / w_g are narrower than the head slice")
    if use_pe:
        if pe is None:
            raise ValueError("use_pe needs the PE tables")
        for tab, n in ((pe.pe_t, grid.t), (pe.pe_x, grid.h), (pe.pe_y, grid.w)):
            if tab.shape != (n, params.d_model) or tab.dtype != torch.float32 or not tab.is_contiguous():
                raise ValueError("PE tables must be contiguous float32 [grid axis, d_model]")
    return _lib.TokenArgs(x.data_ptr(), x.stride(1), head_offset, params.d_model, grid.t, grid.h, grid.w,
                          int(bool(use_pe)), _ptr(pe.pe_t) if use_pe else None, _ptr(pe.pe_x) if use_pe else None,
                          _ptr(pe.pe_y) if use_pe else None, params.alpha.data_ptr(), params.w_g.data_ptr(),
                          _ptr(nonfinite))


_TABLES: "OrderedDict[tuple, tuple]" = OrderedDict()  # key -> (tables, dependencies)


def linear_tables(x: torch.Tensor, grid: GridShape, params: MechanismParams, pe: Optional[PETables], use_pe: bool,
                  lin_weights: Sequence[torch.Tensor], head_offset: int = 0, H_local: Optional[int] = None
                  ) -> torch.Tensor:
    """The parameter-only PE fold of the linear compensator (x_hat W = x W +
    (alpha * PE) W as per-axis tables, include/ropeslr_b200.h
    ropeslr_linear_tables), cached while alpha / the PE tables / the backbone
    weights / w_g are unchanged (keyed on storage and version counters)."""
    H = params.n_heads if H_local is None else H_local
    d = params.d_h
    B, L, _ = x.shape
    tok = _token_args(x, grid, params, pe, use_pe, head_offset, H, d)
    shp = _lib.Shape(B, H, L, d, 1, _dtype_code(x))
    nbytes = _lib.lib().ropeslr_linear_tables_bytes(ctypes_ref(shp), ctypes_ref(tok))
    if nbytes == 0:
        raise ValueError("the PE-injecting linear compensator runs bf16 with d_h = 128 on grids whose "
                         "T + H + W tables fit in shared memory; pass x_hat projections instead")
    wq, wk, wv = (w.contiguous() for w in lin_weights)
    for w in (wq, wk, wv):
        if w.shape != (H, params.d_model, d) or w.dtype != torch.float32 or w.device != x.device:
            raise ValueError(f"linear backbone weights must be float32 [{H}, {params.d_model}, {d}] on X's device")
    deps = [params.alpha, params.w_g, wq, wk, wv] + ([pe.pe_t, pe.pe_x, pe.pe_y] if use_pe else [])

    def build(tab):
        _lib.call("ropeslr_linear_tables", ctypes_ref(shp), ctypes_ref(tok), wq.data_ptr(), wk.data_ptr(),
                  wv.data_ptr(), tab.data_ptr(), tab.numel(), _stream(x.device))

    return _cached_tables(("linear", head_offset, H, grid.as_tuple(), bool(use_pe), x.device), deps, nbytes,
                          x.device, build)


def _cached_tables(tag, deps, nbytes, device, build) -> torch.Tensor:
    """Parameter-only device tables, rebuilt only when a dependency changes.
    The key is each dependency's storage address and version counter; the
    entry holds the dependencies themselves, so a cached address cannot be
    freed and reused by another tensor while the entry lives (64 entries: a
    30-block DiT keeps one per block and tensor kind)."""
    key = (tag, tuple((t.data_ptr(), t._version) for t in deps))
    hit = _TABLES.get(key)
    if hit is not None:
        _TABLES.move_to_end(key)
        return hit[0]
    tab = _workspace(nbytes, device)
    build(tab)
    _TABLES[key] = (tab, list(deps))
    while len(_TABLES) > 64:
        _TABLES.popitem(last=False)
    return tab


def lowrank_tables(x: torch.Tensor, grid: GridShape, params: MechanismParams, pe: Optional[PETables], use_pe: bool,
                   head_offset: int = 0, H_local: Optional[int] = None) -> Optional[torch.Tensor]:
    """The low-rank branch's parameter-only tables (operand images of W_A /
    W_B and the per-axis PE folds, include/ropeslr_b200.h
    ropeslr_lowrank_tables), cached while w_a / w_b / alpha / w_g / the PE
    tables are unchanged; None where the tcgen05 path does not apply."""
    H = params.n_heads if H_local is None else H_local
    d = params.d_h
    B, L, _ = x.shape
    tok = _token_args(x, grid, params, pe, use_pe, head_offset, H, d)
    shp = _lib.Shape(B, H, L, d, 1, _dtype_code(x))
    nbytes = _lib.lib().ropeslr_lowrank_tables_bytes(ctypes_ref(shp), ctypes_ref(tok), params.rank)
    if nbytes == 0:
        return None
    deps = [params.w_a, params.w_b, params.alpha, params.w_g] + ([pe.pe_t, pe.pe_x, pe.pe_y] if use_pe else [])

    def build(tab):
        _lib.call("ropeslr_lowrank_tables", ctypes_ref(shp), ctypes_ref(tok), params.w_a.data_ptr(),
                  params.w_b.data_ptr(), params.rank, tab.data_ptr(), tab.numel(), _stream(x.device))

    return _cached_tables(("lowrank", head_offset, H, grid.as_tuple(), bool(use_pe), x.device), deps, nbytes,
                          x.device, build)


def compensator_branch(x: torch.Tensor, grid: GridShape, params: MechanismParams, settings: ForwardSettings,
                       pe: Optional[PETables] = None, *, head_offset: int = 0,
                       lin_proj: Optional[Sequence[torch.Tensor]] = None, want_o_lr: bool = False,
                       H_local: Optional[int] = None, nonfinite: Optional[torch.Tensor] = None,
                       lin_weights: Optional[Sequence[torch.Tensor]] = None,
                       want_state: bool = False):
    """Low-rank (mechanism.py:225-235, 441-446) or linear (mechanism.py:350-362)
    compensator of the local heads, RMS-normalised with rms_lowrank, plus the
    gate logits over the local columns (mechanism.py:434).

    Linear mode takes the backbone projections in ``lin_proj`` (q, k, v
    [B, H, L, d]).  With ``lin_weights`` (the local heads' W_q, W_k, W_v,
    float32 [H, D_total, d]) they are the projections of the plain X
    (x W, no PE) and the kernels add the PE part from folded tables (the
    tcgen05 path, bf16 with d = 128); without, they are the caller's x_hat W.

    Returns (y_lr [B, L, H, d] in X's dtype, o_lr [B, H, L, d] float32 or None,
    g_logit [B, L] float32 without bias), plus the linear state (S | z,
    float32 [B*H, d, 144]) when ``want_state``."""
    H = params.n_heads if H_local is None else H_local
    d = params.d_h
    B, L, _ = x.shape
    dev = x.device
    tok = _token_args(x, grid, params, pe, settings.use_pe, head_offset, H, d, nonfinite)
    shp = _lib.Shape(B, H, L, d, 1, _dtype_code(x))
    y_lr = torch.empty((B, L, H, d), dtype=x.dtype, device=dev)
    o_lr = torch.empty((B, H, L, d), dtype=torch.float32, device=dev) if want_o_lr else None
    g_logit = torch.empty((B, L), dtype=torch.float32, device=dev)
    state = None
    st = _stream(dev)
    if settings.compensator == "lowrank":
        if params.w_a.shape[0] != H or params.w_b.shape != (H, params.rank, d):
            raise ValueError("compensator weights do not match the head slice")
        tab = lowrank_tables(x, grid, params, pe, settings.use_pe, head_offset, H)
        if tab is not None:
            # parameter-only folds cached across calls: one kernel (+ the gate sum) per call
            ws = _workspace(B * H * L * 4, dev)
            _lib.call("ropeslr_lowrank_branch_folded", ctypes_ref(shp), ctypes_ref(tok), params.rank,
                      tab.data_ptr(), tab.numel(), params.rms_lowrank.data_ptr(), float(settings.rms_eps),
                      y_lr.data_ptr(), _ptr(o_lr), g_logit.data_ptr(), ws.data_ptr(), ws.numel(), st)
        else:
            ws = _workspace(_lib.lib().ropeslr_lowrank_workspace_bytes(ctypes_ref(shp), ctypes_ref(tok),
                                                                       params.rank), dev)
            _lib.call("ropeslr_lowrank_branch", ctypes_ref(shp), ctypes_ref(tok), params.w_a.data_ptr(),
                      params.w_b.data_ptr(), params.rank, params.rms_lowrank.data_ptr(), float(settings.rms_eps),
                      y_lr.data_ptr(), _ptr(o_lr), g_logit.data_ptr(), ws.data_ptr(), ws.numel(), st)
    else:
        if lin_proj is None:
            raise ValueError("the linear compensator needs the projections (q_lin, k_lin, v_lin)")
        ql, kl, vl = (t.contiguous() for t in lin_proj)
        for t in (ql, kl, vl):
            if t.shape != (B, H, L, d) or t.dtype != x.dtype or t.device != dev:
                raise ValueError("linear projections must be [B, H, L, d] in X's dtype on X's device")
        if lin_weights is not None:
            tab = linear_tables(x, grid, params, pe, settings.use_pe, lin_weights, head_offset, H)
            if want_state:
                state = torch.empty((B * H, d, 144), dtype=torch.float32, device=dev)
            ws = _workspace(_lib.lib().ropeslr_linear_pe_workspace_bytes(ctypes_ref(shp), ctypes_ref(tok)), dev)
            _lib.call("ropeslr_linear_branch_pe", ctypes_ref(shp), ctypes_ref(tok), ql.data_ptr(), kl.data_ptr(),
                      vl.data_ptr(), tab.data_ptr(), params.rms_lowrank.data_ptr(), float(settings.rms_eps),
                      y_lr.data_ptr(), _ptr(o_lr), g_logit.data_ptr(), _ptr(state), ws.data_ptr(), ws.numel(), st)
        else:
            _lib.call("ropeslr_gate_logits", ctypes_ref(shp), ctypes_ref(tok), g_logit.data_ptr(), st)
            ws = _workspace(_lib.lib().ropeslr_linear_workspace_bytes(ctypes_ref(shp)), dev)
            _lib.call("ropeslr_linear_branch", ctypes_ref(shp), ql.data_ptr(), kl.data_ptr(), vl.data_ptr(),
                      params.rms_lowrank.data_ptr(), float(settings.rms_eps), y_lr.data_ptr(), _ptr(o_lr),
                      ws.data_ptr(), ws.numel(), st)
    if want_state:
        return y_lr, o_lr, g_logit, state
    return y_lr, o_lr, g_logit


def lowrank_compensator(x: torch.Tensor, grid: GridShape, params: MechanismParams, pe: Optional[PETables] = None,
                        use_pe: bool = True) -> torch.Tensor:
    """Raw compensator outputs sigmoid(sigmoid(x_hat_h W_A[h]) W_B[h]) of every
    head, [B, H, L, d] float32 (mechanism.py:225-235 with the PE injection of
    mechanism.py:429-432)."""
    st = ForwardSettings(SparseSettings(1, topk=1), use_pe=use_pe)
    return compensator_branch(x, grid, params, st, pe, want_o_lr=True)[1]


def gate(x: torch.Tensor, grid: GridShape, params: MechanismParams, pe: Optional[PETables] = None,
         use_pe: bool = True) -> torch.Tensor:
    """g = sigmoid(x_hat . w_g + b_g), [B, L] float32 (mechanism.py:249-255)."""
    H, d = params.d_model // params.d_h, params.d_h
    tok = _token_args(x, grid, params, pe, use_pe, 0, H, d)
    B, L, _ = x.shape
    shp = _lib.Shape(B, H, L, d, 1, _dtype_code(x))
    g = torch.empty((B, L), dtype=torch.float32, device=x.device)
    _lib.call("ropeslr_gate_logits", ctypes_ref(shp), ctypes_ref(tok), g.data_ptr(), _stream(x.device))
    return torch.sigmoid(g + params.b_g)


# ---------------------------------------------------------------------------
# the fused forward


@dataclass
class Prepared:
    """Device state between the two halves of the forward: the routing (K1)
    and the compensator / gate (K3) outputs consumed by the fused attention."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    sel: Selection
    y_lr: torch.Tensor
    o_lr: Optional[torch.Tensor]
    g_logit: torch.Tensor
    block: int
    perm: Optional[torch.Tensor]


def prepare(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, x: torch.Tensor, grid: GridShape,
            params: MechanismParams, settings: ForwardSettings, pe: Optional[PETables] = None, *,
            lin_proj: Optional[Sequence[torch.Tensor]] = None, trace: bool = False,
            head_offset: int = 0, rope: Optional[RopeConfig] = None,
            nonfinite: Optional[torch.Tensor] = None,
            lin_weights: Optional[Sequence[torch.Tensor]] = None) -> Prepared:
    """K1 (routing, mechanism.py:305-320) and K3 (compensator + partial gate
    logits, mechanism.py:429-447) for the local heads.  With ``rope`` the
    given Q/K are un-rotated: the fused RoPE + pooling pre-pass rotates them
    (rope3d.py:102-143) and feeds its block means straight to the selection."""
    _check_qkv(q, k, v)
    B, H, L, d = q.shape
    if x.dtype != q.dtype:
        raise ValueError("X must have the dtype of Q/K/V")
    if params.d_h != d or params.w_a.shape[0] != H:
        raise ValueError("parameters do not match the head count / head dim")
    layout = block_layout(L, settings.sparse, grid, q.device)
    block, perm = layout
    pooled = None
    if rope is not None:
        if perm is not None:
            raise ValueError("the fused RoPE pre-pass takes flat blocks")
        q, k, pooled = rope_pool(q, k, grid, rope, block)
    if perm is not None:
        pl = perm.long()
        q, k, v = q.index_select(2, pl), k.index_select(2, pl), v.index_select(2, pl)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    sel = select_blocks(q, k, settings.sparse, want_mask=trace, _layout=layout, pooled=pooled, nonfinite=nonfinite)
    y_lr, o_lr, g_logit = compensator_branch(x, grid, params, settings, pe, head_offset=head_offset,
                                             lin_proj=lin_proj, want_o_lr=trace, H_local=H, nonfinite=nonfinite,
                                             lin_weights=lin_weights)
    return Prepared(q=q, k=k, v=v, sel=sel, y_lr=y_lr, o_lr=o_lr, g_logit=g_logit, block=block, perm=perm)


def attend_workspace(prep: Prepared, impl: str = "auto") -> torch.Tensor:
    """A workspace for attend() (include/ropeslr_b200.h ropeslr_attend_fused);
    pass it as ``workspace`` to reuse it and to read fallback_units()."""
    shp = _shape(prep.q, prep.block)
    return _workspace(_lib.lib().ropeslr_attend_workspace_bytes(ctypes_ref(shp), _lib.IMPL[impl]), prep.q.device)


def fallback_units(prep: Prepared, workspace: torch.Tensor) -> int:
    """(head, query block) units of the last attend() on `workspace` whose
    fixed exponent reference failed and which the running-max kernel
    recomputed (the workspace's int32 at [2 NU], NU = B * H * nb; tcgen05
    path).  Synchronises."""
    B, H, L, d = prep.q.shape
    nu = B * H * (-(-L // prep.block))
    return int(workspace[:4 * (2 * nu + 1)].view(torch.int32)[2 * nu].item())


def attend(prep: Prepared, params: MechanismParams, settings: ForwardSettings, *, impl: str = "auto",
           want_o_sparse: bool = False, out: Optional[torch.Tensor] = None, out_dtype: Optional[torch.dtype] = None,
           workspace: Optional[torch.Tensor] = None, q_blocks: Optional[Tuple[int, int]] = None):
    """K2 + K4: block-sparse attention with the fused RMSNorm / gate / combine
    epilogue (mechanism.py:321-326, 435-451).  Returns (out [B, L, H*d],
    o_sparse [B, H, L, d] float32 or None).  out_dtype: Q's dtype (default)
    or torch.float32 (the fused result before any bf16 rounding).
    ``q_blocks=(qb0, qb1)`` computes only those query blocks of every head
    (their output rows; the rest of ``out`` is left as it was): a share of a
    head for a sequence-parallel rank (ulysses.py)."""
    q = prep.q
    B, H, L, d = q.shape
    dev = q.device
    if out_dtype is None:
        out_dtype = out.dtype if out is not None else q.dtype
    if out_dtype not in (q.dtype, torch.float32):
        raise ValueError(f"out_dtype must be {q.dtype} or torch.float32, got {out_dtype}")
    if out is None:
        out = torch.empty((B, L, H, d), dtype=out_dtype, device=dev)
    else:
        if tuple(out.shape) not in ((B, L, H, d), (B, L, H * d)):
            raise ValueError(f"out must have shape {(B, L, H, d)} or {(B, L, H * d)}, got {tuple(out.shape)}")
        if out.dtype != out_dtype or out.device != dev or not out.is_contiguous():
            raise ValueError("out must be a contiguous tensor of out_dtype on Q's device")
    o_sparse = torch.empty((B, H, L, d), dtype=torch.float32, device=dev) if want_o_sparse else None
    shp = _shape(q, prep.block)
    if q_blocks is not None:
        nb = -(-L // prep.block)
        qb0, qb1 = (int(b) for b in q_blocks)
        if not (0 <= qb0 < qb1 <= nb):
            raise ValueError(f"q_blocks must satisfy 0 <= qb0 < qb1 <= {nb}, got {q_blocks}")
        if prep.perm is not None:
            raise ValueError("q_blocks takes flat blocks")
        shp.qb_begin, shp.qb_end = qb0, qb1
    impl_code = _lib.IMPL[impl]
    ws = workspace
    if ws is None or ws.numel() < _lib.lib().ropeslr_attend_workspace_bytes(ctypes_ref(shp), impl_code):
        ws = _workspace(_lib.lib().ropeslr_attend_workspace_bytes(ctypes_ref(shp), impl_code), dev)
    _lib.call("ropeslr_attend_fused", ctypes_ref(shp), q.data_ptr(), prep.k.data_ptr(), prep.v.data_ptr(),
              prep.sel.idx.data_ptr(), prep.sel.kmax, prep.sel.cnt.data_ptr(), _ptr(prep.perm), prep.y_lr.data_ptr(),
              prep.g_logit.data_ptr(), float(params.b_g), params.rms_sparse.data_ptr(), float(settings.rms_eps),
              out.data_ptr(), _dtype_code(out), _ptr(o_sparse), impl_code, ws.data_ptr(), ws.numel(), _stream(dev))
    return out.view(B, L, H * d), o_sparse


def forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, x: torch.Tensor, grid: GridShape,
            params: MechanismParams, settings: ForwardSettings, pe: Optional[PETables] = None, *,
            lin_proj: Optional[Sequence[torch.Tensor]] = None, trace: bool = False, impl: str = "auto",
            head_offset: int = 0, gate_reduce: Optional[Callable[[torch.Tensor], None]] = None,
            rope: Optional[RopeConfig] = None, check_finite: bool = False,
            out_dtype: Optional[torch.dtype] = None, lin_weights: Optional[Sequence[torch.Tensor]] = None,
            q_blocks: Optional[Tuple[int, int]] = None, out: Optional[torch.Tensor] = None):
    """RoPeSLR forward (mechanism.py:491-512, Algorithm 1).

    q, k, v: post-RoPE [B, H, L, d] (bf16 or f32); x: token features
    [B, L, H*d] of the same dtype (may be a column slice of a wider X for a
    head-parallel rank, with ``head_offset`` its first global head and
    ``gate_reduce`` an in-place all-reduce of the partial gate logits).
    With ``rope`` (a RopeConfig), q and k are the un-rotated projections and
    the fused RoPE + pooling pre-pass rotates them on the way in.

    With ``check_finite`` a NaN or infinite value in Q, K or X raises
    ValueError like the reference (linalg.py:17-20); the kernels flag it on
    values they already reduce (block means, gate logits), and the check
    costs one 4-byte read-back (a stream synchronisation).

    Linear compensator: ``lin_proj`` holds the backbone projections (q, k, v);
    with ``lin_weights`` (W_q, W_k, W_v of the local heads, float32
    [H, D_total, d]) they are x W and the PE part is added in the kernels
    (see compensator_branch), else they are x_hat W.

    ``q_blocks=(qb0, qb1)`` runs the sparse attention for those query
    blocks only (rows outside are left as ``out`` holds them).

    ``out_dtype=torch.float32`` returns the fused output in float32 (the
    epilogue's result before the bf16 rounding of a bf16 output).

    Returns the output [B, L, H*d] (x's dtype), or a ForwardTrace when
    ``trace`` (adds the float32 branch outputs, the gate and the masks)."""
    flag = torch.zeros(1, dtype=torch.int32, device=q.device) if check_finite else None
    prep = prepare(q, k, v, x, grid, params, settings, pe, lin_proj=lin_proj, trace=trace, head_offset=head_offset,
                   rope=rope, nonfinite=flag, lin_weights=lin_weights)
    if flag is not None:
        raise_nonfinite(flag)
    if gate_reduce is not None:
        gate_reduce(prep.g_logit)
    out, o_sparse = attend(prep, params, settings, impl=impl, want_o_sparse=trace, out_dtype=out_dtype,
                           q_blocks=q_blocks, out=out)
    if not trace:
        return out
    L = q.shape[2]
    sparsity = 1.0 - prep.sel.attended.to(torch.float64) / float(L) ** 2
    return ForwardTrace(output=out, o_sparse=o_sparse, o_lowrank=prep.o_lr, g=torch.sigmoid(prep.g_logit + params.b_g),
                        sparsity=sparsity, selected=prep.sel.mask, attended=prep.sel.attended)


def raise_nonfinite(flag: torch.Tensor) -> None:
    """ValueError when a kernel flagged non-finite inputs (linalg.py:17-20)."""
    bits = int(flag.item())
    if bits:
        what = [n for b, n in ((_lib.NONFINITE_QK, "Q/K"), (_lib.NONFINITE_X, "X")) if bits & b]
        raise ValueError(f"input contains non-finite values ({', '.join(what)})")


def project_and_rotate(x: torch.Tensor, grid: GridShape, cfg: RopeConfig, backbone: Backbone,
                       dtype: torch.dtype) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Caller-side step of the reference (mechanism.py:301-303): frozen
    projections, 3D RoPE in float64, cast to the op dtype.  Returns [B,H,L,d]."""
    xb = x if x.dim() == 3 else x.unsqueeze(0)
    x64 = xb.to(torch.float64)
    proj = lambda w: torch.einsum("bld,hde->bhle", x64, w.to(torch.float64))  # noqa: E731
    q = rotate_rows(proj(backbone.w_q), grid, cfg).to(dtype)
    k = rotate_rows(proj(backbone.w_k), grid, cfg).to(dtype)
    v = proj(backbone.w_v).to(dtype)
    return q, k, v


def forward_from_x(x: torch.Tensor, grid: GridShape, cfg: RopeConfig, backbone: Backbone, params: MechanismParams,
                   settings: ForwardSettings, pe: Optional[PETables] = None, *, dtype: torch.dtype = torch.float32,
                   trace: bool = True, impl: str = "auto"):
    """Drop-in for the reference ``mechanism.forward(x, grid, cfg, backbone,
    params, settings)`` (mechanism.py:491-512): x is (L, d_model) or
    (B, L, d_model) on the device; projections + RoPE run on the device as
    the caller-side step, then the B200 op.  With ``pe=None`` and
    ``use_pe`` the reference's sinusoidal table is used (mechanism.py:497)."""
    xb = x if x.dim() == 3 else x.unsqueeze(0)
    if xb.shape[1:] != (grid.size, backbone.d_model):
        raise ValueError(f"expected input shape {(grid.size, backbone.d_model)}, got {tuple(xb.shape[1:])}")
    if settings.use_pe and pe is None:
        pe = PETables.sinusoidal(grid, backbone.d_model, cfg, device=xb.device)
    q, k, v = project_and_rotate(xb, grid, cfg, backbone, dtype)
    xd = xb.to(dtype).contiguous()
    lin, lin_w = None, None
    if settings.compensator == "linear":
        # the backbone projections are the caller-side step (like Q/K/V):
        # on the tensor-core path x W of the stored X, and the kernels add
        # the PE part (alpha * PE) W from folded tables; otherwise x_hat W
        tc_path = dtype == torch.bfloat16 and backbone.d_h == 128
        x_src = xd.to(torch.float64) if tc_path else xb.to(torch.float64)
        if settings.use_pe and not tc_path:
            x_src = x_src + params.alpha.to(torch.float64)[None, None, :] * pe.dense(grid).to(torch.float64)[None]
        lin = tuple(torch.einsum("bld,hde->bhle", x_src, w.to(torch.float64)).to(dtype)
                    for w in (backbone.w_q, backbone.w_k, backbone.w_v))
        if tc_path:
            lin_w = tuple(w.to(torch.float32).contiguous() for w in (backbone.w_q, backbone.w_k, backbone.w_v))
    return forward(q, k, v, xd, grid, params, settings, pe, lin_proj=lin, trace=trace, impl=impl, lin_weights=lin_w)


def forward_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, x: torch.Tensor, grid: GridShape,
                 params: MechanismParams, settings: ForwardSettings, pe: Optional[PETables] = None, *,
                 out: Optional[torch.Tensor] = None, head_offset: int = 0,
                 gate_reduce: Optional[Callable[[torch.Tensor], None]] = None, chunk_heads: int = 0,
                 device=None, sync: bool = True, want_attended: bool = False):
    """The forward from HOST tensors, the reference's calling convention
    (NumPy arrays in host memory, mechanism.py:491-512), through the C ABI
    ``ropeslr_forward_host``: the host->device copies of X and of Q/K/V (in
    head chunks) and the device->host copy of each chunk's output overlap the
    kernels.  q, k, v: CPU [B, H, L, d] post-RoPE; x: CPU [B, L, H*d] (or a
    column slice of a wider X); pinned memory gives the overlap.  Low-rank
    compensator only.  Returns out (CPU [B, L, H*d]), plus the attended-pair
    counts [B, H] when ``want_attended``."""
    if settings.compensator != "lowrank":
        raise ValueError("forward_host supports the low-rank compensator")
    if isinstance(settings.sparse.block, tuple):
        raise ValueError("forward_host takes flat blocks; use forward() for 3D tiles")
    for t in (q, k, v, x):
        if t.is_cuda:
            raise ValueError("forward_host takes host tensors; use forward() for device tensors")
    if q.dim() != 4 or k.shape != q.shape or v.shape != q.shape:
        raise ValueError(f"expected host Q/K/V of one shape [B, H, L, d], got {tuple(q.shape)}")
    if not (q.dtype == k.dtype == v.dtype == x.dtype):
        raise ValueError("Q/K/V/X dtypes differ")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    B, H, L, d = q.shape
    if x.dim() != 3 or x.shape[:2] != (B, L) or x.shape[2] < H * d or x.stride(2) != 1:
        raise ValueError(f"expected host X [B, L, >= H*d] with unit column stride, got {tuple(x.shape)}")
    if B > 1 and x.stride(0) != L * x.stride(1):
        raise ValueError("X rows must have batch stride L * row stride")
    if params.d_h != d or params.w_a.shape[0] != H:
        raise ValueError("parameters do not match the head count / head dim")
    dev = torch.device(device) if device is not None else params.w_a.device
    if out is None:
        out = torch.empty((B, L, H * d), dtype=q.dtype, pin_memory=q.is_pinned())
    if out.is_cuda or out.shape[:2] != (B, L) or out.shape[2] < H * d or out.stride(2) != 1 or out.dtype != q.dtype:
        raise ValueError("out must be a host tensor [B, L, >= H*d] of the input dtype")
    attended = torch.zeros((B, H), dtype=torch.int64) if want_attended else None
    flag = torch.zeros(1, dtype=torch.int32, device=dev)  # non-finite inputs (linalg.py:17-20)
    tok = _token_args(x, grid, params, pe, settings.use_pe, head_offset, H, d, flag)
    args = _lib.HostForward()
    args.shape = _lib.Shape(B, H, L, d, settings.sparse.block, _dtype_code(q))
    args.sel = _lib.SelectParams(int(settings.sparse.topk), float(settings.sparse.keep), flag.data_ptr())
    args.q, args.k, args.v = q.data_ptr(), k.data_ptr(), v.data_ptr()
    args.tok = tok
    args.w_a, args.w_b, args.rank = params.w_a.data_ptr(), params.w_b.data_ptr(), params.rank
    args.rms_sparse, args.rms_lowrank = params.rms_sparse.data_ptr(), params.rms_lowrank.data_ptr()
    args.b_g, args.eps = float(params.b_g), float(settings.rms_eps)
    args.out, args.out_row_stride = out.data_ptr(), out.stride(1)
    args.attended = _ptr(attended)
    args.chunk_heads = int(chunk_heads)
    hook, hook_error = None, []
    if gate_reduce is not None:
        def _hook(g_ptr, n, stream_ptr, _user):
            try:
                g = _device_view_f32(g_ptr, n, dev).view(B, L)
                cur = torch.cuda.current_stream(dev)
                if (stream_ptr or 0) == cur.cuda_stream:
                    gate_reduce(g)
                else:
                    with torch.cuda.stream(torch.cuda.ExternalStream(stream_ptr, device=dev)):
                        gate_reduce(g)
            except BaseException as e:  # noqa: BLE001 -- re-raised after the C call returns
                hook_error.append(e)
        hook = _lib.GateHook(_hook)
        args.gate_hook = hook
    ws_bytes = _lib.lib().ropeslr_forward_host_workspace_bytes(ctypes_ref(args))
    if ws_bytes == 0:
        raise ValueError("forward_host: inconsistent arguments")
    with torch.cuda.device(dev):
        ws = _workspace(ws_bytes, dev)
        st = _stream(dev)
        _lib.call("ropeslr_forward_host", ctypes_ref(args), ws.data_ptr(), ws.numel(), st)
        if hook_error:
            torch.cuda.current_stream(dev).synchronize()
            raise hook_error[0]
        if sync:
            torch.cuda.current_stream(dev).synchronize()
            raise_nonfinite(flag)
        else:
            # keep the workspace alive until the stream reaches this point
            ws.record_stream(torch.cuda.current_stream(dev))
    del hook
    return (out, attended) if want_attended else out


def _device_view_f32(ptr: int, n: int, dev) -> torch.Tensor:
    """A float32 tensor over n elements of device memory owned by the caller."""
    class _Buf:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4", "data": (int(ptr), False), "version": 3}

    return torch.as_tensor(_Buf(), device=dev)
