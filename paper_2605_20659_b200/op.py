"""The RoPeSLR path as PyTorch custom ops (stream-ordered on the current CUDA
stream, fake kernels for tracing):

* ``torch.ops.ropeslr.attn_fwd``        the whole forward (mechanism.forward);
* ``torch.ops.ropeslr.select_blocks``   K1, the block routing (idx, cnt, attended);
* ``torch.ops.ropeslr.compensator_fwd`` K3, the low-rank branch and gate logits."""

from __future__ import annotations

from typing import List, Optional

import torch

from .mechanism import (ForwardSettings, MechanismParams, PETables, SparseSettings, compensator_branch, forward,
                        select_blocks as _select_blocks)
from .rope3d import GridShape


@torch.library.custom_op("ropeslr::attn_fwd", mutates_args=())
def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, x: torch.Tensor, pe_t: torch.Tensor,
             pe_x: torch.Tensor, pe_y: torch.Tensor, alpha: torch.Tensor, w_a: torch.Tensor, w_b: torch.Tensor,
             w_g: torch.Tensor, b_g: float, rms_sparse: torch.Tensor, rms_lowrank: torch.Tensor, grid: List[int],
             block: int, topk: int, keep: float, use_pe: bool, eps: float, compensator: str = "lowrank",
             q_lin: Optional[torch.Tensor] = None, k_lin: Optional[torch.Tensor] = None,
             v_lin: Optional[torch.Tensor] = None, w_lin_q: Optional[torch.Tensor] = None,
             w_lin_k: Optional[torch.Tensor] = None, w_lin_v: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The whole forward.  compensator "linear" takes the backbone projections
    q_lin/k_lin/v_lin [B, H, L, d]: of the plain X when w_lin_q/k/v (float32
    [H, D, d]) are given (the PE part is added in the kernels), else of x_hat."""
    params = MechanismParams(w_a=w_a.contiguous(), w_b=w_b.contiguous(), alpha=alpha.contiguous(),
                             w_g=w_g.contiguous(), b_g=b_g, rms_sparse=rms_sparse.contiguous(),
                             rms_lowrank=rms_lowrank.contiguous())
    st = ForwardSettings(SparseSettings(block=block, keep=keep, topk=topk), compensator=compensator, use_pe=use_pe,
                         rms_eps=eps)
    pe = PETables(pe_t.contiguous(), pe_x.contiguous(), pe_y.contiguous())
    lin = None
    lin_w = None
    if compensator == "linear":
        if q_lin is None or k_lin is None or v_lin is None:
            raise ValueError("the linear compensator needs q_lin, k_lin and v_lin")
        lin = (q_lin, k_lin, v_lin)
        if w_lin_q is not None:
            if w_lin_k is None or w_lin_v is None:
                raise ValueError("w_lin_q, w_lin_k and w_lin_v go together")
            lin_w = (w_lin_q, w_lin_k, w_lin_v)
    return forward(q, k, v, x, GridShape(*grid), params, st, pe, lin_proj=lin, lin_weights=lin_w)


@attn_fwd.register_fake
def _(q, k, v, x, pe_t, pe_x, pe_y, alpha, w_a, w_b, w_g, b_g, rms_sparse, rms_lowrank, grid, block, topk, keep,
      use_pe, eps, compensator="lowrank", q_lin=None, k_lin=None, v_lin=None, w_lin_q=None, w_lin_k=None,
      w_lin_v=None):
    B, H, L, d = q.shape
    return q.new_empty((B, L, H * d))


@torch.library.custom_op("ropeslr::select_blocks", mutates_args=())
def select_blocks(q: torch.Tensor, k: torch.Tensor, block: int, topk: int,
                  keep: float) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """(idx [B, H, nb, kmax] int32 ascending, cnt [B, H, nb] int32, attended
    [B, H] int64) for flat blocks (mechanism.py:305-320)."""
    sel = _select_blocks(q, k, SparseSettings(block=block, keep=keep, topk=topk), want_mask=False)
    return sel.idx, sel.cnt, sel.attended


@select_blocks.register_fake
def _(q, k, block, topk, keep):
    B, H, L, d = q.shape
    nb = -(-L // block)
    kmax = min(topk, nb) if topk > 0 else nb
    return (q.new_empty((B, H, nb, kmax), dtype=torch.int32), q.new_empty((B, H, nb), dtype=torch.int32),
            q.new_empty((B, H), dtype=torch.int64))


@torch.library.custom_op("ropeslr::compensator_fwd", mutates_args=())
def compensator_fwd(x: torch.Tensor, pe_t: torch.Tensor, pe_x: torch.Tensor, pe_y: torch.Tensor, alpha: torch.Tensor,
                    w_a: torch.Tensor, w_b: torch.Tensor, w_g: torch.Tensor, rms_lowrank: torch.Tensor,
                    grid: List[int], use_pe: bool, eps: float) -> tuple[torch.Tensor, torch.Tensor]:
    """(y_lr [B, L, H, d] in X's dtype, g_logit [B, L] float32 without bias):
    the low-rank compensator with its RMSNorm and the gate logits
    (mechanism.py:225-255, 429-447)."""
    H, d = w_a.shape[0], w_a.shape[1]
    params = MechanismParams(w_a=w_a.contiguous(), w_b=w_b.contiguous(), alpha=alpha.contiguous(),
                             w_g=w_g.contiguous(), b_g=0.0, rms_sparse=torch.ones_like(rms_lowrank),
                             rms_lowrank=rms_lowrank.contiguous())
    st = ForwardSettings(SparseSettings(block=1, topk=1), use_pe=use_pe, rms_eps=eps)
    pe = PETables(pe_t.contiguous(), pe_x.contiguous(), pe_y.contiguous())
    y_lr, _, g_logit = compensator_branch(x, GridShape(*grid), params, st, pe, H_local=H)
    return y_lr, g_logit


@compensator_fwd.register_fake
def _(x, pe_t, pe_x, pe_y, alpha, w_a, w_b, w_g, rms_lowrank, grid, use_pe, eps):
    B, L, _ = x.shape
    H, d = w_a.shape[0], w_a.shape[1]
    return x.new_empty((B, L, H, d)), x.new_empty((B, L), dtype=torch.float32)
