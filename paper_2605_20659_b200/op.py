"""``torch.ops.ropeslr.attn_fwd``: the RoPeSLR forward as a PyTorch custom op
(stream-ordered on the current CUDA stream, fake kernel for tracing)."""

from __future__ import annotations

from typing import List

import torch

from .mechanism import ForwardSettings, MechanismParams, PETables, SparseSettings, forward
from .rope3d import GridShape


@torch.library.custom_op("ropeslr::attn_fwd", mutates_args=())
def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, x: torch.Tensor, pe_t: torch.Tensor,
             pe_x: torch.Tensor, pe_y: torch.Tensor, alpha: torch.Tensor, w_a: torch.Tensor, w_b: torch.Tensor,
             w_g: torch.Tensor, b_g: float, rms_sparse: torch.Tensor, rms_lowrank: torch.Tensor, grid: List[int],
             block: int, topk: int, keep: float, use_pe: bool, eps: float) -> torch.Tensor:
    params = MechanismParams(w_a=w_a.contiguous(), w_b=w_b.contiguous(), alpha=alpha.contiguous(),
                             w_g=w_g.contiguous(), b_g=b_g, rms_sparse=rms_sparse.contiguous(),
                             rms_lowrank=rms_lowrank.contiguous())
    st = ForwardSettings(SparseSettings(block=block, keep=keep, topk=topk), use_pe=use_pe, rms_eps=eps)
    pe = PETables(pe_t.contiguous(), pe_x.contiguous(), pe_y.contiguous())
    return forward(q, k, v, x, GridShape(*grid), params, st, pe)


@attn_fwd.register_fake
def _(q, k, v, x, pe_t, pe_x, pe_y, alpha, w_a, w_b, w_g, b_g, rms_sparse, rms_lowrank, grid, block, topk, keep,
      use_pe, eps):
    B, H, L, d = q.shape
    return q.new_empty((B, L, H * d))
