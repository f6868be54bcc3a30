"""Head-parallel execution across the GPUs of one node.

Heads are independent in selection, sparse attention, compensator and
RMSNorm (mechanism.py:439-452, 498-499); rank r owns heads
[r*H/W, (r+1)*H/W).  The only cross-head coupling is the gate, a dot over
the full model width (mechanism.py:434): each rank computes the partial
logits over its own columns and one all-reduce of a [B, L] float32 vector
(NCCL over NVLink, or gloo in the CPU tests) completes it before the fused
epilogue.  Outputs stay head-sharded [B, L, H/W * d].
"""

from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def head_slice(n_heads: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced head range of `rank` (the first H % W ranks take one extra)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    if n_heads < world:
        raise ValueError(f"{n_heads} heads cannot be split over {world} ranks")
    base, extra = divmod(n_heads, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gate_allreduce(group: Optional[dist.ProcessGroup] = None):
    """In-place sum of the partial gate logits over the head-parallel group."""

    def reduce_(g_logit: torch.Tensor) -> None:
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(g_logit, op=dist.ReduceOp.SUM, group=group)

    return reduce_


def forward_head_parallel(q, k, v, x_full, grid, params, settings, pe=None, *, group=None, impl="auto",
                          trace=False):
    """Run this rank's head slice.  q/k/v: this rank's heads [B, H_local, L, d];
    x_full: [B, L, H_total * d] (only the local columns are read); params:
    full-model parameters (sliced here).  Returns [B, L, H_local * d]."""
    from .mechanism import forward

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    H_total = params.n_heads
    h0, h1 = head_slice(H_total, world, rank)
    if q.shape[1] != h1 - h0:
        raise ValueError(f"rank {rank} owns heads [{h0}, {h1}) but got {q.shape[1]}")
    d = params.d_h
    x_local = x_full[:, :, h0 * d:h1 * d]
    return forward(q, k, v, x_local, grid, params.heads(h0, h1), settings, pe, head_offset=h0,
                   gate_reduce=gate_allreduce(group), impl=impl, trace=trace)
