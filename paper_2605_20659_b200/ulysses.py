"""Sequence-parallel RoPeSLR attention (BASELINE config 4).

In a sequence-sharded model, rank r holds the tokens [L_r0, L_r1) of every
head.  RoPeSLR needs whole sequences per head (block selection looks at all
key blocks), so around the op the layout switches between sequence and head
parallelism with two all-to-alls, as in DeepSpeed-Ulysses:

    Q/K/V [B, L_r, H, d] and X [B, L_r, H*d] on rank r
      --all_to_all-->  Q/K/V [B, H_s, L, d] and X [B, L, H_s*d] on rank s
      --RoPeSLR (head-parallel, gate partials all-reduced)-->
    out [B, L, H_s*d]  --all_to_all-->  out [B, L_r, H*d] on rank r

Heads are split with distributed.head_slice, so H need not divide by the
world size (12 heads on 8 ranks: 2,2,2,2,1,1,1,1); sequence shards are
split the same way (the first L % W ranks take one extra token).  Each
all-to-all is one NCCL all_to_all_single over NVLink with per-peer split
sizes: the payload is packed peer-major in a contiguous buffer, then
unpacked.  The op is injectable so the data movement can be tested on CPU
(gloo) with a reference stand-in.
"""

from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .distributed import head_slice


def seq_slice(L: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous token range of `rank` (the first L % W ranks take one extra)."""
    return head_slice(L, world, rank)


def _world(group) -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _all_to_all(out: torch.Tensor, inp: torch.Tensor, out_splits: List[int], in_splits: List[int], group) -> None:
    world, _ = _world(group)
    if world == 1:
        out.copy_(inp)
        return
    dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=group)


def seq_to_head(ts: Sequence[torch.Tensor], H: int, L: int, group=None) -> List[torch.Tensor]:
    """[B, L_r, H, d] sequence shards -> [B, H_s, L, d] head shards (one
    all-to-all for all tensors of the list)."""
    world, rank = _world(group)
    B, Lr, H_, d = ts[0].shape
    if H_ != H:
        raise ValueError(f"expected {H} heads, got {H_}")
    r0, r1 = seq_slice(L, world, rank)
    if Lr != r1 - r0:
        raise ValueError(f"rank {rank} holds {Lr} tokens, expected {r1 - r0}")
    nt = len(ts)
    h0, h1 = head_slice(H, world, rank)
    Hs = h1 - h0
    # send buffer: peer-major [peer][tensor][B][heads of peer][L_r][d]
    send, in_splits = [], []
    for s in range(world):
        a, b = head_slice(H, world, s)
        chunk = torch.stack([t[:, :, a:b, :].permute(0, 2, 1, 3) for t in ts])  # [nt, B, Hp, L_r, d]
        send.append(chunk.reshape(-1))
        in_splits.append(chunk.numel())
    send = torch.cat(send)
    out_splits = []
    for s in range(world):
        a, b = seq_slice(L, world, s)
        out_splits.append(nt * B * Hs * (b - a) * d)
    recv = torch.empty(sum(out_splits), dtype=ts[0].dtype, device=ts[0].device)
    _all_to_all(recv, send, out_splits, in_splits, group)
    # receive buffer: [peer][tensor][B][H_s][L_peer][d] -> [tensor][B][H_s][L][d]
    outs = torch.empty((nt, B, Hs, L, d), dtype=ts[0].dtype, device=ts[0].device)
    off = 0
    for s in range(world):
        a, b = seq_slice(L, world, s)
        n = out_splits[s]
        outs[:, :, :, a:b, :] = recv[off:off + n].view(nt, B, Hs, b - a, d)
        off += n
    return [outs[i] for i in range(nt)]


def seq_to_head_cols(x: torch.Tensor, H: int, d: int, L: int, group=None) -> torch.Tensor:
    """X [B, L_r, H*d] sequence shard -> [B, L, H_s*d] (the rank's head columns)."""
    B, Lr, D = x.shape
    if D != H * d:
        raise ValueError(f"X has {D} columns, expected {H * d}")
    return seq_to_head([x.view(B, Lr, H, d)], H, L, group)[0].permute(0, 2, 1, 3).reshape(B, L, -1)


def head_to_seq(out: torch.Tensor, H: int, d: int, L: int, group=None) -> torch.Tensor:
    """[B, L, H_s*d] head shard -> [B, L_r, H*d] sequence shard."""
    world, rank = _world(group)
    B = out.shape[0]
    h0, h1 = head_slice(H, world, rank)
    Hs = h1 - h0
    o = out.view(B, L, Hs, d)
    send, in_splits = [], []
    for s in range(world):
        a, b = seq_slice(L, world, s)
        chunk = o[:, a:b].contiguous()  # [B, L_s, H_s, d]
        send.append(chunk.reshape(-1))
        in_splits.append(chunk.numel())
    send = torch.cat(send)
    r0, r1 = seq_slice(L, world, rank)
    Lr = r1 - r0
    out_splits = []
    for s in range(world):
        a, b = head_slice(H, world, s)
        out_splits.append(B * Lr * (b - a) * d)
    recv = torch.empty(sum(out_splits), dtype=out.dtype, device=out.device)
    _all_to_all(recv, send, out_splits, in_splits, group)
    res = torch.empty((B, Lr, H, d), dtype=out.dtype, device=out.device)
    off = 0
    for s in range(world):
        a, b = head_slice(H, world, s)
        n = out_splits[s]
        res[:, :, a:b, :] = recv[off:off + n].view(B, Lr, b - a, d)
        off += n
    return res.view(B, Lr, H * d)


OpFn = Callable[..., torch.Tensor]


def ulysses_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, x: torch.Tensor, grid, params, settings,
                      pe=None, *, group=None, op: Optional[OpFn] = None, rope=None) -> torch.Tensor:
    """RoPeSLR forward on a sequence-sharded rank.

    q, k, v: [B, L_r, H, d] (this rank's tokens, all heads; post-RoPE unless
    ``rope`` is given); x: [B, L_r, H*d]; params: the full model's
    MechanismParams.  Returns this rank's tokens of the output, [B, L_r, H*d].
    ``op(q, k, v, x, grid, params_slice, settings, pe, head_offset=, gate_reduce=, rope=)``
    defaults to mechanism.forward."""
    from .distributed import gate_allreduce
    from .mechanism import forward

    world, rank = _world(group)
    B, Lr, H, d = q.shape
    L = grid.size
    qh, kh, vh = seq_to_head([q, k, v], H, L, group)
    xh = seq_to_head_cols(x, H, d, L, group)
    h0, h1 = head_slice(H, world, rank)
    fn = forward if op is None else op
    reduce_ = gate_allreduce(group) if world > 1 else None
    out = fn(qh.contiguous(), kh.contiguous(), vh.contiguous(), xh.contiguous(), grid, params.heads(h0, h1),
             settings, pe, head_offset=h0, gate_reduce=reduce_, rope=rope)
    return head_to_seq(out, H, d, L, group)
