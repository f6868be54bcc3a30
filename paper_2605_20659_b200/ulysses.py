"""Sequence-parallel RoPeSLR attention (BASELINE config 4, SURVEY.md 8e/8f,
SURVEY 7 hard part 6).

In a sequence-sharded model rank r holds the tokens [L_r0, L_r1) of every
head.  RoPeSLR needs whole sequences per head (block selection looks at all
key blocks), so around the op the layout switches between sequence and head
parallelism with two all-to-alls, as in DeepSpeed-Ulysses -- but the work is
split by (head x query-block range), not by whole heads:

* the H * nb query blocks of the layer are laid end to end and cut into W
  equal spans (``work_items``); 12 heads on 8 ranks give every rank 1.5
  heads of query blocks (whole heads would give 2,2,2,2,1,1,1,1 and leave
  four ranks idle for half of the attention);
* a head shared by two ranks goes (Q, K, V and its X columns, all tokens)
  to both; each runs the op with ``q_blocks`` = its range, so only its
  query blocks' units run in K2 (K1 / K3 of the shared head run on both, a
  few percent of its cost);
* the gate logit of a token needs every head's X columns
  (mechanism.py:434): each rank computes it for its own tokens over all
  columns before the exchange (ropeslr_gate_logits with a token offset) and
  the logits are exchanged with the data, so no all-reduce is left;
* each all-to-all is one NCCL all_to_all_single over NVLink with per-peer
  split sizes, packed and unpacked by one segmented row-copy kernel each
  (ropeslr_copy_rows); the outbound exchange is posted asynchronously and
  the gate logits are computed while it is in flight.

The op, the gate and the copies are injectable so the data movement can be
tested on CPU (gloo) with stand-ins.
"""

from __future__ import annotations

import ctypes
from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .distributed import head_slice

Item = Tuple[int, int, int]  # (head, first query block, end query block)


def seq_slice(L: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous token range of `rank` (the first L % W ranks take one extra)."""
    return head_slice(L, world, rank)


def work_items(H: int, nb: int, world: int) -> List[List[Item]]:
    """Per rank, its (head, qb0, qb1) pieces of the H * nb query blocks cut
    into `world` contiguous spans of equal size (+-1 block)."""
    if H < 1 or nb < 1 or world < 1:
        raise ValueError(f"bad split: H={H}, nb={nb}, world={world}")
    total = H * nb
    if total < world:
        raise ValueError(f"{total} query blocks cannot be split over {world} ranks")
    out = []
    for r in range(world):
        a, b = r * total // world, (r + 1) * total // world
        items = []
        for h in range(a // nb, (b - 1) // nb + 1):
            qb0, qb1 = max(a - h * nb, 0), min(b - h * nb, nb)
            if qb1 > qb0:
                items.append((h, qb0, qb1))
        out.append(items)
    return out


def heads_of(items: Sequence[Item]) -> List[int]:
    return sorted({h for h, _, _ in items})


def _world(group) -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _all_to_all(out: torch.Tensor, inp: torch.Tensor, out_splits: List[int], in_splits: List[int], group,
                async_op: bool = False):
    """Splits count dim-0 rows of out / inp."""
    world, _ = _world(group)
    if world == 1:
        out.copy_(inp)
        return None
    return dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                  group=group, async_op=async_op)


# ---------------------------------------------------------------- row copies
class Segments:
    """Row-copy segments (src tensor view, dst tensor view) -> one launch of
    ropeslr_copy_rows for CUDA tensors; CPU tensors (the gloo tests) copy
    with torch."""

    def __init__(self):
        self.views: List[Tuple[torch.Tensor, torch.Tensor]] = []

    def add(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        """src, dst: 2-D views [rows, cols] with unit column stride."""
        if src.shape != dst.shape:
            raise ValueError(f"segment shapes differ: {tuple(src.shape)} vs {tuple(dst.shape)}")
        if src.shape[0] > 0:
            self.views.append((src, dst))

    def run(self) -> None:
        if not self.views:
            return
        if not self.views[0][0].is_cuda:
            for s, d in self.views:
                d.copy_(s)
            return
        from . import _lib

        dev = self.views[0][0].device
        rows = torch.empty((len(self.views), 7), dtype=torch.int64)  # ropeslr_row_segment: 56 bytes
        row0 = 0
        for i, (s, d) in enumerate(self.views):
            es = s.element_size()
            if s.stride(1) != 1 or d.stride(1) != 1 or s.dtype != d.dtype:
                raise ValueError("segments need unit column stride and one dtype")
            row_bytes = s.shape[1] * es
            if row_bytes % 16 or (s.stride(0) * es) % 16 or (d.stride(0) * es) % 16 or s.data_ptr() % 16 \
                    or d.data_ptr() % 16:
                raise ValueError("segments need 16-byte aligned rows")
            rows[i, 0] = s.data_ptr()
            rows[i, 1] = d.data_ptr()
            rows[i, 2] = s.stride(0) * es
            rows[i, 3] = d.stride(0) * es
            rows[i, 4] = s.shape[0]
            rows[i, 5] = row0
            rows[i, 6] = row_bytes  # int32 row_bytes, int32 pad (little endian)
            row0 += s.shape[0]
        table = rows.pin_memory().to(dev, non_blocking=True)
        stream = torch.cuda.current_stream(dev)
        _lib.call("ropeslr_copy_rows", ctypes.c_void_p(table.data_ptr()), len(self.views), row0, stream.cuda_stream)
        table.record_stream(stream)


# ---------------------------------------------------------------- the plan
class Plan:
    """Who computes what: per rank its work items, heads and token range."""

    def __init__(self, H: int, L: int, block: int, world: int):
        self.H, self.L, self.block, self.world = H, L, block, world
        self.nb = -(-L // block)
        self.items = work_items(H, self.nb, world)
        self.heads = [heads_of(it) for it in self.items]
        self.tokens = [seq_slice(L, world, r) for r in range(world)]

    def item_rows(self, item: Item, rank: int) -> Tuple[int, int]:
        """Rows of `rank`'s tokens inside the item's query blocks (absolute)."""
        _, qb0, qb1 = item
        a, b = self.tokens[rank]
        return max(qb0 * self.block, a), min(min(qb1 * self.block, self.L), b)


def seq_to_head(plan: Plan, ts: Sequence[torch.Tensor], rank: int, group, async_op: bool = False):
    """Q/K/V/X shards [B, L_r, H, d] (X viewed per head) -> for each of this
    rank's heads the full sequence: returns (out [nt, B, H_me, L, d], finish)
    where finish() waits for the exchange and unpacks."""
    nt = len(ts)
    B, Lr, H, d = ts[0].shape
    dt, dev = ts[0].dtype, ts[0].device
    world = plan.world
    send_rows = [len(plan.heads[s]) * nt * B * Lr for s in range(world)]
    send = torch.empty((sum(send_rows), d), dtype=dt, device=dev)
    seg = Segments()
    off = 0
    for s in range(world):
        for h in plan.heads[s]:
            for z in range(nt):
                for b in range(B):
                    seg.add(ts[z][b, :, h, :], send[off:off + Lr])
                    off += Lr
    seg.run()
    me = plan.heads[rank]
    recv_rows = [len(me) * nt * B * (plan.tokens[r][1] - plan.tokens[r][0]) for r in range(world)]
    recv = torch.empty((sum(recv_rows), d), dtype=dt, device=dev)
    work = _all_to_all(recv, send, recv_rows, send_rows, group,
                       async_op=async_op)
    out = torch.empty((nt, B, len(me), plan.L, d), dtype=dt, device=dev)

    def finish():
        if work is not None:
            work.wait()
        seg2 = Segments()
        o = 0
        for r in range(world):
            a, b_ = plan.tokens[r]
            for j in range(len(me)):
                for z in range(nt):
                    for b in range(B):
                        seg2.add(recv[o:o + b_ - a], out[z, b, j, a:b_])
                        o += b_ - a
        seg2.run()
        return out

    return out, finish


def head_to_seq(plan: Plan, outs: Sequence[Tuple[Item, torch.Tensor]], rank: int, B: int, d: int, dtype, device,
                group) -> torch.Tensor:
    """The rows each work item produced ([B, L, d] per item, full-length
    layout) -> this rank's tokens of every head, [B, L_r, H * d].  Send
    layout, peer-major: per item in this rank's order, per batch, its rows
    inside the peer's token range; the receiver derives the same layout from
    the plan."""
    world = plan.world
    seg, send_rows = Segments(), []
    for r in range(world):
        n = 0
        for item, _ in outs:
            a, b_ = plan.item_rows(item, r)
            n += B * max(0, b_ - a)
        send_rows.append(n)
    send = torch.empty((sum(send_rows), d), dtype=dtype, device=device)
    off = 0
    for r in range(world):
        for item, o in outs:
            a, b_ = plan.item_rows(item, r)
            if b_ > a:
                for b in range(B):
                    seg.add(o[b, a:b_], send[off:off + b_ - a])
                    off += b_ - a
    seg.run()
    r0, r1 = plan.tokens[rank]
    Lr = r1 - r0
    recv_rows = []
    for s in range(world):
        n = 0
        for item in plan.items[s]:
            a, b_ = plan.item_rows(item, rank)
            n += B * max(0, b_ - a)
        recv_rows.append(n)
    recv = torch.empty((sum(recv_rows), d), dtype=dtype, device=device)
    _all_to_all(recv, send, recv_rows, send_rows, group)
    res = torch.empty((B, Lr, plan.H, d), dtype=dtype, device=device)
    seg2, o = Segments(), 0
    for s in range(world):
        for item in plan.items[s]:
            a, b_ = plan.item_rows(item, rank)
            if b_ > a:
                for b in range(B):
                    seg2.add(recv[o:o + b_ - a], res[b, a - r0:b_ - r0, item[0], :])
                    o += b_ - a
    seg2.run()
    return res.view(B, Lr, plan.H * d)


def exchange_gate(plan: Plan, g_local: torch.Tensor, rank: int, group) -> torch.Tensor:
    """Every rank's own-token gate logits [B, L_r] -> the full [B, L]."""
    world = plan.world
    B, Lr = g_local.shape
    if world == 1:
        return g_local.contiguous()
    send = g_local.contiguous().view(-1).repeat(world)
    out_splits = [B * (b - a) for a, b in plan.tokens]
    recv = torch.empty(sum(out_splits), dtype=g_local.dtype, device=g_local.device)
    _all_to_all(recv, send, out_splits, [B * Lr] * world, group)
    full = torch.empty((B, plan.L), dtype=g_local.dtype, device=g_local.device)
    off = 0
    for (a, b), n in zip(plan.tokens, out_splits):
        full[:, a:b] = recv[off:off + n].view(B, b - a)
        off += n
    return full


OpFn = Callable[..., torch.Tensor]
GateFn = Callable[..., torch.Tensor]


def own_gate_logits(x: torch.Tensor, grid, params, settings, pe, token_offset: int) -> torch.Tensor:
    """x_hat . w_g over ALL columns for a sequence shard's own tokens (no
    bias): ropeslr_gate_logits with the shard's token offset."""
    from . import _lib
    from .mechanism import _dtype_code, _stream, _token_args, ctypes_ref

    B, Lr, D = x.shape
    H, d = params.n_heads, params.d_h
    tok = _token_args(x, grid, params, pe, settings.use_pe, 0, H, d, check_grid=False)
    tok.token_offset = int(token_offset)
    shp = _lib.Shape(B, H, Lr, d, 1, _dtype_code(x))
    g = torch.empty((B, Lr), dtype=torch.float32, device=x.device)
    _lib.call("ropeslr_gate_logits", ctypes_ref(shp), ctypes_ref(tok), g.data_ptr(), _stream(x.device))
    return g


def ulysses_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, x: torch.Tensor, grid, params, settings,
                      pe=None, *, group=None, op: Optional[OpFn] = None, gate_fn: Optional[GateFn] = None,
                      rope=None) -> torch.Tensor:
    """RoPeSLR forward on a sequence-sharded rank.

    q, k, v: [B, L_r, H, d] (this rank's tokens, all heads; post-RoPE unless
    ``rope`` is given); x: [B, L_r, H*d]; params: the full model's
    MechanismParams.  Returns this rank's tokens of the output, [B, L_r, H*d].
    ``op(q, k, v, x, grid, params_slice, settings, pe, head_offset=,
    gate_reduce=, rope=, q_blocks=)`` defaults to mechanism.forward;
    ``gate_fn(x, grid, params, settings, pe, token_offset)`` to
    own_gate_logits."""
    from .mechanism import forward

    world, rank = _world(group)
    B, Lr, H, d = q.shape
    L = grid.size
    block = settings.sparse.block
    if isinstance(block, tuple):
        raise ValueError("the sequence-parallel path takes flat blocks")
    plan = Plan(H, L, int(block), world)
    r0, r1 = plan.tokens[rank]
    if Lr != r1 - r0:
        raise ValueError(f"rank {rank} holds {Lr} tokens, expected {r1 - r0}")
    xv = x.view(B, Lr, H, d)
    full, finish = seq_to_head(plan, [q, k, v, xv], rank, group, async_op=True)
    # the own-token gate logits while the exchange is in flight
    gfn = own_gate_logits if gate_fn is None else gate_fn
    g_full = exchange_gate(plan, gfn(x, grid, params, settings, pe, r0), rank, group)
    full = finish()
    me = plan.heads[rank]
    fn = forward if op is None else op

    def use_full_gate(g):
        g.copy_(g_full)

    # consecutive whole heads run as one call; a head shared with another
    # rank runs alone on its query-block range
    groups: List[List[Item]] = []
    for item in plan.items[rank]:
        whole = item[1] == 0 and item[2] == plan.nb
        if whole and groups and groups[-1][-1][1] == 0 and groups[-1][-1][2] == plan.nb \
                and groups[-1][-1][0] + 1 == item[0]:
            groups[-1].append(item)
        else:
            groups.append([item])
    outs = []
    for grp in groups:
        h0, h1 = grp[0][0], grp[-1][0] + 1
        qb0, qb1 = grp[0][1], grp[0][2]
        j0 = me.index(h0)
        nh = h1 - h0
        qh, kh, vh = (full[z, :, j0:j0 + nh] for z in range(3))
        xcols = full[3, :, j0:j0 + nh].permute(0, 2, 1, 3).reshape(B, L, nh * d)
        o = fn(qh, kh, vh, xcols, grid, params.heads(h0, h1), settings, pe, head_offset=h0,
               gate_reduce=use_full_gate, rope=rope, q_blocks=None if (qb0, qb1) == (0, plan.nb) else (qb0, qb1))
        o = o.view(B, L, nh, d)
        for i, item in enumerate(grp):
            outs.append((item, o[:, :, i]))
    return head_to_seq(plan, outs, rank, B, d, q.dtype, q.device, group)
