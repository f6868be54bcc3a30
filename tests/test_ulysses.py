"""Sequence <-> head all-to-all around the op (config 4, ulysses.py) on CPU
with gloo at world sizes 2, 3 and 8 (12 heads: 1.5 heads of query blocks
per rank): uneven token splits, heads shared by two ranks (each runs its
query-block range), a stand-in op that needs whole sequences per head and
the full gate, compared with the same op on the unsharded tensors."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


BLOCK = 4


def _standin_op(q, k, v, x, grid, params, settings, pe, *, head_offset=0, gate_reduce=None, rope=None,
                q_blocks=None):
    """Depends on the whole sequence of each head (q summed over L) and on
    every head's columns of X (the gate: the caller's full logits replace
    the partial ones, as ulysses.py does); with q_blocks only those query
    blocks' rows are produced (the others stay NaN)."""
    B, H, L, d = q.shape
    g = x.sum(-1)  # [B, L] partial over this call's heads
    if gate_reduce is not None:
        gate_reduce(g)
    s = q.sum(dim=2, keepdim=True)
    o = (v * s + k).permute(0, 2, 1, 3)  # [B, L, H, d]
    hid = torch.arange(H, dtype=q.dtype).view(1, 1, H, 1) + head_offset + 1
    o = o + g[:, :, None, None] * hid
    if q_blocks is not None:
        keep = torch.zeros(L, dtype=torch.bool)
        keep[q_blocks[0] * BLOCK:q_blocks[1] * BLOCK] = True
        o[:, ~keep] = float("nan")
    return o.reshape(B, L, H * d)


def _standin_gate(x, grid, params, settings, pe, token_offset):
    return x.sum(-1)  # every column of the shard's own tokens


class _Params:
    def __init__(self, H):
        self.H = H

    def heads(self, a, b):
        return _Params(b - a)


class _Settings:
    class sparse:
        block = BLOCK


def _worker(rank, world, port, H, grid_s, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, repo)
        from paper_2605_20659_b200.rope3d import GridShape
        from paper_2605_20659_b200.ulysses import seq_slice, ulysses_attention

        grid = GridShape(*grid_s)
        L, d, B = grid.size, 4, 2
        g = torch.Generator().manual_seed(0)
        q, k, v = (torch.randn((B, L, H, d), generator=g, dtype=torch.float64) for _ in range(3))
        x = torch.randn((B, L, H * d), generator=g, dtype=torch.float64)
        a, b = seq_slice(L, world, rank)
        got = ulysses_attention(q[:, a:b].contiguous(), k[:, a:b].contiguous(), v[:, a:b].contiguous(),
                                x[:, a:b].contiguous(), grid, _Params(H), _Settings, op=_standin_op,
                                gate_fn=_standin_gate)
        want = _standin_op(q.permute(0, 2, 1, 3), k.permute(0, 2, 1, 3), v.permute(0, 2, 1, 3), x, grid, _Params(H),
                           None, None)[:, a:b]
        ok = torch.tensor([1 if torch.allclose(got, want, rtol=1e-12, atol=1e-12) else 0])
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if rank == 0:
            torch.save(ok, result)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,grid_s", [(2, 3, (2, 3, 5)), (3, 4, (1, 5, 7)), (2, 12, (3, 2, 3)),
                                             (8, 12, (2, 4, 5))])
def test_ulysses_all_to_all(tmp_path, world, H, grid_s):
    result = str(tmp_path / "ok.pt")
    mp.spawn(_worker, args=(world, _free_port(), H, grid_s, result), nprocs=world, join=True)
    assert int(torch.load(result)) == 1


def test_seq_slice_partition():
    from paper_2605_20659_b200.ulysses import seq_slice

    for L, W in ((32760, 8), (7, 3), (5, 5)):
        cuts = [seq_slice(L, W, r) for r in range(W)]
        assert cuts[0][0] == 0 and cuts[-1][1] == L
        assert all(cuts[i][1] == cuts[i + 1][0] for i in range(W - 1))
        assert max(b - a for a, b in cuts) - min(b - a for a, b in cuts) <= 1


def test_work_items_balance():
    """(head x query-block range) split: 12 heads of 512 blocks on 8 ranks give
    every rank 768 blocks (1.5 heads) in at most two pieces, every block
    exactly once, and a head on at most two ranks."""
    from paper_2605_20659_b200.ulysses import heads_of, work_items

    for H, nb, W in ((12, 512, 8), (12, 256, 8), (24, 929, 8), (3, 7, 2), (12, 5, 8)):
        items = work_items(H, nb, W)
        sizes = [sum(b - a for _, a, b in it) for it in items]
        assert max(sizes) - min(sizes) <= 1
        cover = {}
        for r, it in enumerate(items):
            for h, a, b in it:
                for qb in range(a, b):
                    assert (h, qb) not in cover
                    cover[(h, qb)] = r
        assert len(cover) == H * nb
        if nb * 1.0 >= H * nb / W:
            assert all(len(heads_of(it)) <= 2 for it in items)
    assert [len(it) for it in work_items(12, 512, 8)] == [2] * 8
