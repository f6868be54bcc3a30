"""Sequence <-> head all-to-all around the op (config 4, ulysses.py) on CPU
with gloo at world sizes 2 and 3: uneven head and token splits, a stand-in
op that needs whole sequences per head and the all-reduced gate, compared
with the same op on the unsharded tensors."""

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


def _standin_op(q, k, v, x, grid, params, settings, pe, *, head_offset=0, gate_reduce=None, rope=None):
    """Depends on the whole sequence of each head (q summed over L) and on
    every head's columns of X (the gate partial, all-reduced)."""
    B, H, L, d = q.shape
    g = x.sum(-1)  # [B, L] partial over this rank's heads
    if gate_reduce is not None:
        gate_reduce(g)
    s = q.sum(dim=2, keepdim=True)
    o = (v * s + k).permute(0, 2, 1, 3)  # [B, L, H, d]
    hid = torch.arange(H, dtype=q.dtype).view(1, 1, H, 1) + head_offset + 1
    o = o + g[:, :, None, None] * hid
    return o.reshape(B, L, H * d)


class _Params:
    def __init__(self, H):
        self.H = H

    def heads(self, a, b):
        return _Params(b - a)


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
                                x[:, a:b].contiguous(), grid, _Params(H), None, op=_standin_op)
        want = _standin_op(q.permute(0, 2, 1, 3), k.permute(0, 2, 1, 3), v.permute(0, 2, 1, 3), x, grid, _Params(H),
                           None, None)[:, a:b]
        ok = torch.tensor([1 if torch.allclose(got, want, rtol=1e-12, atol=1e-12) else 0])
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if rank == 0:
            torch.save(ok, result)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,grid_s", [(2, 3, (2, 3, 5)), (3, 4, (1, 5, 7)), (2, 12, (3, 2, 3))])
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
