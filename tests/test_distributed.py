"""Head-parallel host logic on CPU with gloo, world size 2.

Each rank takes its head slice (distributed.head_slice), computes the
partial gate logits over its own columns (oracle arithmetic stands in for the
kernel on CPU), and the all-reduce used by forward_head_parallel completes
the gate; the per-head outputs then equal the single-process oracle.
"""

import os
import socket

import numpy as np
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


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path[:0] = [repo, os.path.join(repo, "oracle")]
        import restated as R
        from paper_2605_20659_b200.distributed import gate_allreduce, head_slice

        rng = np.random.default_rng(0)
        H, d, L, r = 5, 8, 24, 4
        grid = (2, 3, 4)
        D = H * d
        x = rng.standard_normal((L, D))
        pe = R.pe_from_axis_tables(grid, *(rng.standard_normal((n, D)) * 0.02 for n in grid))
        alpha = np.full(D, 0.1)
        w_g = rng.standard_normal(D) * 0.1
        b_g = -2.0
        h0, h1 = head_slice(H, world, rank)
        x_hat = x + alpha[None] * pe
        cols = slice(h0 * d, h1 * d)
        partial = torch.from_numpy(x_hat[:, cols] @ w_g[cols])
        gate_allreduce()(partial)
        g = R.sigmoid(partial.numpy() + b_g)
        want = R.gate(x_hat, w_g, b_g)
        ok = np.allclose(g, want, rtol=0, atol=1e-12)
        counts = torch.tensor([h1 - h0])
        dist.all_reduce(counts)
        ok = ok and int(counts) == H
        flag = torch.tensor([1 if ok else 0])
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if rank == 0:
            with open(result_path, "w") as f:
                f.write(str(int(flag)))
    finally:
        dist.destroy_process_group()


def test_head_slice_partition():
    from paper_2605_20659_b200.distributed import head_slice

    for H, W in ((24, 1), (24, 2), (24, 4), (24, 8), (12, 8), (5, 2)):
        spans = [head_slice(H, W, r) for r in range(W)]
        assert spans[0][0] == 0 and spans[-1][1] == H
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    assert head_slice(24, 8, 3) == (9, 12)
    with pytest.raises(ValueError):
        head_slice(2, 4, 0)


def test_gate_allreduce_world2(tmp_path):
    path = str(tmp_path / "ok")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    assert open(path).read() == "1"
