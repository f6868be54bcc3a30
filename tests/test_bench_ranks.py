"""bench.py's N > 1 rank logic on CPU (gloo, world size 2).

Each rank takes its head slice, runs a stand-in for the op on its heads (the
oracle's selection, whose attended-pair count is what the bench's FLOP
total is built from), and reports a per-rank time; ``bench.reduce_over_ranks``
must give the max of the times and the sum of the attended pairs, equal to
the single-process totals.  The launcher side (``--gpus N`` without
torchrun re-launching itself) is checked for its argument handling."""

import os
import socket
import subprocess
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _attended_of_heads(h0, h1):
    import restated as R

    rng = np.random.default_rng(3)
    L, d, block, topk = 200, 16, 32, 2
    members = R.flat_block_members(L, block)
    total = 0
    for h in range(6):
        q, k = rng.standard_normal((2, L, d))
        if h0 <= h < h1:
            sel, _ = R.select_blocks(R.block_scores(q, k, members), topk=topk)
            total += R.attended_pairs(members, sel)
    return total


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path[:0] = [REPO, os.path.join(REPO, "oracle")]
        import bench
        from paper_2605_20659_b200.distributed import head_slice

        h0, h1 = head_slice(6, world, rank)
        att = _attended_of_heads(h0, h1)
        times = [10.0 + rank, 5.0 - rank, 7.0 * (rank + 1)]
        (ms, k2, e2e), att_total = bench.reduce_over_ranks(times, att, "cpu", world)
        ok = (ms, k2, e2e) == (10.0 + world - 1, 5.0, 7.0 * world) and att_total == _attended_of_heads(0, 6)
        ok = ok and bench.heads_per_rank(6, world) == [3, 3] and bench.heads_per_rank(24, 8) == [3] * 8
        if rank == 0:
            with open(result_path, "w") as f:
                f.write("1" if ok else "0")
    finally:
        dist.destroy_process_group()


def test_reduce_over_ranks_world2(tmp_path):
    path = str(tmp_path / "ok")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    assert open(path).read() == "1"


def test_bench_rejects_mismatched_world():
    """A launcher world size that disagrees with --gpus exits non-zero instead
    of silently running every head on one rank."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--impl", "reference"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in (r.stderr + r.stdout)
