"""K1 experiments at the config-3 shape: time the selection (pool + scores +
top-k) with the DMMA vs CUDA-core block scores, and check both give the
same index lists."""
import os, sys
sys.path[:0] = ['.', 'tests', 'oracle']
import torch
import paper_2605_20659_b200 as P
import gpu_helpers as G
H = int(os.environ.get("EXP_HEADS", "24"))
q, k, v, x, params, pe, grid = G.make_full_inputs((33, 45, 80), H, 128, (16, 56, 56), 64, seed=0)
L = grid.size
sp = P.SparseSettings.for_sparsity(128, L, 0.9)
res = {}


def timed(fn, n=int(os.environ.get("EXP_ITERS", "20"))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for rep in range(int(os.environ.get("EXP_REPS", "2"))):
    for sc in ("dmma-pipe", "fma"):
        with P._lib.option("scores", "f" if sc == "fma" else 0):
            ms = timed(lambda: P.select_blocks(q, k, sp, want_mask=False))
            out = P.select_blocks(q, k, sp, want_mask=False)
        torch.cuda.synchronize()
        print(f"scores={sc:9s} select_blocks {ms:.3f} ms", flush=True)
        res[sc] = out.idx.clone()
ref = res["dmma-pipe"]
print("identical index lists:", all(torch.equal(ref, t) for t in res.values()))
# the stages alone
pooled = torch.empty((2, H, -(-L // 128), 128), dtype=torch.float64, device=q.device)
print(f"scores+select from pooled {timed(lambda: P.select_blocks(q, k, sp, want_mask=False, pooled=P.rope_pool(q, k, grid, P.RopeConfig(16, 56, 56), 128)[2])):.3f} ms (incl. rope_pool)")
