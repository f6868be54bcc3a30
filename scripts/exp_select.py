"""K1 experiments: time the selection (pool + scores + top-k) at the config-3
shape, CUDA-core vs DMMA block scores (ROPESLR_SCORES), and check that both
give the same index lists."""
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
for mode in ("fma", "dmma", "fma", "dmma"):
    P._lib.set_option("scores", mode[0])
    for _ in range(2):
        sel = P.select_blocks(q, k, sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sel = P.select_blocks(q, k, sp)
    e1.record()
    torch.cuda.synchronize()
    print(f"{mode:5s} select_blocks {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
    res[mode] = sel.idx.clone()
print("identical index lists:", torch.equal(res["fma"], res["dmma"]))
