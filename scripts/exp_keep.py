"""Keep-mode (cumulative-mass) selection at a BASELINE shape: time and
selected-block statistics, vs top-k at the same average k."""
import os, sys
sys.path[:0] = ['.', 'tests', 'oracle']
import torch
import paper_2605_20659_b200 as P
import gpu_helpers as G
grid_s = (21, 30, 52); H = int(os.environ.get("EXP_HEADS", "12"))
q, k, v, x, params, pe, grid = G.make_full_inputs(grid_s, H, 128, (44, 42, 42), 64, seed=0)
L = grid.size
def run(st, label):
    for _ in range(2):
        P.forward(q, k, v, x, grid, params, st, pe)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        P.forward(q, k, v, x, grid, params, st, pe)
    e1.record(); torch.cuda.synchronize()
    tr = P.forward(q, k, v, x, grid, params, st, pe, trace=True)
    cnt = tr.selected.sum(-1).float()
    att = int(tr.attended.sum())
    ms = e0.elapsed_time(e1) / 3
    print(f"{label:22s} {ms:8.3f} ms  blocks/row mean {cnt.mean():.1f} min {cnt.min():.0f} max {cnt.max():.0f}  "
          f"{4 * 128 * att / ms / 1e9:.0f} TFLOP/s (sparse part)", flush=True)
for keep in (0.3, 0.6, 0.9):
    run(P.ForwardSettings(P.SparseSettings(64, keep=keep)), f"keep {keep}")
run(P.ForwardSettings(P.SparseSettings.for_sparsity(64, L, 0.9)), "top-51 (90%)")
# skewed rows (per query block scale of Q, as on real data): the longest-first
# unit schedule against the plain persistent stride (ROPESLR_SCHEDULE=0)
from test_gpu_parity import _skew_blocks
q, k = _skew_blocks(q, k, 64, spread=float(os.environ.get("EXP_SPREAD", "2.0")))
for keep in (0.5, 0.8):
    for sched in (1, 0):
        with P._lib.option("schedule", sched):
            run(P.ForwardSettings(P.SparseSettings(64, keep=keep)), f"skew keep {keep} sched {sched}")
