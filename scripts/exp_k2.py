"""K2 experiments: time the fused attention alone at cfg3 shape (a head
subset), under the ROPESLR_DEBUG_MODE variants (modes 2-4 need the measurement
build: scripts/build_variant.sh measure attn_sm100 csrc/attn_sm100.cu -DROPESLR_K2_MEASURE=1,
then ROPESLR_LIBRARY=paper_2605_20659_b200/_variants/measure.so), plus a clock64 trace."""
import os, sys
sys.path[:0] = ['.', 'tests', 'oracle']
import torch
import paper_2605_20659_b200 as P
import gpu_helpers as G
H = int(os.environ.get("EXP_HEADS", "8"))
q, k, v, x, params, pe, grid = G.make_full_inputs((33, 45, 80), H, 128, (16, 56, 56), 64, seed=0)
L = grid.size
st = P.ForwardSettings(P.SparseSettings.for_sparsity(128, L, 0.9))
print("inputs ready", flush=True)
prep = P.prepare(q, k, v, x, grid, params, st, pe)
torch.cuda.synchronize()
print("prepare done", flush=True)
out = torch.empty((1, L, H, 128), dtype=torch.bfloat16, device='cuda')
torch.cuda.synchronize()
att = int(prep.sel.attended.sum())
def timeit(n=int(os.environ.get('EXP_ITERS', '5'))):
    for i in range(2):
        P.attend(prep, params, st, out=out)
        torch.cuda.synchronize()
        print("warm-up attend", i, "done", flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): P.attend(prep, params, st, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    return ms, 4 * 128 * att / ms / 1e9
for mode in os.environ.get("EXP_MODES", "0 1 2 3").split():
    os.environ["ROPESLR_DEBUG_MODE"] = mode
    ms, tf = timeit()
    print(f"mode {mode}: {ms:.3f} ms  {tf:.1f} TFLOP/s")
os.environ["ROPESLR_DEBUG_MODE"] = "0"
os.environ["ROPESLR_K2_TRACE"] = "gpurun_out/k2_trace.txt"
P.attend(prep, params, st, out=out); torch.cuda.synchronize()
del os.environ["ROPESLR_K2_TRACE"]
rows = [l.split() for l in open("gpurun_out/k2_trace.txt")]
import statistics
for w in (0, 1):
    r = [list(map(int, x[2:])) for x in rows if int(x[0]) == w]
    r = [x for x in r if min(x) >= 0]
    sm = [x[1] - x[0] for x in r[4:]]
    per = [r[i + 1][0] - r[i][0] for i in range(4, len(r) - 1)]
    print(f"WG{w}: softmax {statistics.median(sm)} cyc, S->S period {statistics.median(per)} cyc per tile")
