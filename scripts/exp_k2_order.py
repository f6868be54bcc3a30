"""K2 at config 3 with a given build (ROPESLR_LIBRARY): 30 back-to-back
launches (sustained, power-capped) and the output checksum, for unit-order
experiments."""
import os, sys
sys.path[:0] = ['.']
import torch
import bench as Bm
import paper_2605_20659_b200 as P
dev = torch.device("cuda", 0)
cfg = Bm.CONFIGS["cfg3"]
q, k, v, x, params, pe, grid = Bm.make_inputs(cfg, 0, cfg["H"], dev)
st = P.ForwardSettings(P.SparseSettings.for_sparsity(cfg["block"], grid.size, cfg["sparsity"]))
prep = P.prepare(q, k, v, x, grid, params, st, pe)
ws = P.attend_workspace(prep)
out = torch.empty((1, grid.size, cfg["H"], cfg["d"]), dtype=torch.bfloat16, device=dev)
n = int(os.environ.get("N", "30"))
for _ in range(3):
    P.attend(prep, params, st, out=out, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    P.attend(prep, params, st, out=out, workspace=ws)
e1.record()
torch.cuda.synchronize()
print(os.environ.get("ROPESLR_LIBRARY", "default")[-10:], f"{e0.elapsed_time(e1) / n:.3f} ms/launch",
      "checksum", float(out.float().abs().sum()), flush=True)
if os.environ.get("DUMP"):
    torch.save(out.cpu(), os.environ["DUMP"])
