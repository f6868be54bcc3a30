"""A/B of the K3 (low-rank) kernel between two builds at the config-3 shape:
python scripts/exp_k3ab.py (ROPESLR_LIBRARY selects the build)."""
import os, sys
sys.path[:0] = ['.']
import torch
import bench as Bm
import paper_2605_20659_b200 as P
dev = torch.device("cuda", 0)
cfg = Bm.CONFIGS[os.environ.get("CFG", "cfg3")]
q, k, v, x, params, pe, grid = Bm.make_inputs(cfg, 0, cfg["H"], dev)
settings = P.ForwardSettings(P.SparseSettings.for_sparsity(cfg["block"], grid.size, cfg["sparsity"]))
fn = lambda: P.compensator_branch(x, grid, params, settings, pe)
for _ in range(5):
    fn()
torch.cuda.synchronize()
for rep in range(3):
    ms = Bm.graph_ms(fn, 50, dev, torch.cuda.current_stream(dev))
    print(os.environ.get("ROPESLR_LIBRARY", "default")[-14:], cfg["name"][:20], f"{ms:.4f} ms (graph replay)")
