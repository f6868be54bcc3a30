"""K1 in keep mode at the config-3 shape (float64 scores + sort + mass
scan): kernel times for the ncu launch list / capture."""
import sys
sys.path[:0] = ['.']
import torch
import bench as Bm
import paper_2605_20659_b200 as P
dev = torch.device("cuda", 0)
cfg = Bm.CONFIGS["cfg3"]
q, k, v, x, params, pe, grid = Bm.make_inputs(cfg, 0, cfg["H"], dev)
sp = P.SparseSettings(cfg["block"], keep=float(sys.argv[1]) if len(sys.argv) > 1 else 0.9)
for _ in range(3):
    P.select_blocks(q, k, sp, grid, want_mask=False)
torch.cuda.synchronize()
print("k1 keep ms", Bm.graph_ms(lambda: P.select_blocks(q, k, sp, grid, want_mask=False), 10, dev,
                                torch.cuda.current_stream(dev)))
