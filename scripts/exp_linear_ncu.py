"""Linear-compensator branch at the config-3 shape, a few calls: for the
ncu capture of the state / apply kernels."""
import math, sys
sys.path[:0] = ['.']
import torch
import bench as Bm
import paper_2605_20659_b200 as P
dev = torch.device("cuda", 0)
cfg = Bm.CONFIGS["cfg3"]
H, d = cfg["H"], cfg["d"]
q, k, v, x, params, pe, grid = Bm.make_inputs(cfg, 0, H, dev)
del q, k, v
L, D = grid.size, H * d
gen = torch.Generator(device=dev).manual_seed(11)
W = [torch.randn((H, D, d), generator=gen, device=dev) / math.sqrt(D) for _ in range(3)]
lin = tuple(torch.einsum("bld,hde->bhle", x, w.to(torch.bfloat16)).contiguous() for w in W)
st = P.ForwardSettings(P.SparseSettings.for_sparsity(cfg["block"], L, cfg["sparsity"]), compensator="linear")
fn = lambda: P.compensator_branch(x, grid, params, st, pe, lin_proj=lin, lin_weights=W)
for _ in range(4):
    fn()
torch.cuda.synchronize()
print("branch ms (graph)", Bm.graph_ms(fn, 20, dev, torch.cuda.current_stream(dev)))
