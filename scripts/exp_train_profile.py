"""Kernel-time breakdown of one Stage-I training step at the config-1 shape."""
import sys
sys.path[:0] = ['.']
import torch
import bench as Bm
import paper_2605_20659_b200 as P
from paper_2605_20659_b200 import training as T
dev = torch.device("cuda", 0)
cfg = Bm.CONFIGS["cfg1"]
q, k, v, x, params, pe, grid = Bm.make_inputs(cfg, 0, cfg["H"], dev)
settings = P.ForwardSettings(P.SparseSettings.for_sparsity(cfg["block"], grid.size, cfg["sparsity"]))
target = torch.randn(x.shape, device=dev).to(x.dtype)
prepared = T.prepare([T.Stage1Sample(q=q, k=k, v=v, x=x, target=target)], grid, params, settings, pe)
pe_dense = T.pe_head_major(pe, grid, params.n_heads, params.d_h)
for _ in range(2):
    T.loss_and_grads(prepared, params, settings, pe_dense)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    T.loss_and_grads(prepared, params, settings, pe_dense)
    torch.cuda.synchronize()
rows = sorted(((e.key, e.device_time_total / 1e3, e.count) for e in prof.key_averages() if e.device_time_total > 0),
              key=lambda r: -r[1])
print(f"total {sum(r[1] for r in rows):.2f} ms")
for key, ms, n in rows[:int(sys.argv[1]) if len(sys.argv) > 1 else 25]:
    print(f"{ms:7.3f} ms {n:4d}x {key[:100]}")
