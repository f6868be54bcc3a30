"""Linear compensator (mechanism.py:33-36, 347-362; K3 `linear` mode) at the
config-3 shape: time and HBM rate of ropeslr_linear_branch."""
import sys
sys.path[:0] = ['.', 'tests', 'oracle']
import torch
import paper_2605_20659_b200 as P
import gpu_helpers as G
H = 24
q, k, v, x, params, pe, grid = G.make_full_inputs((33, 45, 80), H, 128, (16, 56, 56), 64, seed=0)
st = P.ForwardSettings(P.SparseSettings.for_sparsity(128, grid.size, 0.9), compensator="linear")
lin = (q.contiguous(), k.contiguous(), v.contiguous())
for _ in range(2):
    P.compensator_branch(x, grid, params, st, pe, lin_proj=lin)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    P.compensator_branch(x, grid, params, st, pe, lin_proj=lin)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
by = (4 + 1) * q.numel() * 2  # q, k, v, x read + y_lr written (bf16)
print(f"linear compensator branch: {ms:.3f} ms, {by / (ms * 1e-3) / 1e9:.0f} GB/s over {by / 1e9:.2f} GB")
