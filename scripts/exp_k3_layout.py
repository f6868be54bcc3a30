"""Experiment: K3 time vs X layout (24 heads of a [L, 3072] X, vs one head
over a [24 L, 128] X: same bytes, contiguous rows)."""
import sys, os
sys.path[:0] = ['.', 'tests', 'oracle']
import torch, math
import paper_2605_20659_b200 as P

def run(Lgrid, H, label):
    grid = P.GridShape(*Lgrid)
    L = grid.size
    d, r = 128, 64
    D = H * d
    x = torch.randn((1, L, D), device='cuda').to(torch.bfloat16)
    pe = P.PETables(*(torch.randn((n, D), device='cuda') * 0.02 for n in Lgrid))
    params = P.MechanismParams(w_a=torch.randn((H, d, r), device='cuda') / 11, w_b=torch.randn((H, r, d), device='cuda') / 11,
                               alpha=torch.full((D,), 0.1, device='cuda'), w_g=torch.randn((D,), device='cuda') * 0.05,
                               b_g=-2.0, rms_sparse=torch.ones(d, device='cuda'), rms_lowrank=torch.ones(d, device='cuda'))
    st = P.ForwardSettings(P.SparseSettings(128, topk=1))
    for _ in range(3):
        P.compensator_branch(x, grid, params, st, pe)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 20
    for _ in range(n):
        P.compensator_branch(x, grid, params, st, pe)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    gb = 2 * L * D * 2 / 1e9
    # plain strided copy of the same bytes for reference
    y = torch.empty_like(x)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n):
        y.copy_(x)
    e1.record(); torch.cuda.synchronize()
    cms = e0.elapsed_time(e1) / n
    print(f"{label}: K3 step {ms:.3f} ms ({gb/ms:.2f} TB/s incl. fold+gate), torch copy {cms:.3f} ms ({gb/cms:.2f} TB/s)")

run((33, 45, 80), 24, "cfg3 24 heads")
run((33 * 24, 45, 80), 1, "1 head, 24x tokens")
run((33, 45, 80), 12, "12 heads")
