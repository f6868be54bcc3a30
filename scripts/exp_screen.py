"""K1 at the config-3 shape: select_blocks with the screening path against
the float64-everywhere path (option screen=0); same index lists, and the
time of each."""
import os
import sys

sys.path[:0] = ['.', 'tests', 'oracle']
import torch

import paper_2605_20659_b200 as P
import gpu_helpers as G

H = int(os.environ.get("EXP_HEADS", "24"))
q, k, v, x, params, pe, grid = G.make_full_inputs((33, 45, 80), H, 128, (16, 56, 56), 64, seed=0)
sp = P.SparseSettings.for_sparsity(128, grid.size, 0.9)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


res = {}
for rep in range(2):
    for scr in (1, 0):
        with P._lib.option("screen", scr):
            ms = timed(lambda: P.select_blocks(q, k, sp, want_mask=False))
            res[scr] = P.select_blocks(q, k, sp, want_mask=False)
        torch.cuda.synchronize()
        print(f"screen={scr} select_blocks {ms:.3f} ms", flush=True)
print("identical:", all(torch.equal(getattr(res[0], f), getattr(res[1], f)) for f in ("idx", "cnt", "attended")))

# band sizes and bisection steps per row (the screening path's diagnostics)
import ctypes
from paper_2605_20659_b200 import _lib, mechanism as M

sys.path.insert(0, "tests")
import test_gpu_screen as T

for name, (qq, kk) in {"cfg3": (q, k)}.items():
    pooled, approx, full = T._raw_screen(qq, kk, sp.topk, 128)
    diag = T._raw_screen.diag
    band, steps = (diag & 0xffff), (diag >> 16)
    print(name, "full rows", full, "band mean", band.float().mean().item(), "max", band.max().item(),
          "hist", torch.bincount(band.clamp(max=64).long(), minlength=65)[:20].tolist(),
          "steps mean", steps.float().mean().item(), "max", steps.max().item())
    qn = pooled[0].norm(dim=-1)
    print("q norm mean", qn.mean().item(), "approx std", approx.float().std().item())

# skewed (structured) block scores, as real attention has (test_gpu_parity._skew_blocks)
from test_gpu_parity import _skew_blocks
for strength in (4.0, 8.0):
    qs, ks = _skew_blocks(q, k, 128, strength=strength)
    for scr in (1, 0):
        with P._lib.option("screen", scr):
            ms = timed(lambda: P.select_blocks(qs, ks, sp, want_mask=False))
            res[scr] = P.select_blocks(qs, ks, sp, want_mask=False)
        torch.cuda.synchronize()
        print(f"skew {strength}: screen={scr} select_blocks {ms:.3f} ms", flush=True)
    print("identical:", all(torch.equal(getattr(res[0], f), getattr(res[1], f)) for f in ("idx", "cnt", "attended")))
    pooled, approx, full = T._raw_screen(qs, ks, sp.topk, 128)
    diag = T._raw_screen.diag
    band, steps = (diag & 0xffff), (diag >> 16)
    ok = diag >= 0
    print("skew", strength, "deferred rows", full, "band mean", band[ok].float().mean().item(), "max", band[ok].max().item(),
          "steps mean", steps[ok].float().mean().item())
