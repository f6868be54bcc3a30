"""Stage-I training step at the config-1 shape under torch.profiler: kernel
durations (real, not serialised like ncu), GPU busy time against the step
time, and the idle gaps between kernels."""
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
lr = 1e-3


if len(sys.argv) > 1 and sys.argv[1] == "eager":
    def step():
        loss, grads = T.loss_and_grads(prepared, params, settings, pe_dense)
        with torch.no_grad():
            for name in T.PARAM_NAMES:
                getattr(params, name).sub_(lr * grads[name].to(getattr(params, name).dtype))
        params.b_g = float(params.b_g) - lr * grads["b_g"]
        return loss
else:
    runner = T.Stage1Step(prepared, params, settings, pe_dense, lr)

    def step():
        return runner.step()


for _ in range(3):
    step()
torch.cuda.synchronize()
N = 3
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for _ in range(N):
        step()
    torch.cuda.synchronize()
kern = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0]
kern.sort(key=lambda e: e.time_range.start)
t0, t1 = kern[0].time_range.start, kern[-1].time_range.end
busy = 0
end = t0
for e in kern:
    s, t = e.time_range.start, e.time_range.end
    if t > end:
        busy += t - max(s, end)
        end = t
print(f"{N} steps: span {(t1 - t0) / 1e3:.3f} ms, GPU busy {busy / 1e3:.3f} ms, kernels {len(kern)}")
agg = {}
for e in kern:
    k = e.name[:70]
    a = agg.setdefault(k, [0.0, 0])
    a[0] += (e.time_range.end - e.time_range.start) / 1e3
    a[1] += 1
for k, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{ms / N:8.3f} ms/step {n // N:3d}x {k}")
# the gaps
gaps = []
for a, b in zip(kern, kern[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 5:
        gaps.append((g, a.name[:40], b.name[:40]))
gaps.sort(reverse=True)
print("largest gaps (us):")
for g, a, b in gaps[:12]:
    print(f"  {g:7.1f}  {a} -> {b}")
