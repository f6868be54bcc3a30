"""One forward step at config 3 (bench.py's step) under torch.profiler: every
kernel / memset / copy of the step with its real duration, and the gaps."""
import sys
sys.path[:0] = ['.']
import torch
import bench as Bm
import paper_2605_20659_b200 as P
dev = torch.device("cuda", 0)
cfg = Bm.CONFIGS["cfg3"]
q, k, v, x, params, pe, grid = Bm.make_inputs(cfg, 0, cfg["H"], dev)
settings = P.ForwardSettings(P.SparseSettings.for_sparsity(cfg["block"], grid.size, cfg["sparsity"]))
out_buf = torch.empty((1, grid.size, cfg["H"], cfg["d"]), dtype=torch.bfloat16, device=dev)
ws = []


def step():
    prep = P.prepare(q, k, v, x, grid, params, settings, pe)
    if not ws:
        ws.append(P.attend_workspace(prep))
    P.attend(prep, params, settings, out=out_buf, workspace=ws[0])


for _ in range(3):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev = t0
for e in ev:
    s, t = e.time_range.start, e.time_range.end
    print(f"{(s - t0) / 1e3:8.3f} ms  gap {(s - prev):7.1f} us  dur {(t - s):9.1f} us  {e.name[:70]}")
    prev = t
