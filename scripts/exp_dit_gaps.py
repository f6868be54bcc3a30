"""GPU idle gaps inside one config-4 DiT step: kernel timeline from the
torch profiler, gaps > 10 us listed with the kernels on either side and
the CPU ops running at the time."""
import json
import sys
sys.path[:0] = ['.']
import torch
from paper_2605_20659_b200.dit import WanConfig, make_model
dev = torch.device("cuda", 0)
cfg = WanConfig()
model = make_model(cfg, device=dev)
gen = torch.Generator(device=dev).manual_seed(0)
latent = torch.randn((1, cfg.in_channels, 21, 60, 104), generator=gen, device=dev).to(torch.bfloat16)
text = torch.randn((1, cfg.text_len, cfg.text_dim), generator=gen, device=dev).to(torch.bfloat16)
t = torch.tensor([500.0], device=dev)
with torch.no_grad():
    for _ in range(2):
        model(latent, t, text)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
        model(latent, t, text)
        torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/dit_trace.json")
tr = json.load(open("gpurun_out/dit_trace.json"))
ev = tr["traceEvents"] if isinstance(tr, dict) else tr
gpu = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("cpu_op", "cuda_runtime", "cuda_driver")]
t0, t1 = gpu[0]["ts"], gpu[-1]["ts"] + gpu[-1]["dur"]
busy = sum(e["dur"] for e in gpu)
print(f"span {(t1 - t0) / 1e3:.2f} ms, kernels {busy / 1e3:.2f} ms, {len(gpu)} launches")
gaps = []
for a, b in zip(gpu, gpu[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    if g > 10:
        gaps.append((g, a, b))
tot = sum(g for g, _, _ in gaps)
print(f"gaps > 10 us: {len(gaps)}, {tot / 1e3:.2f} ms")
from collections import Counter
c = Counter()
for g, a, b in gaps:
    c[(a["name"][:60], b["name"][:60])] += g
for (an, bn), g in c.most_common(15):
    print(f"{g / 1e3:7.2f} ms  {an}  ->  {bn}")
# the cpu ops overlapping the largest gaps
for g, a, b in sorted(gaps, key=lambda x: -x[0])[:6]:
    s, e = a["ts"] + a["dur"], b["ts"]
    ops = [x["name"] for x in cpu if x["ts"] < e and x["ts"] + x["dur"] > s and x["dur"] < 5000][:12]
    print(f"gap {g:.0f} us after {a['name'][:50]}: {ops}")
