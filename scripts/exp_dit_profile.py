"""Kernel-time breakdown of one config-4 DiT denoising step (torch profiler):
which share is RoPeSLR (our kernels) and which is the caller's GEMMs and
elementwise ops."""
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
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        model(latent, t, text)
        torch.cuda.synchronize()
ev = prof.key_averages()
rows = sorted(((e.key, e.device_time_total / 1e3, e.count) for e in ev if e.device_time_total > 0), key=lambda r: -r[1])
tot = sum(r[1] for r in rows)
print(f"total device time {tot:.1f} ms")
ours = 0.0
for k, ms, n in rows[:30]:
    mine = any(s in k for s in ("sparse_attn", "pool", "block_scores", "select_", "screen_", "lowrank", "gate_sum", "rope_pool", "rope_tables", "schedule_units", "dit_", "copy_rows", "ropeslr"))
    ours += ms if mine else 0.0
    print(f"{ms:8.2f} ms {n:5d}x {'*' if mine else ' '} {k[:90]}")
print(f"ours (top 30) {ours:.1f} ms")
