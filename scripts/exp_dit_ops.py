"""Torch ops of one config-4 DiT step by device time, with input shapes."""
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
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU],
                                record_shapes=True) as prof:
        model(latent, t, text)
        torch.cuda.synchronize()
print(prof.key_averages(group_by_input_shape=True).table(sort_by="self_device_time_total", row_limit=40,
                                                          max_name_column_width=40, max_shapes_column_width=90))
