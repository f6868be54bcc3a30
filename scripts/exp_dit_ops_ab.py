"""Time the DiT row kernels (ln_modulate, ln_affine, rms_heads, gated_add) on
a [32760, 1536] bf16 row set with CUDA-graph replay (ROPESLR_LIBRARY picks
the build)."""
import os, sys
sys.path[:0] = ['.']
import torch
import bench as Bm
import paper_2605_20659_b200.dit as dit
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
L, D, H = 32760, 1536, 12
x = torch.randn((1, L, D), generator=g, device=dev).to(torch.bfloat16)
y = torch.randn((1, L, D), generator=g, device=dev).to(torch.bfloat16)
sh = torch.randn((1, 1, D), generator=g, device=dev) * 0.1
sc = torch.randn((1, 1, D), generator=g, device=dev) * 0.1
w = torch.ones(D, device=dev, dtype=torch.bfloat16)
st = torch.cuda.current_stream(dev)
tag = os.environ.get("ROPESLR_LIBRARY", "default")[-12:]
for name, fn in (("ln_modulate", lambda: dit.ln_modulate(x, sh, sc, 1e-6)),
                 ("rms_heads", lambda: dit.rms_heads(x, w, 1e-6, H)),
                 ("gated_add", lambda: dit.gated_add(x, y, sc))):
    ms = Bm.graph_ms(fn, 50, dev, st)
    print(tag, name, f"{ms * 1e3:.1f} us", f"{(2 if name != 'gated_add' else 3) * x.numel() * 2 / (ms * 1e-3) / 1e9:.0f} GB/s")
