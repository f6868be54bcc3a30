"""Overlap of the selected key-block sets of adjacent query blocks (2i, 2i+1)
at block 64: on config-1 inputs (seeded N(0,1) + RoPE) and on the q/k of
the config-4 DiT's first layers (random-init weights, synthetic latent)."""
import sys
sys.path[:0] = ['.']
import torch
import bench as Bm
import paper_2605_20659_b200 as P
import paper_2605_20659_b200.dit as dit
dev = torch.device("cuda", 0)


def overlap(idx, cnt, nb):
    # idx [B, H, nb, kmax], cnt [B, H, nb]
    B, H, _, kmax = idx.shape
    m = torch.zeros((B, H, nb, nb), dtype=torch.bool, device=idx.device)
    live = torch.arange(kmax, device=idx.device) < cnt[..., None]
    m.scatter_(3, torch.where(live, idx, 0).long(), live)
    a, b = m[:, :, 0:nb - 1:2], m[:, :, 1:nb:2]
    inter = (a & b).sum(-1).float()
    union = (a | b).sum(-1).float()
    k = cnt.float().mean()
    return float(inter.mean() / k), float(union.mean() / (2 * k))


cfg = Bm.CONFIGS["cfg1"]
q, k, v, x, params, pe, grid = Bm.make_inputs(cfg, 0, cfg["H"], dev)
sp = P.SparseSettings.for_sparsity(64, grid.size, 0.9)
sel = P.select_blocks(q, k, sp)
nb = -(-grid.size // 64)
print("cfg1 random: shared fraction %.3f, union / 2k %.3f" % overlap(sel.idx, sel.cnt, nb))

# DiT layer q/k: hook the attention inputs of the first blocks
cfgw = dit.WanConfig()
model = dit.make_model(cfgw, device=dev)
gen = torch.Generator(device=dev).manual_seed(0)
latent = torch.randn((1, cfgw.in_channels, 21, 60, 104), generator=gen, device=dev).to(torch.bfloat16)
text = torch.randn((1, cfgw.text_len, cfgw.text_dim), generator=gen, device=dev).to(torch.bfloat16)
t = torch.tensor([500.0], device=dev)
seen = []
orig = dit.forward


def spy(q, k, v, x, grid, params, settings, pe=None, **kw):
    if len(seen) < 6:
        s = P.select_blocks(q, k, settings.sparse)
        nbb = -(-grid.size // settings.sparse.block)
        seen.append(overlap(s.idx, s.cnt, nbb))
    return orig(q, k, v, x, grid, params, settings, pe, **kw)


dit.forward = spy
with torch.no_grad():
    model(latent, t, text)
for i, (sh, un) in enumerate(seen):
    print(f"DiT layer {i}: shared fraction {sh:.3f}, union / 2k {un:.3f}")
