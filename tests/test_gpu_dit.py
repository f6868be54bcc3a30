"""Config-4 caller: a reduced Wan-style DiT with RoPeSLR self-attention runs
end to end on the device, deterministically, and the sequence-parallel
wrapper (ulysses_attention) at world size 1 equals the direct op call."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _small_cfg():
    from paper_2605_20659_b200.dit import WanConfig

    return WanConfig(dim=256, heads=2, ffn=512, blocks=2, text_len=16, text_dim=64, rank=16, block=64,
                     sparsity=0.5, rope_split=(44, 42, 42))


def test_small_dit_forward_deterministic():
    from paper_2605_20659_b200.dit import make_model

    cfg = _small_cfg()
    model = make_model(cfg)
    g = torch.Generator(device="cuda").manual_seed(0)
    latent = torch.randn((1, 16, 3, 8, 16), generator=g, device="cuda").to(torch.bfloat16)
    text = torch.randn((1, cfg.text_len, cfg.text_dim), generator=g, device="cuda").to(torch.bfloat16)
    t = torch.tensor([500.0], device="cuda")
    with torch.no_grad():
        y1 = model(latent, t, text)
        y2 = model(latent, t, text)
    torch.cuda.synchronize()
    assert y1.shape == (1, 3 * 4 * 8, 64)
    assert torch.isfinite(y1.float()).all()
    assert torch.equal(y1, y2)


def test_layer_tables_built_once():
    """Each layer's parameter-only tables are built on the first step and
    reused after (dit.DiTBlock.ropeslr_params keeps the float32 copies);
    an in-place parameter update rebuilds them."""
    import paper_2605_20659_b200.mechanism as M
    from paper_2605_20659_b200.dit import make_model

    cfg = _small_cfg()
    model = make_model(cfg)
    g = torch.Generator(device="cuda").manual_seed(5)
    latent = torch.randn((1, 16, 3, 8, 16), generator=g, device="cuda").to(torch.bfloat16)
    text = torch.randn((1, cfg.text_len, cfg.text_dim), generator=g, device="cuda").to(torch.bfloat16)
    t = torch.tensor([500.0], device="cuda")
    M._TABLES.clear()
    with torch.no_grad():
        y1 = model(latent, t, text)
        keys = list(M._TABLES.keys())
        y2 = model(latent, t, text)
        assert list(M._TABLES.keys()) == keys and len(keys) == cfg.blocks
        assert torch.equal(y1, y2)
        model.blocks[0].w_a.mul_(1.5)
        y3 = model(latent, t, text)
    assert len(M._TABLES) == cfg.blocks + 1
    assert not torch.equal(y1, y3)


def test_ulysses_world1_equals_direct_forward():
    import gpu_helpers as G
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200.ulysses import ulysses_attention

    q, k, v, x, params, pe, grid = G.make_full_inputs((2, 8, 16), 2, 128, (16, 56, 56), 64, seed=1)
    st = P.ForwardSettings(P.SparseSettings.for_sparsity(64, grid.size, 0.75))
    want = P.forward(q, k, v, x, grid, params, st, pe)
    got = ulysses_attention(q.permute(0, 2, 1, 3).contiguous(), k.permute(0, 2, 1, 3).contiguous(),
                            v.permute(0, 2, 1, 3).contiguous(), x, grid, params, st, pe)
    torch.cuda.synchronize()
    # the wrapper takes the gate from the own-token gate kernel (all columns),
    # the direct call from the compensator's fused gate columns: same math,
    # different rounding, so the bf16 bar rather than bit equality
    G.assert_close(got.float().cpu().numpy(), want.float().cpu().numpy(), "bf16", "ulysses world 1")


def test_own_gate_logits_token_offset():
    """ropeslr_gate_logits on a sequence shard (token offset: the PE rows of
    the shard's grid positions) equals the full-sequence gate's rows."""
    import gpu_helpers as G
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200.ulysses import own_gate_logits

    q, k, v, x, params, pe, grid = G.make_full_inputs((3, 8, 16), 3, 128, (44, 42, 42), 64, seed=2)
    st = P.ForwardSettings(P.SparseSettings(64, topk=1))
    full = own_gate_logits(x, grid, params, st, pe, 0)
    for a, b in ((0, 100), (100, 384), (77, 78)):
        part = own_gate_logits(x[:, a:b].contiguous(), grid, params, st, pe, a)
        assert torch.equal(part, full[:, a:b])
    with pytest.raises(ValueError):
        own_gate_logits(x[:, :10].contiguous(), grid, params, st, pe, grid.size - 5)


def test_copy_rows_segments():
    """The pack / unpack kernel (ropeslr_copy_rows) equals torch copies,
    segments of different strides and lengths in one launch."""
    from paper_2605_20659_b200.ulysses import Segments

    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn((2, 300, 6, 128), generator=g, device="cuda").to(torch.bfloat16)
    dst = torch.zeros((2000, 128), dtype=torch.bfloat16, device="cuda")
    seg, want, off = Segments(), [], 0
    for b, h, r0, r1 in ((0, 1, 0, 300), (1, 5, 17, 200), (0, 3, 299, 300)):
        seg.add(a[b, r0:r1, h, :], dst[off:off + r1 - r0])
        want.append((a[b, r0:r1, h, :], (off, off + r1 - r0)))
        off += r1 - r0
    seg.run()
    torch.cuda.synchronize()
    for src, (o0, o1) in want:
        assert torch.equal(dst[o0:o1], src)
    assert bool((dst[off:] == 0).all())


def test_fused_block_ops_match_torch(monkeypatch):
    """The fused token-wise ops (csrc/dit_ops.cu: modulated LayerNorm,
    RMSNorm into the head-major layout, gated residual) give the plain
    PyTorch composition's block output within bf16 rounding."""
    import paper_2605_20659_b200.dit as dit

    cfg = _small_cfg()
    model = dit.make_model(cfg)
    g = torch.Generator(device="cuda").manual_seed(3)
    latent = torch.randn((1, 16, 3, 8, 16), generator=g, device="cuda").to(torch.bfloat16)
    text = torch.randn((1, cfg.text_len, cfg.text_dim), generator=g, device="cuda").to(torch.bfloat16)
    t = torch.tensor([250.0], device="cuda")
    outs = {}
    for fused in (True, False):
        monkeypatch.setattr(dit, "FUSED_OPS", fused)
        with torch.no_grad():
            outs[fused] = model(latent, t, text).float()
    torch.cuda.synchronize()
    a, b = outs[True], outs[False]
    scale = b.abs().max().item()
    assert torch.isfinite(a).all()
    assert (a - b).abs().max().item() <= 3e-2 * scale
    assert ((a - b).abs().mean() / b.abs().mean()).item() <= 1e-2


def test_fused_ops_unit():
    """Each fused op against its PyTorch definition on random rows."""
    import torch.nn.functional as F

    import paper_2605_20659_b200.dit as dit

    g = torch.Generator(device="cuda").manual_seed(4)
    L, D, H = 333, 1536, 12
    x = torch.randn((1, L, D), generator=g, device="cuda").to(torch.bfloat16)
    sh = torch.randn((1, 1, D), generator=g, device="cuda") * 0.1
    sc = torch.randn((1, 1, D), generator=g, device="cuda") * 0.1
    want = (F.layer_norm(x.float(), (D,), eps=1e-6) * (1 + sc) + sh).to(torch.bfloat16)
    got = dit.ln_modulate(x, sh, sc, 1e-6)
    assert (got.float() - want.float()).abs().max().item() <= 2e-2
    ln = torch.nn.LayerNorm(D, eps=1e-6, elementwise_affine=True).cuda().to(torch.bfloat16)
    with torch.no_grad():
        ln.weight.copy_(1 + 0.1 * torch.randn(D, generator=g, device="cuda"))
        ln.bias.copy_(0.1 * torch.randn(D, generator=g, device="cuda"))
        want_ln = ln(x)
    got_ln = dit.ln_affine(x, ln)
    assert (got_ln.float() - want_ln.float()).abs().max().item() <= 3e-2
    w = (1 + 0.1 * torch.randn(D, generator=g, device="cuda")).to(torch.bfloat16)
    xf = x.float()
    rms = ((xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-6)).to(torch.bfloat16) * w)
    got_h = dit.rms_heads(x, w, 1e-6, H)
    torch.testing.assert_close(got_h, rms.view(1, L, H, D // H).permute(0, 2, 1, 3), atol=2e-2, rtol=1e-2)
    got_t = dit.rms_heads(x, w, 1e-6, H, head_major=False)
    torch.testing.assert_close(got_t, rms.view(1, L, H, D // H), atol=2e-2, rtol=1e-2)
    assert torch.equal(dit.rms_heads(x, None, 0.0, H), x.view(1, L, H, D // H).permute(0, 2, 1, 3))
    wide = torch.randn((1, L, 3 * D), generator=g, device="cuda").to(torch.bfloat16)  # a fused QKV row set
    for j in range(3):
        part = wide[..., j * D:(j + 1) * D]
        assert torch.equal(dit.rms_heads(part, w, 1e-6, H), dit.rms_heads(part.contiguous(), w, 1e-6, H))
    y = torch.randn((1, L, D), generator=g, device="cuda").to(torch.bfloat16)
    gate = torch.randn((1, 1, D), generator=g, device="cuda")
    want_x = x + (y.float() * gate).to(torch.bfloat16)
    got_x = dit.gated_residual_(x.clone(), y, gate)
    assert torch.equal(got_x, want_x)
    x0 = x.clone()
    assert torch.equal(dit.gated_add(x, y, gate), want_x)
    assert torch.equal(x, x0)
    a = torch.randn((2, H, L, D // H), generator=g, device="cuda").to(torch.bfloat16)
    assert torch.equal(dit.heads_to_tokens(a), a.transpose(1, 2).reshape(2, L, D))
