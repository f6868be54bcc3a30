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
    assert torch.equal(got, want)
