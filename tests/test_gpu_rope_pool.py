"""Fused 3D RoPE + block pooling pre-pass (SURVEY.md 8f "next" #1).

The rotated Q/K must equal the package's torch rotation (rope3d.rotate_rows,
the restatement of rope3d.py:102-143, float64 then cast) bit for bit; the
block means must equal K1's pooling of those rotated tensors bit for bit;
and a forward from un-rotated Q/K must reproduce the forward from
pre-rotated Q/K exactly (masks, attended counts, output)."""

import math

import numpy as np
import pytest
import torch

import restated as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _pool_torch(t, block):
    """float64 block means of a [B, H, L, d] tensor, [B*H, nb, d]: exact sum
    (bf16 / small f32 sums are exact in float64), then one correctly rounded
    division (NumPy; torch's scalar division multiplies by the reciprocal)."""
    B, H, L, d = t.shape
    nb = -(-L // block)
    x = t.double().reshape(B * H, L, d).cpu().numpy()
    out = np.empty((B * H, nb, d))
    for b in range(nb):
        rows = x[:, b * block:min(L, (b + 1) * block)]
        out[:, b] = rows.sum(1) / rows.shape[1]
    return torch.from_numpy(out).to(t.device)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("grid_s,split,block", [((3, 8, 16), (16, 56, 56), 128), ((2, 5, 9), (44, 42, 42), 64),
                                                ((4, 7, 7), (16, 24, 24), 32),
                                                # TMA-tiled kernel edges: 5-row ragged last blocks, 8-row blocks
                                                ((1, 7, 19), (16, 56, 56), 128), ((1, 7, 19), (16, 56, 56), 8)])
def test_rope_pool_matches_torch_rotation(dtype, grid_s, split, block):
    import paper_2605_20659_b200 as P

    grid = P.GridShape(*grid_s)
    cfg = P.RopeConfig(*split)
    d = cfg.d_h
    g = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn((2, 3, grid.size, d), generator=g, device="cuda").to(dtype)
    k = torch.randn((2, 3, grid.size, d), generator=g, device="cuda").to(dtype)
    qr, kr, pooled = P.rope_pool(q, k, grid, cfg, block)
    want_q = P.rotate_rows(q, grid, cfg).to(dtype)
    want_k = P.rotate_rows(k, grid, cfg).to(dtype)
    torch.cuda.synchronize()
    assert torch.equal(qr, want_q), "rotated Q differs from rope3d.rotate_rows"
    assert torch.equal(kr, want_k), "rotated K differs from rope3d.rotate_rows"
    assert torch.equal(pooled[0], _pool_torch(want_q, block))
    assert torch.equal(pooled[1], _pool_torch(want_k, block))


def test_rope_pool_matches_numpy_oracle_rotation():
    """The oracle's float64 rotation (oracle/restated.py) agrees to rounding."""
    import paper_2605_20659_b200 as P

    grid_s, split = (3, 4, 5), (8, 12, 12)
    grid, cfg = P.GridShape(*grid_s), P.RopeConfig(*split)
    rng = np.random.default_rng(3)
    q = torch.from_numpy(rng.standard_normal((1, 1, grid.size, cfg.d_h))).float().cuda()
    qr, _, _ = P.rope_pool(q, q, grid, cfg, 16)
    want = R.rotate_rows(q[0, 0].double().cpu().numpy(), grid_s, split)
    np.testing.assert_allclose(qr[0, 0].double().cpu().numpy(), want, rtol=0, atol=2e-6)


def test_forward_from_unrotated_equals_prerotated():
    import gpu_helpers as G
    import paper_2605_20659_b200 as P

    grid_s, split = (3, 8, 40), (16, 56, 56)
    q, k, v, x, params, pe, grid = G.make_full_inputs(grid_s, 4, 128, split, 64, seed=9)
    cfg = P.RopeConfig(*split)
    gen = torch.Generator(device="cuda").manual_seed(5)
    qu = torch.randn(q.shape, generator=gen, device="cuda").to(torch.bfloat16)
    ku = torch.randn(k.shape, generator=gen, device="cuda").to(torch.bfloat16)
    st = P.ForwardSettings(P.SparseSettings.for_sparsity(128, grid.size, 0.7))
    fused = P.forward(qu, ku, v, x, grid, params, st, pe, trace=True, rope=cfg)
    qr = P.rotate_rows(qu, grid, cfg).to(torch.bfloat16)
    kr = P.rotate_rows(ku, grid, cfg).to(torch.bfloat16)
    ref = P.forward(qr, kr, v, x, grid, params, st, pe, trace=True)
    torch.cuda.synchronize()
    assert torch.equal(fused.selected, ref.selected)
    assert torch.equal(fused.attended, ref.attended)
    assert torch.equal(fused.output, ref.output)


def test_rope_pool_rejects_bad_split():
    import paper_2605_20659_b200 as P

    grid = P.GridShape(2, 2, 2)
    q = torch.zeros((1, 1, 8, 16), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        P.rope_pool(q, q, grid, P.RopeConfig(4, 4, 4), 4)  # 12 != 16
