"""K1 under the cumulative-mass (`keep`) rule (csrc/select.cu,
select_keep_kernel): rows ordered by a radix sort on float32 score keys,
the exact float64 order restored inside runs of equal keys, then the mass
scan (mechanism.py:310-320, decomposition.py:105-111).  It must select
exactly what the round-1 bitonic-sort kernel (option keep_bitonic) selects,
on random rows and on rows built to stress the key: clusters of blocks
whose scores agree to far below float32 resolution, exact duplicates,
score spreads past the probability underflow, all-equal rows -- and the
oracle's selection on a small case."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _both(q, k, keep, block):
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import _lib

    sp = P.SparseSettings(block=block, keep=keep)
    with _lib.option("keep_bitonic", 0):
        a = P.select_blocks(q, k, sp)
    with _lib.option("keep_bitonic", 1):
        b = P.select_blocks(q, k, sp)
    torch.cuda.synchronize()
    for f in ("cnt", "attended", "mask"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f"keep={keep}: radix-sorted selection differs in {f}"
    # index lists: the first cnt entries of each row (the rest is not written)
    live = torch.arange(a.idx.shape[-1], device=a.idx.device) < a.cnt.unsqueeze(-1)
    assert torch.equal(torch.where(live, a.idx, -1), torch.where(live, b.idx, -1)), f"keep={keep}: idx differs"
    return a


def _rows(qb, kb, block):
    nb, d = qb.shape
    q = torch.from_numpy(np.repeat(qb, block, axis=0)).float().view(1, 1, nb * block, d).cuda()
    k = torch.from_numpy(np.repeat(kb, block, axis=0)).float().view(1, 1, nb * block, d).cuda()
    return q, k


KEEPS = (1e-9, 0.3, 0.9, 0.999, 1.0)


@pytest.mark.parametrize("nb,block,ragged", [(100, 64, 0), (300, 32, 5), (929, 128, 112), (1024, 32, 0)])
def test_keep_random(nb, block, ragged):
    g = torch.Generator(device="cuda").manual_seed(nb)
    L = nb * block - ragged
    q = torch.randn((1, 3, L, 128), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((1, 3, L, 128), generator=g, device="cuda").to(torch.bfloat16)
    for keep in KEEPS:
        _both(q, k, keep, block)


def test_keep_clusters_duplicates_and_underflow():
    rng = np.random.default_rng(5)
    nb, block, d = 320, 16, 64
    # clusters: 32 centres x 10 blocks within 1e-9 (one float32 key per cluster)
    centres = rng.standard_normal((32, d))
    kb = np.repeat(centres, 10, axis=0) + 1e-9 * rng.standard_normal((nb, d))
    kb[::7] = kb[1]  # exact duplicates
    qb = rng.standard_normal((nb, d))
    q, k = _rows(qb, kb, block)
    for keep in KEEPS:
        _both(q, k, keep, block)
    # spreads of ~1e4: most blocks underflow to probability 0 and tie
    q, k = _rows(40.0 * rng.standard_normal((nb, d)), 40.0 * rng.standard_normal((nb, d)), block)
    for keep in KEEPS:
        _both(q, k, keep, block)
    # one run over the whole row: every score equal to float32 resolution
    # but distinct in float64, in random order (the full-key radix path)
    base = rng.standard_normal(d)
    q, k = _rows(np.tile(rng.standard_normal(d), (nb, 1)), base + 1e-9 * rng.standard_normal((nb, d)), block)
    for keep in KEEPS:
        _both(q, k, keep, block)
    # every score equal: ties to the lower blocks
    z = np.zeros((nb, d))
    q, k = _rows(z, z, block)
    for keep in KEEPS:
        a = _both(q, k, keep, block)
    assert int(a.cnt.max()) == nb  # keep = 1 on a flat row takes every block


def test_keep_matches_oracle_small():
    import gpu_helpers as G

    rng = np.random.default_rng(9)
    nb, block, d = 96, 16, 64
    qb, kb = rng.standard_normal((nb, d)), rng.standard_normal((nb, d)) * 3.0
    q, k = _rows(qb, kb, block)
    qn, kn = q[0, 0].double().cpu().numpy(), k[0, 0].double().cpu().numpy()
    members = [np.arange(b * block, (b + 1) * block) for b in range(nb)]
    for keep in (0.2, 0.7, 0.95):
        a = _both(q, k, keep, block)
        want, _ = G.R.select_blocks(G.R.block_scores(qn, kn, members), keep=keep)
        got = a.mask[0, 0].cpu().numpy().astype(bool)
        assert np.array_equal(got, want), f"keep={keep}"
