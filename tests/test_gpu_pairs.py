"""Block-64 K2 units of two adjacent query blocks over the union of their
selections (csrc/attn_sm100.cu, sparse_attn_fixed_kernel<128, 64, true>,
union_pairs_kernel): every row must attend exactly its own query block's
selection.  Checked against the float64 oracle and against the one-block
units (option pairs64 = 0) on rows whose neighbours share almost all of
their selection (the config-4 DiT's case), share none of it, on an odd
block count with a ragged last block, and under the keep rule."""

import numpy as np
import pytest
import torch

import gpu_helpers as G
from test_gpu_parity import _oracle_sparse, _small

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _run(q, k, v, sp, pairs):
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import _lib

    with _lib.option("pairs64", pairs):
        res = P.block_sparse_attention(q, k, v, sp)
    torch.cuda.synchronize()
    return res


def _check(q, k, v, sp, **rule):
    a = _run(q, k, v, sp, 1)
    b = _run(q, k, v, sp, 0)
    assert torch.equal(a.selected, b.selected)
    ref_out, ref_sel = _oracle_sparse(q, k, v, 64, **rule)
    np.testing.assert_array_equal(a.selected[0].cpu().numpy(), ref_sel)
    got = a.output[0].double().cpu().numpy()
    scale = float(np.sqrt(np.mean(ref_out ** 2)))
    G.assert_close(got / scale, ref_out / scale, "bf16", "pairs vs oracle")
    G.assert_close(got / scale, b.output[0].double().cpu().numpy() / scale, "bf16", "pairs vs single units")
    return a


@pytest.mark.parametrize("share", ["high", "none"])
def test_pairs_against_oracle(share):
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((3, 11, 19), H=2)  # L = 627: nb = 10, last block 51 rows
    if share == "high":
        # the second block of each pair repeats the first one's queries plus
        # noise: nearly the same selection, not the same
        L = q.shape[2]
        qf = q.float()
        for p0 in range(0, L - 64, 128):
            n = min(64, L - p0 - 64)
            qf[:, :, p0 + 64:p0 + 64 + n] = qf[:, :, p0:p0 + n] + 0.3 * torch.randn_like(qf[:, :, p0:p0 + n])
        q = qf.to(q.dtype)
    else:
        # adjacent blocks select disjoint key blocks: opposite query directions
        qf = q.float()
        L = q.shape[2]
        for p0 in range(0, L - 64, 128):
            n = min(64, L - p0 - 64)
            qf[:, :, p0 + 64:p0 + 64 + n] = -qf[:, :, p0:p0 + n]
        q = qf.to(q.dtype)
    sp = P.SparseSettings(block=64, topk=3)
    _check(q, k, v, sp, topk=3)


def test_pairs_keep_rule_odd_blocks():
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((1, 9, 25), H=3)  # L = 225: nb = 4 ... ragged
    q2, k2, v2, _, _, _, _ = _small((5, 9, 15), H=2, seed=3)  # L = 675: nb = 11 (odd), last block 35 rows
    for (qq, kk, vv) in ((q, k, v), (q2, k2, v2)):
        for keep in (0.3, 0.8):
            _check(qq, kk, vv, P.SparseSettings(block=64, keep=keep), keep=keep)
