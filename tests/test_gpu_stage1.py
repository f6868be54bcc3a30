"""Stage-I training on the device (training.py): loss and gradients against
the float64 oracle restatement of mechanism._fused_backward on the same
cached sparse branch, and a few gradient-descent steps reduce the loss."""

import math

import numpy as np
import pytest
import torch

import gpu_helpers as G
import restated as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _setup(dtype=torch.float32, seed=2):
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import training as T

    grid_s, split = (2, 4, 16), (16, 24, 24)
    H, d, r = 2, 64, 16
    q, k, v, x, params, pe, grid = G.make_full_inputs(grid_s, H, d, split, r, seed=seed, dtype=dtype)
    gen = torch.Generator(device="cuda").manual_seed(seed + 1)
    target = torch.randn((1, grid.size, H * d), generator=gen, device="cuda") * 0.5
    st = P.ForwardSettings(P.SparseSettings(block=32, topk=2))
    return P, T, q, k, v, x, params, pe, grid, target, st


def test_stage1_grads_match_oracle():
    P, T, q, k, v, x, params, pe, grid, target, st = _setup()
    prep = T.prepare([T.Stage1Sample(q, k, v, x, target)], grid, params, st, pe)
    pe_dense = pe.dense(grid).float()
    loss, grads = T.loss_and_grads(prep, params, st, T.pe_head_major(pe, grid, params.n_heads, params.d_h))
    torch.cuda.synchronize()
    H = params.n_heads
    p_np = {n: getattr(params, n).double().cpu().numpy() for n in T.PARAM_NAMES}
    p_np["b_g"] = params.b_g
    sparse = [prep[0].o_sparse[h].double().cpu().numpy() for h in range(H)]
    ref_loss, ref = R.align_loss_and_grads(x[0].double().cpu().numpy(), sparse, pe_dense.double().cpu().numpy(),
                                           target[0].double().cpu().numpy(), p_np)
    assert abs(loss - ref_loss) <= 1e-5 * abs(ref_loss)
    for name in T.PARAM_NAMES:
        got = grads[name].double().cpu().numpy()
        want = ref[name]
        scale = max(np.abs(want).max(), 1e-12)
        assert np.abs(got - want).max() <= 2e-4 * scale, name
    assert abs(grads["b_g"] - ref["b_g"]) <= 2e-4 * max(abs(ref["b_g"]), 1e-9)


def test_stage1_training_reduces_loss():
    P, T, q, k, v, x, params, pe, grid, target, st = _setup(seed=4)
    res = T.train_stage1([T.Stage1Sample(q, k, v, x, target)], grid, params, st, pe, lr=0.5, steps=5)
    assert not res.diverged
    assert res.final_loss < res.initial_loss
