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


@pytest.mark.parametrize("path", ["fused", "composed"])
def test_stage1_grads_match_oracle(path):
    P, T, q, k, v, x, params, pe, grid, target, st = _setup()
    prep = T.prepare([T.Stage1Sample(q, k, v, x, target)], grid, params, st, pe)
    pe_dense = pe.dense(grid).float()
    fn = T.loss_and_grads if path == "fused" else T._loss_and_grads_composed
    loss, grads = fn(prep, params, st, T.pe_head_major(pe, grid, params.n_heads, params.d_h))
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


@pytest.mark.parametrize("d,split,r,nsamp", [(128, (16, 56, 56), 64, 1), (64, (16, 24, 24), 16, 2)])
def test_stage1_captured_step_equals_eager(d, split, r, nsamp):
    """The CUDA-graph step (training.Stage1Step: loss, gradients and the
    device-side update) against the eager loop of the same kernels: the
    same losses and bit-identical parameters after three steps; a diverging
    step leaves the parameters untouched."""
    import copy

    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import training as T

    grid_s, H = (2, 6, 20), 2
    q, k, v, x, params, pe, grid = G.make_full_inputs(grid_s, H, d, split, r, seed=9, dtype=torch.bfloat16)
    gen = torch.Generator(device="cuda").manual_seed(10)
    samples = [T.Stage1Sample(q, k, v, x, torch.randn((1, grid.size, H * d), generator=gen, device="cuda").to(
        torch.bfloat16)) for _ in range(nsamp)]
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=2))
    prep = T.prepare(samples, grid, params, st, pe)
    pe_hm = T.pe_head_major(pe, grid, H, d)
    lr = 0.05
    p_eager = copy.deepcopy(params)
    eager = []
    for _ in range(3):
        loss, grads = T.loss_and_grads(prep, p_eager, st, pe_hm)
        eager.append(loss)
        with torch.no_grad():
            for name in T.PARAM_NAMES:
                getattr(p_eager, name).sub_(lr * grads[name].to(getattr(p_eager, name).dtype))
        p_eager.b_g = float(p_eager.b_g) - lr * grads["b_g"]
    runner = T.Stage1Step(prep, params, st, pe_hm, lr)
    captured = [runner.step() for _ in range(3)]
    runner.sync_bias()
    assert captured == eager
    for name in T.PARAM_NAMES:
        assert torch.equal(getattr(params, name), getattr(p_eager, name)), name
    assert params.b_g == p_eager.b_g
    # a non-finite loss: no update
    before = {n: getattr(params, n).clone() for n in T.PARAM_NAMES}
    prep[0].target.fill_(float("nan"))
    assert not math.isfinite(runner.step())
    for name in T.PARAM_NAMES:
        assert torch.equal(getattr(params, name), before[name]), name


@pytest.mark.parametrize("use_pe", [True, False])
@pytest.mark.parametrize("d,split,r", [(128, (16, 56, 56), 32), (32, (8, 12, 12), 16)])
def test_stage1_fused_equals_composed(use_pe, d, split, r):
    """The fused row kernels (csrc/stage1.cu: 1 and 4 values per lane;
    d = 128 is the bench shape) against the torch composition of the same
    math, two samples (gradients accumulate over samples)."""
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import training as T

    grid_s, H = (2, 6, 20), 3
    q, k, v, x, params, pe, grid = G.make_full_inputs(grid_s, H, d, split, r, seed=6, dtype=torch.float32)
    gen = torch.Generator(device="cuda").manual_seed(8)
    samples = [T.Stage1Sample(q, k, v, x, torch.randn((1, grid.size, H * d), generator=gen, device="cuda") * 0.5)
               for _ in range(2)]
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=2), use_pe=use_pe)
    prep = T.prepare(samples, grid, params, st, pe)
    pe_hm = T.pe_head_major(pe, grid, H, d) if use_pe else None
    loss_f, gf = T.loss_and_grads(prep, params, st, pe_hm)
    loss_c, gc = T._loss_and_grads_composed(prep, params, st, pe_hm)
    assert abs(loss_f - loss_c) <= 1e-6 * abs(loss_c)
    for name in T.PARAM_NAMES:
        if name == "alpha" and not use_pe:
            assert torch.count_nonzero(gf[name]) == 0
            continue
        scale = float(gc[name].abs().max()) or 1.0
        assert float((gf[name] - gc[name]).abs().max()) <= 2e-5 * scale, name
    assert abs(gf["b_g"] - gc["b_g"]) <= 2e-5 * max(abs(gc["b_g"]), 1e-9)


@pytest.mark.parametrize("K,N", [(128, 64), (64, 128), (128, 128)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_stage1_tensor_core_gemms_float32_grade(K, N, epi):
    """The tcgen05 GEMMs of the step (bf16 hi + lo split, three MMAs): rows
    C = epi(A B) and gram A^T B against float64, within 5e-5 relative (float32
    grade, far inside the 2e-4 gradient bar); ragged L."""
    from paper_2605_20659_b200 import training as T

    g = torch.Generator(device="cuda").manual_seed(K + N + epi)
    H, L = 3, 1000
    A = torch.randn((H, L, K), generator=g, device="cuda")
    B = torch.randn((H, K, N), generator=g, device="cuda") / K ** 0.5
    aux = torch.rand((H, L, N), generator=g, device="cuda")
    got = T._rows(A, B, epi=epi, aux=aux if epi == 2 else None)
    want = torch.bmm(A.double(), B.double())
    if epi == 1:
        want = torch.sigmoid(want)
    elif epi == 2:
        want = want * aux.double() * (1 - aux.double())
    rel = ((got.double() - want).abs().max() / want.abs().max()).item()
    assert rel < 5e-5, rel
    got_t = T._rows(A, B.transpose(1, 2).contiguous(), b_trans=True)
    rel = ((got_t.double() - torch.bmm(A.double(), B.double())).abs().max() / want.abs().max()).item()
    assert rel < 5e-5, rel
    if K == 128:
        Bt = torch.randn((H, L, N), generator=g, device="cuda")
        out = torch.zeros((H, 128, N), device="cuda")
        T._gram_into(out, A, Bt, transpose=False)
        ref = torch.bmm(A.double().transpose(1, 2), Bt.double())
        assert ((out.double() - ref).abs().max() / ref.abs().max()).item() < 5e-5
        out_t = torch.ones((H, N, 128), device="cuda")
        T._gram_into(out_t, A, Bt, transpose=True)
        assert ((out_t.double() - 1 - ref.transpose(1, 2)).abs().max() / ref.abs().max()).item() < 5e-5
