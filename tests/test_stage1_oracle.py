"""The Stage-I backward restatement (oracle/restated.fused_backward):
finite differences on the restatement itself, and the unmodified reference
(mechanism._fused_backward) when /root/reference is present."""

import os
import sys

import numpy as np
import pytest

import restated as R

REF = "/root/reference/pkg/src"


def _problem(seed=0, L=12, H=2, d=4, r=3):
    rng = np.random.default_rng(seed)
    D = H * d
    params = dict(w_a=rng.standard_normal((H, d, r)) * 0.7, w_b=rng.standard_normal((H, r, d)) * 0.7,
                  alpha=rng.standard_normal(D) * 0.3, w_g=rng.standard_normal(D) * 0.3, b_g=-0.4,
                  rms_sparse=1.0 + 0.1 * rng.standard_normal(d), rms_lowrank=1.0 + 0.1 * rng.standard_normal(d))
    x = rng.standard_normal((L, D))
    pe = rng.standard_normal((L, D)) * 0.5
    sparse = [rng.standard_normal((L, d)) for _ in range(H)]
    target = rng.standard_normal((L, D))
    return x, sparse, pe, target, params


def test_fused_backward_matches_finite_differences():
    x, sparse, pe, target, params = _problem()
    _, grads = R.align_loss_and_grads(x, sparse, pe, target, params)
    eps = 1e-6
    worst = 0.0
    for name in ("w_a", "w_b", "alpha", "w_g", "rms_sparse", "rms_lowrank", "b_g"):
        arr = params[name]
        if name == "b_g":
            up = dict(params, b_g=arr + eps)
            dn = dict(params, b_g=arr - eps)
            num = (R.align_loss_and_grads(x, sparse, pe, target, up)[0]
                   - R.align_loss_and_grads(x, sparse, pe, target, dn)[0]) / (2 * eps)
            worst = max(worst, abs(grads[name] - num) / (abs(num) + 1e-8))
            continue
        flat = arr.reshape(-1)
        for i in range(flat.size):
            orig = flat[i]
            flat[i] = orig + eps
            up = R.align_loss_and_grads(x, sparse, pe, target, params)[0]
            flat[i] = orig - eps
            dn = R.align_loss_and_grads(x, sparse, pe, target, params)[0]
            flat[i] = orig
            num = (up - dn) / (2 * eps)
            worst = max(worst, abs(grads[name].reshape(-1)[i] - num) / (abs(num) + 1e-8))
    assert worst < 1e-5, worst


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_fused_backward_matches_live_reference():
    sys.path.insert(0, REF)
    from ropeslr import mechanism as M

    x, sparse, pe, target, p = _problem(seed=3)
    H, d = len(sparse), sparse[0].shape[1]
    params = M.MechanismParams(w_a=p["w_a"].copy(), w_b=p["w_b"].copy(), alpha=p["alpha"].copy(),
                               w_g=p["w_g"].copy(), b_g=p["b_g"], rms_sparse=p["rms_sparse"].copy(),
                               rms_lowrank=p["rms_lowrank"].copy())
    backbone = M.Backbone(w_q=np.zeros((H, H * d, d)), w_k=np.zeros((H, H * d, d)), w_v=np.zeros((H, H * d, d)))
    settings = M.ForwardSettings(sparse=M.SparseSettings(block=(1, 1, 1), keep=1.0))
    out, cache = M._fused_forward(x, sparse, pe, None, None, backbone, params, settings)
    diff = out - target
    g_out = 2.0 * diff / diff.size
    grads = M.zero_grads(params)
    M._fused_backward(g_out, cache, pe, backbone, params, settings, grads)
    loss, mine = R.align_loss_and_grads(x, sparse, pe, target, p)
    assert abs(loss - float(np.mean(diff * diff))) < 1e-14
    for name in ("w_a", "w_b", "alpha", "w_g", "rms_sparse", "rms_lowrank"):
        np.testing.assert_allclose(mine[name], getattr(grads, name), rtol=1e-12, atol=1e-14, err_msg=name)
    assert abs(mine["b_g"] - grads.b_g) < 1e-13
