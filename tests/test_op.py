"""The PyTorch custom ops (paper_2605_20659_b200/op.py): fake kernels give the
shapes / dtypes the CUDA path returns (CPU, no GPU needed), and on a B200
the ops equal the Python mirror they wrap."""

import pytest
import torch

import paper_2605_20659_b200.op  # noqa: F401  (registers torch.ops.ropeslr.*)


def test_fake_kernels_shapes():
    from torch._subclasses.fake_tensor import FakeTensorMode

    with FakeTensorMode():
        q = torch.empty((1, 2, 300, 128), dtype=torch.bfloat16)
        idx, cnt, att = torch.ops.ropeslr.select_blocks(q, q, 64, 2, 1.0)
        assert idx.shape == (1, 2, 5, 2) and idx.dtype == torch.int32
        assert cnt.shape == (1, 2, 5) and att.shape == (1, 2) and att.dtype == torch.int64
        idx, _, _ = torch.ops.ropeslr.select_blocks(q, q, 64, 0, 0.5)
        assert idx.shape == (1, 2, 5, 5)  # keep rule: up to every block
        x = torch.empty((1, 300, 256), dtype=torch.bfloat16)
        y, g = torch.ops.ropeslr.compensator_fwd(x, torch.empty(3, 256), torch.empty(10, 256), torch.empty(10, 256),
                                                 torch.empty(256), torch.empty(2, 128, 64), torch.empty(2, 64, 128),
                                                 torch.empty(256), torch.empty(128), [3, 10, 10], True, 1e-6)
        assert y.shape == (1, 300, 2, 128) and y.dtype == torch.bfloat16
        assert g.shape == (1, 300) and g.dtype == torch.float32
        out = torch.ops.ropeslr.attn_fwd(q, q, q, x, torch.empty(3, 256), torch.empty(10, 256), torch.empty(10, 256),
                                         torch.empty(256), torch.empty(2, 128, 64), torch.empty(2, 64, 128),
                                         torch.empty(256), -2.0, torch.empty(128), torch.empty(128), [3, 10, 10], 64,
                                         2, 1.0, True, 1e-6)
        assert out.shape == (1, 300, 256) and out.dtype == torch.bfloat16


@pytest.mark.gpu
def test_ops_equal_the_mirror():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import gpu_helpers as G

    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = G.make_full_inputs((2, 8, 16), 2, 128, (44, 42, 42), 64, seed=2)
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=2))
    want = P.forward(q, k, v, x, grid, params, st, pe)
    got = torch.ops.ropeslr.attn_fwd(q, k, v, x, pe.pe_t, pe.pe_x, pe.pe_y, params.alpha, params.w_a, params.w_b,
                                     params.w_g, float(params.b_g), params.rms_sparse, params.rms_lowrank,
                                     list(grid.as_tuple()), 64, 2, 1.0, True, st.rms_eps)
    assert torch.equal(got, want)
    sel = P.select_blocks(q, k, st.sparse, want_mask=False)
    idx, cnt, att = torch.ops.ropeslr.select_blocks(q, k, 64, 2, 1.0)
    assert torch.equal(idx, sel.idx) and torch.equal(cnt, sel.cnt) and torch.equal(att, sel.attended)
    y_lr, _, g_logit = P.compensator_branch(x, grid, params, st, pe)
    y2, g2 = torch.ops.ropeslr.compensator_fwd(x, pe.pe_t, pe.pe_x, pe.pe_y, params.alpha, params.w_a, params.w_b,
                                               params.w_g, params.rms_lowrank, list(grid.as_tuple()), True,
                                               st.rms_eps)
    assert torch.equal(y2, y_lr) and torch.equal(g2, g_logit)


def test_attn_fwd_schema_has_the_compensator():
    """torch.ops.ropeslr.attn_fwd carries the compensator mode and the linear
    branch's inputs (fake kernel, CPU)."""
    from torch._subclasses.fake_tensor import FakeTensorMode

    schema = str(torch.ops.ropeslr.attn_fwd.default._schema)
    for name in ("compensator", "q_lin", "k_lin", "v_lin", "w_lin_q", "w_lin_k", "w_lin_v"):
        assert name in schema
    with FakeTensorMode():
        q = torch.empty((1, 2, 300, 128), dtype=torch.bfloat16)
        x = torch.empty((1, 300, 256), dtype=torch.bfloat16)
        out = torch.ops.ropeslr.attn_fwd(q, q, q, x, torch.empty(3, 256), torch.empty(10, 256), torch.empty(10, 256),
                                         torch.empty(256), torch.empty(2, 128, 64), torch.empty(2, 64, 128),
                                         torch.empty(256), -2.0, torch.empty(128), torch.empty(128), [3, 10, 10], 64,
                                         2, 1.0, True, 1e-6, "linear", q, q, q, torch.empty(2, 256, 128),
                                         torch.empty(2, 256, 128), torch.empty(2, 256, 128))
        assert out.shape == (1, 300, 256)


@pytest.mark.gpu
def test_attn_fwd_linear_equals_the_mirror():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import math

    import gpu_helpers as G

    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = G.make_full_inputs((2, 8, 16), 2, 128, (44, 42, 42), 64, seed=5)
    gen = torch.Generator(device="cuda").manual_seed(1)
    W = [torch.randn((2, 256, 128), generator=gen, device="cuda") / math.sqrt(256) for _ in range(3)]
    lin = [torch.einsum("bld,hde->bhle", x.float(), w).to(torch.bfloat16).contiguous() for w in W]
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=2), compensator="linear")
    want = P.forward(q, k, v, x, grid, params, st, pe, lin_proj=lin, lin_weights=W)
    got = torch.ops.ropeslr.attn_fwd(q, k, v, x, pe.pe_t, pe.pe_x, pe.pe_y, params.alpha, params.w_a, params.w_b,
                                     params.w_g, float(params.b_g), params.rms_sparse, params.rms_lowrank,
                                     list(grid.as_tuple()), 64, 2, 1.0, True, st.rms_eps, "linear", *lin, *W)
    assert torch.equal(got, want)
