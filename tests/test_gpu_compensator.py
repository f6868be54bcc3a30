"""K3 (low-rank compensator + PE injection + gate) against the float64
oracle at every rank the kernels specialise: r in {16, 32, 48, 64} runs the
tcgen05/TMA kernel, r = 128 the mma.sync kernel, d = 64 the generic CUDA-core
kernel.  Ragged last token tile, batch 2, PE on and off."""

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


def _inputs(B, H, d, r, grid, seed, dtype=torch.bfloat16):
    import paper_2605_20659_b200 as P

    rng = np.random.default_rng(seed)
    L = grid[0] * grid[1] * grid[2]
    D = H * d
    x = rng.standard_normal((B, L, D))
    pe = [rng.standard_normal((n, D)) * 0.02 for n in grid]
    w_a = rng.standard_normal((H, d, r)) / math.sqrt(d)
    w_b = rng.standard_normal((H, r, d)) / math.sqrt(d)
    params = P.MechanismParams.from_arrays(device="cuda", w_a=w_a, w_b=w_b, alpha=np.full(D, 0.1),
                                           w_g=rng.standard_normal(D) * 0.05, b_g=-2.0,
                                           rms_sparse=np.ones(d), rms_lowrank=1.0 + 0.1 * rng.standard_normal(d))
    xd = torch.from_numpy(x).to(dtype).cuda().contiguous()
    pet = P.PETables(*(torch.from_numpy(t).float().cuda() for t in pe))
    return xd, params, pet, P.GridShape(*grid)


@pytest.mark.parametrize("r", [16, 32, 48, 64, 128])
@pytest.mark.parametrize("use_pe", [True, False])
def test_lowrank_branch_vs_oracle(r, use_pe):
    import paper_2605_20659_b200 as P

    B, H, d = 2, 3, 128
    grid_s = (3, 5, 20)  # L = 300: the last 128-token tile has 44 tokens
    x, params, pe, grid = _inputs(B, H, d, r, grid_s, seed=r + use_pe)
    st = P.ForwardSettings(P.SparseSettings(64, topk=1), use_pe=use_pe)
    y_lr, o_lr, g_logit = P.compensator_branch(x, grid, params, st, pe, want_o_lr=True)
    torch.cuda.synchronize()
    L, D = grid.size, H * d
    c = R.grid_coords(*grid_s)
    pe_np = [t.cpu().numpy().astype(np.float64) for t in (pe.pe_t, pe.pe_x, pe.pe_y)]
    pe_dense = pe_np[0][c[:, 0]] + pe_np[1][c[:, 1]] + pe_np[2][c[:, 2]]
    alpha = params.alpha.cpu().numpy().astype(np.float64)
    w_a = params.w_a.cpu().numpy().astype(np.float64)
    w_b = params.w_b.cpu().numpy().astype(np.float64)
    w_g = params.w_g.cpu().numpy().astype(np.float64)
    rms_lr = params.rms_lowrank.cpu().numpy().astype(np.float64)
    for b in range(B):
        xb = x[b].double().cpu().numpy()
        x_hat = xb + alpha[None] * pe_dense if use_pe else xb
        g_ref = x_hat @ w_g
        np.testing.assert_allclose(g_logit[b].cpu().numpy(), g_ref, rtol=0, atol=2e-3 * max(1.0, np.abs(g_ref).max()))
        for h in range(H):
            o_ref = R.lowrank_compensator(x_hat, w_a, w_b, h)
            G.assert_close(o_lr[b, h].cpu().numpy(), o_ref, "bf16", f"r{r} b{b} h{h} o_lr")
            y_ref = R.rms_norm(o_ref, rms_lr)
            G.assert_close(y_lr[b, :, h].float().cpu().numpy(), y_ref, "bf16", f"r{r} b{b} h{h} y_lr")


def test_lowrank_generic_d64_vs_oracle():
    import paper_2605_20659_b200 as P

    B, H, d, r = 1, 2, 64, 16
    grid_s = (2, 4, 9)
    x, params, pe, grid = _inputs(B, H, d, r, grid_s, seed=7, dtype=torch.float32)
    st = P.ForwardSettings(P.SparseSettings(8, topk=1))
    y_lr, o_lr, g_logit = P.compensator_branch(x, grid, params, st, pe, want_o_lr=True)
    torch.cuda.synchronize()
    c = R.grid_coords(*grid_s)
    pe_np = [t.cpu().numpy().astype(np.float64) for t in (pe.pe_t, pe.pe_x, pe.pe_y)]
    x_hat = x[0].double().cpu().numpy() + params.alpha.cpu().numpy()[None] * (
        pe_np[0][c[:, 0]] + pe_np[1][c[:, 1]] + pe_np[2][c[:, 2]])
    for h in range(H):
        o_ref = R.lowrank_compensator(x_hat, params.w_a.double().cpu().numpy(), params.w_b.double().cpu().numpy(), h)
        G.assert_close(o_lr[0, h].cpu().numpy(), o_ref, "f32", f"d64 h{h} o_lr")


@pytest.mark.parametrize("L_grid", [(2, 25, 50), (1, 8, 16)])
def test_linear_branch_tensor_cores_vs_oracle(L_grid):
    """K3 linear mode (mechanism.py:33-36, 347-362) on the tensor cores
    (linear_tc.cu: bf16, d = 128) against the float64 oracle, with a token
    count that is ragged for both the 1024-token state chunks and the
    128-token apply tiles, batch 2; and against the CUDA-core kernels."""
    import paper_2605_20659_b200 as P

    B, H, d = 2, 2, 128
    L = L_grid[0] * L_grid[1] * L_grid[2]
    x, params, pe, grid = _inputs(B, H, d, 64, L_grid, seed=11)
    rng = np.random.default_rng(12)
    lin = [torch.from_numpy(rng.standard_normal((B, H, L, d)) * 0.5).to(torch.bfloat16).cuda() for _ in range(3)]
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=1), compensator="linear")
    outs = {}
    for mode in ("tc", "simt"):
        with P._lib.option("linear_simt", int(mode == "simt")):
            y_lr, o_lr, _ = P.compensator_branch(x, grid, params, st, pe, lin_proj=lin, want_o_lr=True)
            torch.cuda.synchronize()
        outs[mode] = (y_lr.float().cpu().numpy(), o_lr.cpu().numpy())
    rms = params.rms_lowrank.double().cpu().numpy()
    for b in range(B):
        for h in range(H):
            qh, kh, vh = (t[b, h].double().cpu().numpy() for t in lin)
            o = R.linear_apply(qh, *R.linear_state(kh, vh))
            y = o / np.sqrt((o ** 2).mean(-1, keepdims=True) + st.rms_eps) * rms
            for mode in ("tc", "simt"):
                G.assert_close(outs[mode][1][b, h], o, "bf16", f"o_lr {mode} b{b} h{h}")
                G.assert_close(outs[mode][0][b, :, h], y, "bf16", f"y_lr {mode} b{b} h{h}")


def _linear_pe_case(B, H, d, grid_s, seed, sin_pe=False):
    """Inputs of the PE-injecting linear path: X (bf16), backbone weights
    W_{q,k,v} (float32 [H, D, d]) and the projections x W (bf16, no PE)."""
    import paper_2605_20659_b200 as P

    x, params, pe, grid = _inputs(B, H, d, 64, grid_s, seed=seed)
    D = H * d
    g = torch.Generator(device="cuda").manual_seed(seed)
    W = [torch.randn((H, D, d), generator=g, device="cuda") / math.sqrt(D) for _ in range(3)]
    if sin_pe:  # the reference's sinusoidal table (values up to 1): large PE terms
        pe = P.PETables.sinusoidal(grid, D, P.RopeConfig(44, 42, 42))
    lin = tuple(torch.einsum("bld,hde->bhle", x.double(), w.double()).to(torch.bfloat16).contiguous() for w in W)
    return x, params, pe, grid, W, lin


def _linear_oracle(x, params, pe, grid_s, W, lin, use_pe, b, h):
    """float64 oracle on the kernel's own inputs: k = bf16(x W) + (alpha PE) W
    (mechanism.py:350-362 with x_hat = x + alpha PE, mechanism.py:429-432)."""
    c = R.grid_coords(*grid_s)
    pe_np = [t.cpu().numpy().astype(np.float64) for t in (pe.pe_t, pe.pe_x, pe.pe_y)]
    pe_dense = pe_np[0][c[:, 0]] + pe_np[1][c[:, 1]] + pe_np[2][c[:, 2]]
    alpha = params.alpha.cpu().numpy().astype(np.float64)
    qkv = []
    for z in range(3):
        t = lin[z][b, h].double().cpu().numpy()
        if use_pe:
            t = t + (alpha[None] * pe_dense) @ W[z][h].double().cpu().numpy()
        qkv.append(t)
    smat, svec = R.linear_state(qkv[1], qkv[2])
    o = R.linear_apply(qkv[0], smat, svec)
    xb = x[b].double().cpu().numpy()
    x_hat = xb + alpha[None] * pe_dense if use_pe else xb
    g_ref = x_hat @ params.w_g.cpu().numpy().astype(np.float64)
    return o, smat, svec, g_ref


@pytest.mark.parametrize("grid_s,use_pe,sin_pe", [((3, 7, 11), True, False), ((3, 7, 11), False, False),
                                                   ((2, 16, 40), True, True), ((1, 8, 16), True, False)])
def test_linear_pe_tensor_cores_vs_oracle(grid_s, use_pe, sin_pe):
    """The tcgen05 linear compensator with the PE injection in the kernels
    (csrc/linear_umma.cu): state S, z, the raw output, y_lr and the gate
    logits against the float64 oracle; ragged last tile (L = 231), batch 2."""
    import paper_2605_20659_b200 as P

    B, H, d = 2, 3, 128
    x, params, pe, grid, W, lin = _linear_pe_case(B, H, d, grid_s, seed=31, sin_pe=sin_pe)
    st = P.ForwardSettings(P.SparseSettings(64, topk=1), compensator="linear", use_pe=use_pe)
    y_lr, o_lr, g_logit, state = P.compensator_branch(x, grid, params, st, pe, lin_proj=lin, lin_weights=W,
                                                      want_o_lr=True, want_state=True)
    torch.cuda.synchronize()
    rms = params.rms_lowrank.double().cpu().numpy()
    for b in range(B):
        for h in range(H):
            o, smat, svec, g_ref = _linear_oracle(x, params, pe, grid_s, W, lin, use_pe, b, h)
            s_dev = state[b * H + h].double().cpu().numpy()
            G.assert_close(s_dev[:, :128] / np.abs(smat).max(), smat / np.abs(smat).max(), "bf16", f"S b{b} h{h}")
            G.assert_close(s_dev[:, 128] / np.abs(svec).max(), svec / np.abs(svec).max(), "bf16", f"z b{b} h{h}")
            G.assert_close(o_lr[b, h].cpu().numpy(), o, "bf16", f"o_lr b{b} h{h}")
            y = o / np.sqrt((o ** 2).mean(-1, keepdims=True) + st.rms_eps) * rms
            G.assert_close(y_lr[b, :, h].float().cpu().numpy(), y, "bf16", f"y_lr b{b} h{h}")
            np.testing.assert_allclose(g_logit[b].cpu().numpy(), g_ref, rtol=0,
                                       atol=2e-3 * max(1.0, np.abs(g_ref).max()))


def test_linear_pe_tables_are_cached():
    """The parameter-only PE fold is computed once and reused until a
    parameter changes (version counter)."""
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import mechanism as Mm

    x, params, pe, grid, W, lin = _linear_pe_case(1, 2, 128, (2, 8, 16), seed=3)
    st = P.ForwardSettings(P.SparseSettings(64, topk=1), compensator="linear")
    t1 = Mm.linear_tables(x, grid, params, pe, True, W)
    t2 = Mm.linear_tables(x, grid, params, pe, True, W)
    assert t1.data_ptr() == t2.data_ptr()
    params.alpha.mul_(1.5)
    t3 = Mm.linear_tables(x, grid, params, pe, True, W)
    assert t3.data_ptr() != t1.data_ptr()
    y1 = P.compensator_branch(x, grid, params, st, pe, lin_proj=lin, lin_weights=W)[0]
    y2 = P.compensator_branch(x, grid, params, st, pe, lin_proj=lin, lin_weights=W)[0]
    assert torch.equal(y1, y2)


@pytest.mark.slow
def test_lowrank_tables_are_cached(monkeypatch):
    """The low-rank branch's parameter-only tables (W_A / W_B images, per-axis
    PE folds) are built once and reused until a parameter changes; the folded
    call equals the per-call fold bit for bit."""
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import mechanism as Mm

    q, k, v, x, params, pe, grid = G.make_full_inputs((3, 8, 16), 2, 128, (44, 42, 42), 64, seed=6)
    st = P.ForwardSettings(P.SparseSettings(64, topk=1))
    t1 = Mm.lowrank_tables(x, grid, params, pe, True)
    t2 = Mm.lowrank_tables(x, grid, params, pe, True)
    assert t1 is not None and t1.data_ptr() == t2.data_ptr()
    y1, _, g1 = P.compensator_branch(x, grid, params, st, pe)
    with monkeypatch.context() as m:
        m.setattr(Mm, "lowrank_tables", lambda *a, **kw: None)  # the per-call fold
        y0, _, g0 = P.compensator_branch(x, grid, params, st, pe)
    torch.cuda.synchronize()
    assert torch.equal(y1, y0) and torch.equal(g1, g0)
    params.w_a.mul_(0.5)
    t3 = Mm.lowrank_tables(x, grid, params, pe, True)
    assert t3.data_ptr() != t1.data_ptr()
    y3, _, _ = P.compensator_branch(x, grid, params, st, pe)
    with monkeypatch.context() as m:
        m.setattr(Mm, "lowrank_tables", lambda *a, **kw: None)
        y4, _, _ = P.compensator_branch(x, grid, params, st, pe)
    torch.cuda.synchronize()
    assert torch.equal(y3, y4) and not torch.equal(y3, y1)


def test_linear_forward_config1_fullsize():
    """Linear mode through the whole forward at the config-1 shape (L = 32760,
    H = 12, d = 128, block 64, top-51, bf16): the compensator of three heads
    over every token, and the fused output of sampled query blocks, against
    the float64 oracle."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = G.make_full_inputs((21, 30, 52), 12, 128, (44, 42, 42), 64, seed=4)
    H, d, L = 12, 128, grid.size
    D = H * d
    gen = torch.Generator(device="cuda").manual_seed(9)
    W = [torch.randn((H, D, d), generator=gen, device="cuda") / math.sqrt(D) for _ in range(3)]
    lin = tuple(torch.einsum("bld,hde->bhle", x.double(), w.double()).to(torch.bfloat16).contiguous() for w in W)
    st = P.ForwardSettings(P.SparseSettings.for_sparsity(64, L, 0.9), compensator="linear")
    tr = P.forward(q, k, v, x, grid, params, st, pe, lin_proj=lin, lin_weights=W, trace=True)
    out32 = P.forward(q, k, v, x, grid, params, st, pe, lin_proj=lin, lin_weights=W, out_dtype=torch.float32)
    torch.cuda.synchronize()
    grid_s = (21, 30, 52)
    members = R.flat_block_members(L, 64)
    rng = np.random.default_rng(2)
    x_np = x[0].float().cpu().numpy()
    rms_lr = params.rms_lowrank.double().cpu().numpy()
    g_ref_all = None
    for h in (0, 5, 11):
        o, _, _, g_ref = _linear_oracle(x, params, pe, grid_s, W, lin, True, 0, h)
        g_ref_all = g_ref
        G.assert_close(tr.o_lowrank[0, h].cpu().numpy(), o, "bf16", f"cfg1 linear o_lr h{h}")
        # fused output on sampled query blocks: the oracle's sparse branch and gate
        qh, kh, vh = (t[0, h].double().cpu().numpy() for t in (q, k, v))
        ref_sel, _ = R.select_blocks(R.block_scores(qh, kh, members), topk=st.sparse.topk)
        np.testing.assert_array_equal(tr.selected[0, h].cpu().numpy(), ref_sel)
        qbs = sorted(rng.choice(len(members), size=3, replace=False).tolist() + [len(members) - 1])
        rows = np.concatenate([members[b] for b in qbs])
        o_sp = G.oracle_rows(qh, kh, vh, members, ref_sel, qbs)[rows]
        gate = R.sigmoid(g_ref[rows] + params.b_g)
        y = R.rms_norm(o_sp, params.rms_sparse.double().cpu().numpy()) + gate[:, None] * R.rms_norm(o[rows], rms_lr)
        G.assert_close(out32[0].cpu().numpy()[rows, h * d:(h + 1) * d], y, "bf16", f"cfg1 linear out f32 h{h}")
        G.assert_close_bf16_store(tr.output[0].float().cpu().numpy()[rows, h * d:(h + 1) * d], y,
                                  f"cfg1 linear out h{h}")
    g_dev = tr.g[0].double().cpu().numpy()
    G.assert_close(g_dev, R.sigmoid(g_ref_all + params.b_g), "bf16", "cfg1 linear gate")
