"""Parity of the CUDA path (through the C ABI) with the float64 oracle.

Golden fixtures (tests/golden, generated from the unmodified reference by
oracle/make_golden.py): masks bit-exact, outputs within the north-star
tolerance (bf16: max-abs 2e-2, mean-rel 1e-2; f32: 1e-4 / 1e-5).
"""

import numpy as np
import pytest
import torch

import golden_io
import gpu_helpers as G
import restated as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2605_20659_b200 as P

    assert P.lib().ropeslr_device_check(torch.cuda.current_device()) == 0, "not an sm_100 device"


IMPLS = ["auto", "simt"]


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("name", golden_io.names())
def test_golden_forward(name, impl):
    import paper_2605_20659_b200 as P

    g = golden_io.load(name)
    q, k, v, x, params, pe, st, grid, lin = G.golden_to_device(g)
    tr = P.forward(q, k, v, x, grid, params, st, pe, lin_proj=lin, trace=True, impl=impl)
    torch.cuda.synchronize()
    sel = tr.selected[0].cpu().numpy()
    np.testing.assert_array_equal(sel, g["ref_selected"], err_msg=f"{name}: mask differs from the reference")
    np.testing.assert_allclose(tr.sparsity[0].cpu().numpy(), g["ref_sparsity"], rtol=0, atol=1e-15)
    dt = g["dtype"]
    # the sparse branch before normalisation: relative to its own scale
    o_sp = tr.o_sparse[0].cpu().numpy()
    ref = g["ref_o_sparse"]
    scale = float(np.sqrt(np.mean(ref ** 2)))
    G.assert_close(o_sp / scale, ref / scale, dt, f"{name} o_sparse/rms")
    G.assert_close(tr.o_lowrank[0].cpu().numpy(), g["ref_o_lowrank"], dt, f"{name} o_lowrank")
    G.assert_close(tr.g[0].cpu().numpy(), g["ref_g"], dt, f"{name} gate")
    G.assert_close(tr.output[0].float().cpu().numpy(), g["ref_output"], dt, f"{name} output")


@pytest.mark.parametrize("name", ["bf16_d128_keep", "bf16_d128_b128", "ragged_topk_bf16"])
def test_tcgen05_matches_simt(name):
    """The tensor-core kernel and the CUDA-core kernel agree (independent paths)."""
    import paper_2605_20659_b200 as P

    g = golden_io.load(name)
    q, k, v, x, params, pe, st, grid, lin = G.golden_to_device(g)
    a = P.forward(q, k, v, x, grid, params, st, pe, trace=True, impl="tcgen05")
    b = P.forward(q, k, v, x, grid, params, st, pe, trace=True, impl="simt")
    assert torch.equal(a.selected, b.selected)
    ra, rb = a.o_sparse.double(), b.o_sparse.double()
    rel = (ra - rb).abs().max() / rb.pow(2).mean().sqrt()
    assert rel < 2e-2, f"tcgen05 vs simt o_sparse rel err {rel:.3e}"


def test_deterministic():
    import paper_2605_20659_b200 as P

    g = golden_io.load("bf16_d128_b128")
    q, k, v, x, params, pe, st, grid, lin = G.golden_to_device(g)
    a = P.forward(q, k, v, x, grid, params, st, pe, trace=True)
    b = P.forward(q, k, v, x, grid, params, st, pe, trace=True)
    assert torch.equal(a.output, b.output)
    assert torch.equal(a.o_sparse, b.o_sparse)


# ---------------------------------------------------------------- edge cases


def _small(L_grid=(2, 4, 16), H=2, d=128, seed=0, dtype=torch.bfloat16):
    return G.make_full_inputs(L_grid, H, d, (44, 42, 42) if d == 128 else (16, 24, 24), 64 if d == 128 else 16,
                              seed=seed, dtype=dtype)


def _oracle_sparse(q, k, v, block, keep=None, topk=None):
    out, sels = [], []
    for h in range(q.shape[1]):
        qh, kh, vh = (t[0, h].double().cpu().numpy() for t in (q, k, v))
        members = R.flat_block_members(qh.shape[0], block)
        o, s, _, _, _ = R.block_sparse_attention(qh, kh, vh, members, keep=keep, topk=topk)
        out.append(o)
        sels.append(s)
    return np.stack(out), np.stack(sels)


@pytest.mark.parametrize("impl", ["tcgen05", "simt"])
@pytest.mark.parametrize("grid_shape,block,topk", [
    ((1, 1, 40), 64, 1),        # L < block: one ragged block
    ((1, 5, 13), 64, 1),        # L = 65: last block of one token
    ((3, 7, 11), 128, 2),       # ragged 128 blocks
    ((2, 8, 16), 64, 4),        # topk == nb: full attention
    ((2, 8, 16), 64, 9),        # topk > nb clamps to nb
])
def test_ragged_and_full(grid_shape, block, topk, impl):
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small(grid_shape)
    st = P.ForwardSettings(P.SparseSettings(block=block, topk=topk))
    res = P.block_sparse_attention(q, k, v, st.sparse, impl=impl)
    ref_out, ref_sel = _oracle_sparse(q, k, v, block, topk=topk)
    np.testing.assert_array_equal(res.selected[0].cpu().numpy(), ref_sel)
    got = res.output[0].double().cpu().numpy()
    scale = float(np.sqrt(np.mean(ref_out ** 2)))
    G.assert_close(got / scale, ref_out / scale, "bf16", "o_sparse/rms")
    if topk >= -(-grid.size // block):
        # full coverage == dense softmax attention
        for h in range(q.shape[1]):
            qh, kh, vh = (t[0, h].double() for t in (q, k, v))
            a = torch.softmax(qh @ kh.T / np.sqrt(q.shape[-1]), dim=-1) @ vh
            G.assert_close(got[h] / scale, a.cpu().numpy() / scale, "bf16", "dense")


@pytest.mark.parametrize("keep", [1e-9, 0.3, 0.8, 1.0])
def test_keep_rule(keep):
    """Cumulative-mass rule (mechanism.py:316-320) incl. the floor of one
    block and keep = 1."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((4, 8, 16), H=3)
    sp = P.SparseSettings(block=64, keep=keep)
    res = P.block_sparse_attention(q, k, v, sp)
    ref_out, ref_sel = _oracle_sparse(q, k, v, 64, keep=keep)
    np.testing.assert_array_equal(res.selected[0].cpu().numpy(), ref_sel)
    if keep == 1e-9:
        assert (res.selected.sum(-1) == 1).all()


def test_tie_goes_to_lower_block():
    """Identical key blocks score identically; the stable order keeps the
    lower block index (mechanism.py:317, test_decomposition.py:157-162)."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((2, 8, 16), H=1)
    k = k.clone()
    k[:, :, 128:192] = k[:, :, 0:64]    # block 2 == block 0
    k[:, :, 192:256] = k[:, :, 64:128]  # block 3 == block 1
    res = P.block_sparse_attention(q, k, v, P.SparseSettings(block=64, topk=1))
    sel = res.selected[0, 0].cpu().numpy()
    ref_out, ref_sel = _oracle_sparse(q, k, v, 64, topk=1)
    np.testing.assert_array_equal(sel, ref_sel[0])
    assert not sel[:, 2:].any()


@pytest.mark.parametrize("topk", [1, 3, 7])
def test_all_scores_tied_takes_lowest_indices(topk):
    """Every key block identical -> every score of a row ties -> the first
    top-k block indices (stable descending order)."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((4, 8, 16), H=2)
    k = k[:, :, :64].repeat(1, 1, 8, 1).contiguous()
    res = P.block_sparse_attention(q, k, v, P.SparseSettings(block=64, topk=topk))
    sel = res.selected.cpu().numpy()
    want = np.zeros(8, dtype=bool)
    want[:topk] = True
    assert (sel == want).all()


def test_batch_two_matches_single():
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((2, 8, 16), H=2)
    q2, k2, v2, x2, _, _, _ = _small((2, 8, 16), H=2, seed=5)
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=2))
    qb, kb, vb, xb = (torch.cat(p, 0) for p in ((q, q2), (k, k2), (v, v2), (x, x2)))
    both = P.forward(qb, kb, vb, xb, grid, params, st, pe)
    one = P.forward(q2, k2, v2, x2, grid, params, st, pe)
    assert torch.equal(both[1], one[0])


def test_spec_known_answers():
    """SPEC.md:466, 484, 493 on the device."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((2, 8, 16), H=2)
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=2))
    p0 = P.MechanismParams(**{**params.__dict__, "w_a": torch.zeros_like(params.w_a),
                              "w_b": torch.zeros_like(params.w_b)})
    tr = P.forward(q, k, v, x, grid, p0, st, pe, trace=True)
    assert torch.all(tr.o_lowrank == 0.5)
    p1 = P.MechanismParams(**{**params.__dict__, "w_g": torch.zeros_like(params.w_g), "b_g": 0.0})
    tr = P.forward(q, k, v, x, grid, p1, st, pe, trace=True)
    assert torch.allclose(tr.g, torch.full_like(tr.g, 0.5))
    p2 = P.MechanismParams(**{**params.__dict__, "b_g": -50.0})
    tr = P.forward(q, k, v, x, grid, p2, st, pe, trace=True)
    o = tr.o_sparse[0].double()
    ysp = o / torch.sqrt(o.pow(2).mean(-1, keepdim=True) + 1e-6)
    want = ysp.permute(1, 0, 2).reshape(grid.size, -1)
    G.assert_close(tr.output[0].double().cpu().numpy(), want.cpu().numpy(), "bf16", "gate-off")


def test_zero_values_zero_sparse_branch():
    """Zero V -> zero sparse output -> RMSNorm(0) = 0."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((2, 8, 16), H=1)
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=2), use_pe=False)
    p2 = P.MechanismParams(**{**params.__dict__, "b_g": -50.0})
    tr = P.forward(q, k, v * 0, x, grid, p2, st, None, trace=True)
    assert torch.all(tr.o_sparse == 0)
    assert float(tr.output.float().abs().max()) < 1e-12


def test_bad_inputs_raise_value_error():
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((2, 8, 16), H=1)
    with pytest.raises(ValueError):
        P.block_sparse_attention(q, k[:, :, :-1], v, P.SparseSettings(64, topk=1))
    with pytest.raises(ValueError):
        P.block_sparse_attention(q, k, v, P.SparseSettings((1, 3, 16)), grid=grid)  # 3 does not divide 8
    with pytest.raises(ValueError):
        P.block_sparse_attention(q.half(), k.half(), v.half(), P.SparseSettings(64, topk=1))
    with pytest.raises(ValueError):
        P.forward(q, k, v, x[:, :, :-8], grid, params, P.ForwardSettings(P.SparseSettings(64, topk=1)), pe)


def _skew_blocks(q, k, block, seed=1, strength=4.0, spread=2.0):
    """Give the block scores structure, as real attention has: a shared
    direction u, key block b shifted by strength*c_b*u (c_b ~ N(0, 1)) and
    query block j by strength*a_j*u with a_j = exp(U(-spread, spread)).  Rows
    with a large a_j get a peaked block softmax (few blocks under `keep`),
    rows with a small one a flat softmax (many blocks)."""
    B, H, L, d = q.shape
    nb = -(-L // block)
    g = torch.Generator(device="cpu").manual_seed(seed)
    u = torch.randn(d, generator=g, dtype=torch.float64)
    u = u / u.norm()
    c = torch.randn((B, H, nb), generator=g, dtype=torch.float64)
    a = torch.exp((torch.rand((B, H, nb), generator=g, dtype=torch.float64) * 2 - 1) * spread)

    def shift(t, w):
        w = w.repeat_interleave(block, dim=-1)[..., :L].to(t.device)
        return (t.double() + strength * w[..., None] * u.to(t.device)).to(t.dtype)

    return shift(q, a), shift(k, c)


@pytest.mark.parametrize("block", [64, 128])
def test_keep_schedule_bit_identical(block):
    """The longest-first unit schedule (schedule_units_kernel) only changes
    which CTA runs a (head, query block): the output is bit-identical to the
    unscheduled launch, every row is written, and the counts really vary."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((8, 16, 64), H=4)
    q, k = _skew_blocks(q, k, block)
    st = P.ForwardSettings(P.SparseSettings(block=block, keep=0.6))
    prep = P.prepare(q, k, v, x, grid, params, st, pe)
    cnt = prep.sel.cnt.cpu()
    assert cnt.max() > 2 * cnt.min(), "skewed inputs should give uneven block counts"
    B, H, L, d = q.shape
    outs = []
    for sched in (1, 0):
        with P._lib.option("schedule", sched):
            out = torch.full((B, L, H, d), float("nan"), dtype=q.dtype, device=q.device)
            P.attend(prep, params, st, out=out)
            torch.cuda.synchronize()
        outs.append(out)
    assert torch.isfinite(outs[0].float()).all()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("scale", [1.0, 4.0, 12.0])
@pytest.mark.parametrize("block", [64, 128])
def test_fixed_reference_extreme_logits(scale, block):
    """The fixed-reference K2 (sparse_attn_fixed_kernel) picks one exponent
    reference per row and unit; rows whose scores span too many binary
    orders for it are recomputed by the running-max kernel.  Q and K scaled
    by `scale` give score standard deviations of scale^2 nats: at 12 every
    unit overflows the fixed reference, so the output must equal the
    running-max kernel's bit for bit; at every scale the sparse branch
    matches the float64 oracle."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((4, 16, 64), H=2)
    q = (q.float() * scale).to(q.dtype)
    k = (k.float() * scale).to(k.dtype)
    st = P.ForwardSettings(P.SparseSettings(block=block, topk=6))
    prep = P.prepare(q, k, v, x, grid, params, st, pe)
    outs = {}
    for mode in ("fixed", "online"):
        with P._lib.option("k2_online", int(mode == "online")):
            out, o_sp = P.attend(prep, params, st, want_o_sparse=True)
            torch.cuda.synchronize()
        outs[mode] = (out.clone(), o_sp.clone())
    ref_out, ref_sel = _oracle_sparse(q, k, v, block, topk=6)
    got = outs["fixed"][1][0].cpu().numpy()
    for h in range(q.shape[1]):
        G.assert_close(got[h], ref_out[h], "bf16", f"o_sparse head {h} at scale {scale}")
    assert torch.isfinite(outs["fixed"][0].float()).all()
    if scale >= 12.0:
        assert torch.equal(outs["fixed"][0], outs["online"][0])
        assert torch.equal(outs["fixed"][1], outs["online"][1])


def test_fixed_reference_partial_fallback():
    """One head with extreme logits (every one of its units falls back to the
    running-max kernel) next to normal heads (none does), in the same launch,
    with and without the unit schedule: the fallen-back head equals the
    running-max kernel bit for bit, and every head matches the oracle."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((4, 16, 64), H=3)
    q, k = q.clone(), k.clone()
    q[:, 1] = (q[:, 1].float() * 12.0).to(q.dtype)
    k[:, 1] = (k[:, 1].float() * 12.0).to(k.dtype)
    st = P.ForwardSettings(P.SparseSettings(block=128, topk=5))
    prep = P.prepare(q, k, v, x, grid, params, st, pe)
    ref_out, _ = _oracle_sparse(q, k, v, 128, topk=5)
    res = {}
    for mode, sched in (("fixed", "0"), ("fixed", "1"), ("online", "0")):
        with P._lib.option("k2_online", int(mode == "online")), P._lib.option("schedule", int(sched)):
            _, o_sp = P.attend(prep, params, st, want_o_sparse=True)
            torch.cuda.synchronize()
        res[(mode, sched)] = o_sp.clone()
    for key in (("fixed", "0"), ("fixed", "1")):
        got = res[key][0].cpu().numpy()
        for h in range(3):
            G.assert_close(got[h], ref_out[h], "bf16", f"o_sparse head {h} {key}")
        assert torch.equal(res[key][0, 1], res[("online", "0")][0, 1])
    assert torch.equal(res[("fixed", "0")], res[("fixed", "1")])


def _crafted_scores_inputs(b_vals, a_vals, block=32, d=64):
    """f32 Q/K whose block means are a_i * e0 and b_j * e0 exactly (constant
    rows), so every block score a_i * b_j / sqrt(d) is one exact product on
    both sides and the selection rule itself is what is compared."""
    nb = len(b_vals)
    L = nb * block
    q = torch.zeros((1, 1, L, d), dtype=torch.float32)
    k = torch.zeros((1, 1, L, d), dtype=torch.float32)
    for i in range(nb):
        q[0, 0, i * block:(i + 1) * block, 0] = float(a_vals[i])
        k[0, 0, i * block:(i + 1) * block, 0] = float(b_vals[i])
    return q.cuda(), k.cuda(), torch.zeros_like(q).cuda()


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("rule", [dict(topk=7), dict(topk=1), dict(keep=0.5), dict(keep=0.999)])
@pytest.mark.parametrize("pattern", ["wide", "powers", "dups", "signed_zero"])
def test_selection_extreme_and_tied_scores(pattern, rule, d):
    """Selection on block scores with spreads far beyond the float64 exp
    range (the reference's block probabilities underflow to 0 and tie, so
    those blocks go by index), exact duplicates, powers of two and signed
    zeros: masks bit-exact against the oracle (mechanism.py:309-320).  With
    d = 128 top-k takes the screening path (test_gpu_screen.py)."""
    import paper_2605_20659_b200 as P

    rng = np.random.default_rng(5)
    nb = 40
    if pattern == "wide":
        b = rng.standard_normal(nb) * 3000.0
    elif pattern == "powers":
        b = np.array([(-1) ** j * 2.0 ** (j - 10) for j in range(nb)])
    elif pattern == "dups":
        b = rng.choice([-1.0, 0.0, 1.0, 2.0], size=nb)
    else:
        b = np.where(np.arange(nb) % 2 == 0, -0.0, 0.0)
        b[[5, 17, 30]] = [1.0, 1.0, 0.5]
    a = rng.standard_normal(nb) * 4.0
    a[[3, 11]] = 0.0
    q, k, v = _crafted_scores_inputs(b, a, d=d)
    sp = P.SparseSettings(block=32, **rule)
    sel = P.select_blocks(q, k, sp)
    members = R.flat_block_members(q.shape[2], 32)
    scores = R.block_scores(q[0, 0].double().cpu().numpy(), k[0, 0].double().cpu().numpy(), members)
    ref_sel, _ = R.select_blocks(scores, **rule)
    np.testing.assert_array_equal(sel.mask[0, 0].cpu().numpy(), ref_sel, err_msg=f"{pattern} {rule}")


@pytest.mark.parametrize("impl", ["tcgen05", "simt"])
@pytest.mark.parametrize("name", ["bf16_d128_b128", "bf16_d128_keep", "bf16_3d_tile64", "ragged_topk_bf16"])
def test_float32_output(name, impl):
    """out_dtype=float32 stores the fused epilogue's result before the bf16
    rounding: rounding it to bf16 gives the bf16 output bit for bit, and it
    meets the north-star bar against the reference on its own."""
    import paper_2605_20659_b200 as P

    g = golden_io.load(name)
    q, k, v, x, params, pe, st, grid, lin = G.golden_to_device(g)
    o16 = P.forward(q, k, v, x, grid, params, st, pe, impl=impl)
    o32 = P.forward(q, k, v, x, grid, params, st, pe, impl=impl, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert o32.dtype == torch.float32 and o32.shape == o16.shape
    assert torch.equal(o32.to(torch.bfloat16), o16)
    G.assert_close(o32[0].cpu().numpy(), g["ref_output"], "bf16", f"{name} float32 output")


def test_golden_linear_pe_in_kernel():
    """The reference's linear compensator (bf16_d128_linear, mechanism.py:350-362
    on x_hat = x + alpha PE) through the PE-injecting tensor-core path: the
    caller passes x W and the backbone weights, the kernels add (alpha PE) W."""
    import paper_2605_20659_b200 as P

    g = golden_io.load("bf16_d128_linear")
    q, k, v, x, params, pe, st, grid, _ = G.golden_to_device(g)
    W = [torch.from_numpy(np.ascontiguousarray(g[n])).float().cuda() for n in
         ("ref_w_lin_q", "ref_w_lin_k", "ref_w_lin_v")]
    lin = tuple(torch.einsum("bld,hde->bhle", x.double(), w.double()).to(torch.bfloat16).contiguous() for w in W)
    tr = P.forward(q, k, v, x, grid, params, st, pe, lin_proj=lin, lin_weights=W, trace=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(tr.selected[0].cpu().numpy(), g["ref_selected"])
    G.assert_close(tr.o_lowrank[0].cpu().numpy(), g["ref_o_lowrank"], "bf16", "linear pe o_lowrank")
    G.assert_close(tr.g[0].cpu().numpy(), g["ref_g"], "bf16", "linear pe gate")
    G.assert_close_bf16_store(tr.output[0].float().cpu().numpy(), g["ref_output"], "linear pe output")


@pytest.mark.parametrize("block,rule", [(64, dict(topk=5)), (128, dict(topk=3)), (64, dict(keep=0.6))])
def test_query_block_range(block, rule):
    """q_blocks=(qb0, qb1): only those query blocks run (the share of a head a
    sequence-parallel rank computes); their rows equal the full call's bit for
    bit, every other row keeps the caller's contents."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = _small((3, 16, 40), H=3)  # L = 1920, ragged at block 128
    st = P.ForwardSettings(P.SparseSettings(block=block, **rule))
    full = P.forward(q, k, v, x, grid, params, st, pe)
    B, H, L, d = q.shape
    nb = -(-L // block)
    for qb0, qb1 in ((0, 1), (3, nb), (nb // 3, 2 * nb // 3)):
        out = torch.full((B, L, H * d), 7.0, dtype=q.dtype, device=q.device)
        got = P.forward(q, k, v, x, grid, params, st, pe, q_blocks=(qb0, qb1), out=out)
        torch.cuda.synchronize()
        r0, r1 = qb0 * block, min(L, qb1 * block)
        assert torch.equal(got[:, r0:r1], full[:, r0:r1])
        assert bool((got[:, :r0] == 7.0).all()) and bool((got[:, r1:] == 7.0).all())
    with pytest.raises(ValueError):
        P.forward(q, k, v, x, grid, params, st, pe, q_blocks=(2, 2))
