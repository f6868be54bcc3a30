"""Pin the CPU oracle (oracle/restated.py) before trusting it.

1. Against every committed golden fixture (produced by the unmodified
   reference functions, oracle/make_golden.py) -- always runs.
2. Against the live reference package when /root/reference is present
   (the build container); skipped elsewhere.
3. The reference's own known answers for the selection rule
   (test_decomposition.py:144-162) and the SPEC mechanism examples
   (SPEC.md:433-531).
"""

import math
import os
import sys

import numpy as np
import pytest

import golden_io
import restated as R

REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF_SRC)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="reference package not present")


def oracle_on_golden(g):
    q, k, v = (np.asarray(g[n], np.float64) for n in ("q", "k", "v"))
    H, L, d = q.shape
    if g["source"] == "reference":
        members = R.tile_block_members(g["grid"], g["block3"])
        sel_kw = dict(keep=g["keep"])
    else:
        members = R.flat_block_members(L, g["block3"][2])
        sel_kw = dict(topk=g["topk"])
    outs, sels, spars = [], [], []
    for h in range(H):
        o, s, sp, _, _ = R.block_sparse_attention(q[h], k[h], v[h], members, **sel_kw)
        outs.append(o)
        sels.append(s)
        spars.append(sp)
    pe = R.pe_from_axis_tables(g["grid"], g["pe_t"], g["pe_x"], g["pe_y"])
    params = {n: g[n] for n in ("w_a", "w_b", "alpha", "w_g", "b_g", "rms_sparse", "rms_lowrank")}
    backbone = None
    if g["compensator"] == "linear":
        backbone = dict(w_q=g["ref_w_lin_q"], w_k=g["ref_w_lin_k"], w_v=g["ref_w_lin_v"])
    fused = R.fused_forward(g["x"], outs, pe, params, compensator=g["compensator"],
                            use_pe=g["use_pe"], backbone=backbone)
    return np.stack(sels), np.array(spars), np.stack(outs), fused


@pytest.mark.parametrize("name", golden_io.names())
def test_oracle_matches_golden(name):
    g = golden_io.load(name)
    sel, spars, o_sp, fused = oracle_on_golden(g)
    np.testing.assert_array_equal(sel, g["ref_selected"])
    np.testing.assert_allclose(spars, g["ref_sparsity"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(o_sp, g["ref_o_sparse"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(fused["o_lowrank"], g["ref_o_lowrank"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(fused["g"], g["ref_g"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(fused["output"], g["ref_output"], rtol=0, atol=1e-11)


def test_golden_inventory():
    """Every fixture the CUDA parity tests rely on exists."""
    want = {"cfg0_lowrank", "cfg0_linear", "keep3d_sinpe", "bf16_d128_keep", "bf16_d128_b128",
            "ragged_topk_bf16", "ragged_topk_f32"}
    assert want <= set(golden_io.names())


# ---------------------------------------------------------------------------
# selection-rule known answers (reference tests test_decomposition.py:144-162)


def test_count_for_mass_known_answers():
    assert R.count_for_mass(np.array([1.0, 0.0, 0.0, 0.0]), 0.9) == 1
    assert R.count_for_mass(np.full(10, 0.1), 0.9) == 9
    assert R.count_for_mass(np.array([0.4, 0.4, 0.2]), 0.4) == 1
    # never reached -> everything
    assert R.count_for_mass(np.array([0.1, 0.1]), 0.5) == 2


def test_select_tie_goes_to_lower_index():
    # identical key blocks -> identical scores -> stable order keeps the lower index
    scores = np.array([[0.3, 0.3, 0.1], [0.2, 0.5, 0.5], [0.0, 0.0, 0.0]])
    sel, cnt = R.select_blocks(scores, topk=1)
    np.testing.assert_array_equal(sel, [[1, 0, 0], [0, 1, 0], [1, 0, 0]])
    sel2, cnt2 = R.select_blocks(scores, topk=2)
    np.testing.assert_array_equal(sel2, [[1, 1, 0], [0, 1, 1], [1, 1, 0]])


def test_topk_for_sparsity():
    assert R.topk_for_sparsity(512, 0.9) == 51
    assert R.topk_for_sparsity(929, 0.9) == 93
    assert R.topk_for_sparsity(256, 0.8) == 51
    assert R.topk_for_sparsity(512, 0.95) == 26
    assert R.topk_for_sparsity(4, 0.75) == 1


def test_flat_blocks_equal_rowspanning_tiles():
    """Extension (i) equals the reference's 3D tiles whenever a tile spans
    whole grid rows (config 0: tile (1,8,8) == flat 64)."""
    for grid, tile in (((4, 8, 8), (1, 8, 8)), ((2, 8, 16), (1, 4, 16)), ((3, 8, 16), (1, 8, 16))):
        L = grid[0] * grid[1] * grid[2]
        a = R.tile_block_members(grid, tile)
        b = R.flat_block_members(L, tile[0] * tile[1] * tile[2])
        assert len(a) == len(b)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


def test_ragged_flat_blocks():
    m = R.flat_block_members(130, 64)
    assert [len(x) for x in m] == [64, 64, 2]


# ---------------------------------------------------------------------------
# SPEC mechanism examples on the oracle


def _rand_case(seed=0, H=2, L=64, d=8, r=4, grid=(1, 8, 8)):
    rng = np.random.default_rng(seed)
    D = H * d
    x = rng.standard_normal((L, D))
    sp = [rng.standard_normal((L, d)) for _ in range(H)]
    params = dict(w_a=rng.standard_normal((H, d, r)), w_b=rng.standard_normal((H, r, d)),
                  alpha=np.full(D, 0.1), w_g=rng.standard_normal(D) * 0.1, b_g=-2.0,
                  rms_sparse=np.ones(d), rms_lowrank=np.ones(d))
    pe = R.pe_from_axis_tables(grid, *(rng.standard_normal((n, D)) * 0.02 for n in grid))
    return x, sp, params, pe


def test_spec_zero_compensator_is_half():
    x, sp, params, pe = _rand_case()
    params["w_a"][:] = 0
    params["w_b"][:] = 0
    f = R.fused_forward(x, sp, pe, params)
    np.testing.assert_array_equal(f["o_lowrank"], 0.5)


def test_spec_zero_gate_is_half():
    x, sp, params, pe = _rand_case()
    params["w_g"][:] = 0
    params["b_g"] = 0.0
    f = R.fused_forward(x, sp, pe, params)
    np.testing.assert_array_equal(f["g"], 0.5)


def test_spec_gate_off_gives_normalized_sparse():
    x, sp, params, pe = _rand_case()
    params["b_g"] = -50.0
    f = R.fused_forward(x, sp, pe, params)
    ysp = np.concatenate([R.rms_norm(s, params["rms_sparse"]) for s in sp], axis=1)
    np.testing.assert_allclose(f["output"], ysp, rtol=0, atol=1e-9)


def test_spec_rms_zero_row():
    np.testing.assert_array_equal(R.rms_norm(np.zeros((3, 4)), np.ones(4)), 0.0)


def test_spec_full_coverage_is_full_attention():
    rng = np.random.default_rng(3)
    L, d = 40, 8
    q, k, v = (rng.standard_normal((L, d)) for _ in range(3))
    members = R.flat_block_members(L, L)           # one block covering everything
    out, sel, sp, _, _ = R.block_sparse_attention(q, k, v, members, keep=1.0)
    s = q @ k.T / math.sqrt(d)
    a = np.exp(s - s.max(1, keepdims=True))
    a /= a.sum(1, keepdims=True)
    np.testing.assert_allclose(out, a @ v, rtol=0, atol=1e-12)
    assert sp == 0.0


def test_spec_linear_single_token_returns_v():
    rng = np.random.default_rng(4)
    q, k, v = (rng.standard_normal((1, 6)) for _ in range(3))
    s, z = R.linear_state(k, v)
    np.testing.assert_allclose(R.linear_apply(q, s, z), v, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------------------
# live reference cross-checks (build container only)


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import ropeslr.decomposition as Dm
    import ropeslr.mechanism as M
    import ropeslr.rope3d as Rp
    return M, Rp, Dm


@needs_ref
def test_live_rotate_rows():
    M, Rp, _ = _ref()
    rng = np.random.default_rng(0)
    for grid, split in (((4, 8, 8), (16, 24, 24)), ((3, 5, 7), (44, 42, 42)), ((2, 3, 4), (16, 56, 56))):
        m = rng.standard_normal((grid[0] * grid[1] * grid[2], sum(split)))
        want = Rp.rotate_rows(m, Rp.GridShape(*grid), Rp.RopeConfig(*split))
        np.testing.assert_array_equal(R.rotate_rows(m, grid, split), want)


@needs_ref
def test_live_sinusoidal_pe_decomposition():
    M, Rp, _ = _ref()
    for grid, split, D in (((4, 8, 8), (16, 24, 24), 128), ((2, 3, 5), (4, 2, 2), 16)):
        want = M.build_pe3d(Rp.GridShape(*grid), D, Rp.RopeConfig(*split))
        got = R.pe_from_axis_tables(grid, *R.sinusoidal_axis_tables(grid, D, split))
        np.testing.assert_array_equal(got, want)


@needs_ref
def test_live_count_for_mass():
    _, _, Dm = _ref()
    rng = np.random.default_rng(1)
    for _ in range(200):
        row = np.sort(rng.dirichlet(np.ones(rng.integers(1, 30))))[::-1]
        t = float(rng.uniform(1e-6, 1.0))
        assert R.count_for_mass(row, t) == Dm.count_for_mass(row, t)


@needs_ref
@pytest.mark.parametrize("grid,block,keep", [((2, 4, 6), (1, 2, 3), 0.5), ((4, 4, 4), (2, 2, 2), 0.5),
                                             ((3, 4, 8), (1, 4, 8), 0.9), ((2, 2, 8), (2, 2, 2), 1.0)])
def test_live_block_sparse_attention(grid, block, keep):
    """Restated sparse branch == reference block_sparse_attention (rotation
    in the reference, restated consumes the rotated rows)."""
    M, Rp, _ = _ref()
    H, d = 2, 8
    rng = np.random.default_rng(5)
    L = grid[0] * grid[1] * grid[2]
    D = H * d
    x = rng.standard_normal((L, D))
    bb = M.random_backbone(H, d, 9)
    cfg = Rp.RopeConfig(4, 2, 2)
    gs = Rp.GridShape(*grid)
    members = R.tile_block_members(grid, block)
    for h in range(H):
        want = M.block_sparse_attention(x, gs, cfg, bb, h, M.SparseSettings(block, keep))
        rq = Rp.rotate_rows(x @ bb.w_q[h], gs, cfg)
        rk = Rp.rotate_rows(x @ bb.w_k[h], gs, cfg)
        out, sel, sp, _, _ = R.block_sparse_attention(rq, rk, x @ bb.w_v[h], members, keep=keep)
        np.testing.assert_array_equal(sel, want.selected)
        np.testing.assert_allclose(out, want.output, rtol=0, atol=1e-13)
        assert sp == pytest.approx(want.sparsity, abs=1e-15)


@needs_ref
@pytest.mark.parametrize("compensator", ["lowrank", "linear"])
def test_live_forward(compensator):
    """Restated fusion == reference mechanism.forward end to end (sinusoidal PE)."""
    M, Rp, _ = _ref()
    grid, split, H, d, r = (2, 4, 4), (4, 2, 2), 2, 8, 3
    gs, cfg = Rp.GridShape(*grid), Rp.RopeConfig(*split)
    L, D = gs.size, H * d
    rng = np.random.default_rng(6)
    x = rng.standard_normal((L, D))
    bb = M.random_backbone(H, d, 2)
    params = M.init_params(H, d, r, 3)
    params.w_g = rng.standard_normal(D) * 0.1
    st = M.ForwardSettings(M.SparseSettings((1, 2, 2), 0.7), compensator=compensator)
    tr = M.forward(x, gs, cfg, bb, params, st)
    members = R.tile_block_members(grid, (1, 2, 2))
    outs = []
    for h in range(H):
        rq = Rp.rotate_rows(x @ bb.w_q[h], gs, cfg)
        rk = Rp.rotate_rows(x @ bb.w_k[h], gs, cfg)
        outs.append(R.block_sparse_attention(rq, rk, x @ bb.w_v[h], members, keep=0.7)[0])
    pe = R.pe_from_axis_tables(grid, *R.sinusoidal_axis_tables(grid, D, split))
    pd = dict(w_a=params.w_a, w_b=params.w_b, alpha=params.alpha, w_g=params.w_g, b_g=params.b_g,
              rms_sparse=params.rms_sparse, rms_lowrank=params.rms_lowrank)
    f = R.fused_forward(x, outs, pe, pd, compensator=compensator,
                        backbone=dict(w_q=bb.w_q, w_k=bb.w_k, w_v=bb.w_v))
    np.testing.assert_allclose(f["output"], tr.output, rtol=0, atol=1e-12)
    np.testing.assert_allclose(f["g"], tr.g, rtol=0, atol=1e-14)
    np.testing.assert_allclose(f["o_lowrank"], tr.o_lowrank, rtol=0, atol=1e-12)
