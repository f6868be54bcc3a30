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
