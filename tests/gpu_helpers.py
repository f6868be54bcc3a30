"""Shared helpers for the GPU parity tests: golden fixtures -> device tensors,
seeded full-size inputs, tolerance metrics."""

from __future__ import annotations

import math
import os

import numpy as np
import torch

import restated as R

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# BASELINE north star: masks bit-exact; bf16 outputs within max-abs 2e-2 and
# mean-relative 1e-2 of the float64 reference.  float32 runs get 1e-4.
TOL = {"bf16": dict(max_abs=2e-2, mean_rel=1e-2), "f32": dict(max_abs=1e-4, mean_rel=1e-5)}


def mean_rel(a: np.ndarray, b: np.ndarray) -> float:
    """mean |a - b| / mean |b|."""
    return float(np.mean(np.abs(a - b)) / max(np.mean(np.abs(b)), 1e-30))


def assert_close(got, want, dtype: str, what: str = "", scale: float = 1.0):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    tol = TOL[dtype]
    err = float(np.max(np.abs(got - want))) if got.size else 0.0
    mr = mean_rel(got, want)
    assert err <= tol["max_abs"] * scale, f"{what}: max-abs {err:.3e} > {tol['max_abs'] * scale:.1e}"
    assert mr <= tol["mean_rel"] * scale, f"{what}: mean-rel {mr:.3e} > {tol['mean_rel'] * scale:.1e}"
    return err, mr


def bf16_half_ulp(x) -> np.ndarray:
    """Half a bf16 ulp at |x| (8 significant bits): the rounding error of
    storing x in bf16."""
    a = np.abs(np.asarray(x, np.float64))
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -126)))
    return 2.0 ** (e - 8)


def assert_close_bf16_store(got, want, what: str = ""):
    """A bf16-stored output against the float64 reference: the north-star
    bar (max-abs 2e-2, mean-rel 1e-2) on top of the rounding of the stored
    value itself (half a bf16 ulp of the reference value: 0.0078 at |x| in
    [2, 4), 0.0156 in [4, 8)).  The op's float32 output (out_dtype) is held to
    the bar alone."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    tol = TOL["bf16"]
    excess = np.abs(got - want) - bf16_half_ulp(want)
    err = float(np.max(excess)) if got.size else 0.0
    mr = mean_rel(got, want)
    assert err <= tol["max_abs"], f"{what}: max-abs beyond the bf16 store {err:.3e} > {tol['max_abs']:.1e}"
    assert mr <= tol["mean_rel"], f"{what}: mean-rel {mr:.3e} > {tol['mean_rel']:.1e}"
    return float(np.max(np.abs(got - want))) if got.size else 0.0, mr


def torch_dtype(name: str):
    return torch.bfloat16 if name == "bf16" else torch.float32


def golden_to_device(g, dev="cuda"):
    """Golden fixture -> (q, k, v, x, params, pe, settings, grid, lin_proj)."""
    import paper_2605_20659_b200 as P

    dt = torch_dtype(g["dtype"])
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    q, k, v = (t(g[n]).to(dt)[None].contiguous() for n in ("q", "k", "v"))
    x = t(g["x"]).to(dt)[None].contiguous()
    params = P.MechanismParams.from_arrays(device=dev, **{n: g[n] for n in (
        "w_a", "w_b", "alpha", "w_g", "b_g", "rms_sparse", "rms_lowrank")})
    pe = P.PETables(t(g["pe_t"]).float(), t(g["pe_x"]).float(), t(g["pe_y"]).float())
    grid = P.GridShape(*g["grid"])
    if g["source"] == "reference":
        sp = P.SparseSettings(block=g["block3"], keep=g["keep"])
    else:
        sp = P.SparseSettings(block=g["block3"][2], topk=g["topk"])
    st = P.ForwardSettings(sp, compensator=g["compensator"], use_pe=g["use_pe"])
    lin = None
    if g["compensator"] == "linear":
        pe_dense = R.pe_from_axis_tables(g["grid"], g["pe_t"], g["pe_x"], g["pe_y"])
        x_hat = np.asarray(g["x"], np.float64) + np.asarray(g["alpha"], np.float64)[None] * pe_dense
        lin = tuple(t(np.einsum("ld,hde->hle", x_hat, np.asarray(g[w], np.float64))).to(dt)[None].contiguous()
                    for w in ("ref_w_lin_q", "ref_w_lin_k", "ref_w_lin_v"))
    return q, k, v, x, params, pe, st, grid, lin


def make_full_inputs(L_grid, H, d, split, r, seed=0, dtype=torch.bfloat16, dev="cuda"):
    """Seeded BASELINE-shaped inputs generated on the device: Q, K, V ~ N(0,1)
    rotated in float64 by the 3D RoPE and cast; X ~ N(0,1); per-axis PE
    ~ N(0, 0.02); W_A, W_B ~ N(0, 1/sqrt(d)); alpha 0.1; w_g ~ N(0, 0.05);
    b_g = -2; RMS scales 1."""
    import paper_2605_20659_b200 as P

    grid = P.GridShape(*L_grid)
    cfg = P.RopeConfig(*split)
    L, D = grid.size, H * d
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    qkv = []
    for which in range(3):
        t = torch.randn((1, H, L, d), generator=gen, device=dev, dtype=torch.float32)
        if which < 2:
            t = torch.cat([P.rotate_rows(t[:, h:h + 1], grid, cfg).to(dtype) for h in range(H)], dim=1)
        else:
            t = t.to(dtype)
        qkv.append(t.contiguous())
    x = torch.randn((1, L, D), generator=gen, device=dev, dtype=torch.float32).to(dtype).contiguous()
    pe = P.PETables(*(torch.randn((n, D), generator=gen, device=dev) * 0.02 for n in L_grid))
    params = P.MechanismParams(
        w_a=torch.randn((H, d, r), generator=gen, device=dev) / math.sqrt(d),
        w_b=torch.randn((H, r, d), generator=gen, device=dev) / math.sqrt(d),
        alpha=torch.full((D,), 0.1, device=dev), w_g=torch.randn((D,), generator=gen, device=dev) * 0.05,
        b_g=-2.0, rms_sparse=torch.ones(d, device=dev), rms_lowrank=torch.ones(d, device=dev))
    return (*qkv, x, params, pe, grid)


def oracle_rows(qh, kh, vh, members, selected_oracle, qblocks):
    out, _ = R.attend_selected(qh, kh, vh, members, selected_oracle, qblocks=qblocks)
    return out


def oracle_fused_rows(rows, o_sparse_rows, x, pe_tabs, params_np, grid, head, d, eps=1e-6):
    """Oracle output of head `head` at token rows `rows` (lowrank compensator)."""
    c = R.grid_coords(*grid)[rows]
    D = x.shape[1]
    pe = (pe_tabs[0][c[:, 0]] + pe_tabs[1][c[:, 1]] + pe_tabs[2][c[:, 2]]).astype(np.float64)
    x_hat = x[rows].astype(np.float64) + params_np["alpha"][None] * pe
    g = R.sigmoid(x_hat @ params_np["w_g"] + params_np["b_g"])
    o_lr = R.lowrank_compensator(x_hat, params_np["w_a"], params_np["w_b"], head)
    y = R.rms_norm(o_sparse_rows, params_np["rms_sparse"], eps) + g[:, None] * R.rms_norm(o_lr, params_np["rms_lowrank"], eps)
    return y, g, o_lr
