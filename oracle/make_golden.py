"""Generate golden vectors from the UNMODIFIED reference functions.

TEST INFRASTRUCTURE ONLY.  Run in the build container (where the read-only
reference lives at /root/reference):

    python oracle/make_golden.py [case ...]  # writes tests/golden/*.npz (all cases, or the named ones)

Each fixture stores the exact (post-RoPE, post-cast) inputs the GPU op
consumes and the reference's outputs on those same values:

* the sparse branch comes from ``mechanism.block_sparse_attention``
  (mechanism.py:290-328) driven through a 0/1 "selector backbone" whose
  projections reproduce the stored Q/K/V exactly, with ``rotate_rows``
  replaced by the identity because the stored Q/K are already rotated
  (the probe showed re-rotating after a cast flips masks);
* the fusion comes from ``mechanism._fused_forward`` (mechanism.py:426-453)
  with the real X, the PE table and the parameters.

Fixtures whose blocking the reference cannot express (ragged flat blocks,
fixed top-k) are produced by ``oracle/restated.py`` and marked
``source = "restated"``; that restatement is itself pinned against the
reference fixtures in tests/test_oracle.py.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF_SRC = "/root/reference/pkg/src"
OUT_DIR = os.path.join(REPO, "tests", "golden")

sys.path.insert(0, HERE)
import restated as R  # noqa: E402


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 (exact)."""
    a32 = np.ascontiguousarray(a, dtype=np.float32)
    u = a32.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def cast(a, dtype: str) -> np.ndarray:
    if dtype == "f32":
        return np.asarray(a, np.float32)
    if dtype == "bf16":
        return bf16_round(a)
    raise ValueError(dtype)


def make_inputs(seed, H, d, grid, split, r, dtype, pe_kind="axis", d_model=None):
    """Seeded inputs per BASELINE config 0: Q,K,V ~ N(0,1)
    rotated in fp64 then cast; X ~ N(0,1); per-axis PE ~ N(0,0.02);
    W_A, W_B ~ N(0, 1/sqrt(d)); alpha = 0.1; w_g ~ N(0, 0.05); b_g = -2;
    RMS scales 1.  Parameters are float32 (the op's parameter dtype)."""
    rng = np.random.default_rng(seed)
    L = grid[0] * grid[1] * grid[2]
    D = H * d if d_model is None else d_model
    q = rng.standard_normal((H, L, d))
    k = rng.standard_normal((H, L, d))
    v = rng.standard_normal((H, L, d))
    rq = np.stack([R.rotate_rows(q[h], grid, split) for h in range(H)])
    rk = np.stack([R.rotate_rows(k[h], grid, split) for h in range(H)])
    x = rng.standard_normal((L, D))
    if pe_kind == "axis":
        pe_t = rng.standard_normal((grid[0], D)) * 0.02
        pe_x = rng.standard_normal((grid[1], D)) * 0.02
        pe_y = rng.standard_normal((grid[2], D)) * 0.02
    else:  # reference sinusoidal table, decomposed per axis
        pe_t, pe_x, pe_y = R.sinusoidal_axis_tables(grid, D, split)
    w_a = rng.standard_normal((H, d, r)) / math.sqrt(d)
    w_b = rng.standard_normal((H, r, d)) / math.sqrt(d)
    w_g = rng.standard_normal(D) * 0.05
    f32 = lambda a: np.asarray(a, np.float32)  # noqa: E731
    return dict(
        q=cast(rq, dtype), k=cast(rk, dtype), v=cast(v, dtype), x=cast(x, dtype),
        pe_t=f32(pe_t), pe_x=f32(pe_x), pe_y=f32(pe_y),
        w_a=f32(w_a), w_b=f32(w_b), alpha=f32(np.full(D, 0.1)), w_g=f32(w_g),
        b_g=np.float32(-2.0), rms_sparse=f32(np.ones(d)), rms_lowrank=f32(np.ones(d)),
        grid=np.array(grid), split=np.array(split), dtype=np.array(dtype))


def _import_reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import ropeslr.mechanism as M  # noqa: E402
    from ropeslr.rope3d import GridShape, RopeConfig  # noqa: E402
    return M, GridShape, RopeConfig


def run_reference(inp, block3, keep, compensator="lowrank", use_pe=True, backbone_seed=7):
    """Reference outputs on the stored (already rotated) inputs."""
    M, GridShape, RopeConfig = _import_reference()
    q, k, v = (np.asarray(inp[n], np.float64) for n in ("q", "k", "v"))
    H, L, d = q.shape
    D = inp["x"].shape[1]
    grid = GridShape(*[int(a) for a in inp["grid"]])
    cfg = RopeConfig(*[int(a) for a in inp["split"]])
    # selector backbone: x_sel = [Q_0..Q_H-1 | K_0.. | V_0..], 0/1 projections
    x_sel = np.concatenate([q[h] for h in range(H)] + [k[h] for h in range(H)]
                           + [v[h] for h in range(H)], axis=1)
    sel = np.zeros((3, H, 3 * H * d, d))
    for which in range(3):
        for h in range(H):
            sel[which, h, (which * H + h) * d:(which * H + h + 1) * d, :] = np.eye(d)
    bb_sel = M.Backbone(w_q=sel[0], w_k=sel[1], w_v=sel[2])
    saved = M.rotate_rows
    M.rotate_rows = lambda m, grid_, cfg_: np.asarray(m, np.float64)
    try:
        settings = M.SparseSettings(block=tuple(block3), keep=keep)
        res = [M.block_sparse_attention(x_sel, grid, cfg, bb_sel, h, settings) for h in range(H)]
    finally:
        M.rotate_rows = saved
    o_sparse = [r_.output for r_ in res]
    # real backbone for the linear compensator (random, frozen), dims-only otherwise
    rng = np.random.default_rng(backbone_seed)
    w_lin = [np.asarray(cast(rng.standard_normal((H, D, d)) / math.sqrt(D), "f32"), np.float64)
             for _ in range(3)]
    bb = M.Backbone(w_q=w_lin[0], w_k=w_lin[1], w_v=w_lin[2])
    params = M.MechanismParams(
        w_a=np.asarray(inp["w_a"], np.float64), w_b=np.asarray(inp["w_b"], np.float64),
        alpha=np.asarray(inp["alpha"], np.float64), w_g=np.asarray(inp["w_g"], np.float64),
        b_g=float(inp["b_g"]), rms_sparse=np.asarray(inp["rms_sparse"], np.float64),
        rms_lowrank=np.asarray(inp["rms_lowrank"], np.float64))
    pe = R.pe_from_axis_tables(tuple(grid_ for grid_ in inp["grid"]), inp["pe_t"], inp["pe_x"], inp["pe_y"])
    fs = M.ForwardSettings(sparse=M.SparseSettings(block=tuple(block3), keep=keep),
                           compensator=compensator, use_pe=use_pe)
    out, (x_hat, g, heads) = M._fused_forward(np.asarray(inp["x"], np.float64), o_sparse, pe if use_pe else None,
                                              grid, cfg, bb, params, fs)
    res_d = dict(
        selected=np.stack([r_.selected for r_ in res]),
        sparsity=np.array([r_.sparsity for r_ in res]),
        o_sparse=np.stack(o_sparse),
        o_lowrank=np.stack([hh[4] for hh in heads]),
        g=g, output=out)
    if compensator == "linear":
        res_d.update(w_lin_q=np.asarray(w_lin[0], np.float32), w_lin_k=np.asarray(w_lin[1], np.float32),
                     w_lin_v=np.asarray(w_lin[2], np.float32))
    return res_d


def run_restated(inp, block, keep=None, topk=None, compensator="lowrank", use_pe=True):
    """Flat ragged blocks / fixed top-k fixtures (reference cannot express them)."""
    q, k, v = (np.asarray(inp[n], np.float64) for n in ("q", "k", "v"))
    H, L, d = q.shape
    members = R.flat_block_members(L, block)
    outs, sels, spars = [], [], []
    for h in range(H):
        o, s, sp, _, _ = R.block_sparse_attention(q[h], k[h], v[h], members, keep=keep, topk=topk)
        outs.append(o)
        sels.append(s)
        spars.append(sp)
    pe = R.pe_from_axis_tables(tuple(int(a) for a in inp["grid"]), inp["pe_t"], inp["pe_x"], inp["pe_y"])
    params = {n: inp[n] for n in ("w_a", "w_b", "alpha", "w_g", "b_g", "rms_sparse", "rms_lowrank")}
    fused = R.fused_forward(inp["x"], outs, pe, params, compensator=compensator, use_pe=use_pe)
    return dict(selected=np.stack(sels), sparsity=np.array(spars), o_sparse=np.stack(outs),
                o_lowrank=fused["o_lowrank"], g=fused["g"], output=fused["output"])


CASES = {
    # BASELINE config 0: tile (1,8,8) == flat 64, keep -> top-1, fp32
    "cfg0_lowrank": dict(inputs=dict(seed=0, H=2, d=64, grid=(4, 8, 8), split=(16, 24, 24), r=16, dtype="f32"),
                         ref=dict(block3=(1, 8, 8), keep=1e-12, compensator="lowrank")),
    "cfg0_linear": dict(inputs=dict(seed=0, H=2, d=64, grid=(4, 8, 8), split=(16, 24, 24), r=16, dtype="f32"),
                        ref=dict(block3=(1, 8, 8), keep=1e-12, compensator="linear")),
    # reference-native cumulative-mass rule on true 3D tiles, sinusoidal PE
    "keep3d_sinpe": dict(inputs=dict(seed=1, H=2, d=64, grid=(4, 8, 8), split=(16, 24, 24), r=16, dtype="f32",
                                     pe_kind="sin"),
                         ref=dict(block3=(2, 4, 4), keep=0.6, compensator="lowrank")),
    # bf16, d=128 (the tensor-core path), tile (1,4,16) == flat 64, keep 0.35, no PE
    "bf16_d128_keep": dict(inputs=dict(seed=2, H=2, d=128, grid=(2, 8, 16), split=(44, 42, 42), r=64, dtype="bf16"),
                           ref=dict(block3=(1, 4, 16), keep=0.35, compensator="lowrank", use_pe=False)),
    # bf16, d=128, flat 128-token blocks == tile (1,8,16), top-1 via keep->0
    "bf16_d128_b128": dict(inputs=dict(seed=3, H=1, d=128, grid=(3, 8, 16), split=(16, 56, 56), r=64, dtype="bf16"),
                           ref=dict(block3=(1, 8, 16), keep=1e-12, compensator="lowrank")),
    # bf16, d=128, TRUE 3D tiles (not whole grid rows): the tcgen05 kernel's
    # row_perm path, tile-major token order; 64-token tiles (2,4,8) and
    # 128-token tiles (2,4,16) on a (4,8,16) grid, keep rule, learnable PE
    "bf16_3d_tile64": dict(inputs=dict(seed=6, H=2, d=128, grid=(4, 8, 16), split=(44, 42, 42), r=64, dtype="bf16"),
                           ref=dict(block3=(2, 4, 8), keep=0.5, compensator="lowrank")),
    "bf16_3d_tile128": dict(inputs=dict(seed=7, H=2, d=128, grid=(4, 8, 16), split=(16, 56, 56), r=64,
                                        dtype="bf16"),
                            ref=dict(block3=(2, 4, 16), keep=0.4, compensator="lowrank")),
    # bf16, d=128 linear compensator (the tensor-core linear path) from the reference
    "bf16_d128_linear": dict(inputs=dict(seed=8, H=2, d=128, grid=(2, 8, 16), split=(44, 42, 42), r=64,
                                         dtype="bf16"),
                             ref=dict(block3=(1, 4, 16), keep=0.35, compensator="linear")),
    # ragged flat blocks + fixed top-k (restated; L = 196, block 64 -> last block 4 tokens)
    "ragged_topk_bf16": dict(inputs=dict(seed=4, H=2, d=128, grid=(4, 7, 7), split=(44, 42, 42), r=64, dtype="bf16"),
                             restated=dict(block=64, topk=2, compensator="lowrank")),
    "ragged_topk_f32": dict(inputs=dict(seed=5, H=3, d=64, grid=(3, 5, 9), split=(16, 24, 24), r=16, dtype="f32"),
                            restated=dict(block=32, topk=3, compensator="lowrank")),
}


# Cases run through the reference's real mechanism.forward(x, grid, cfg,
# backbone, params, settings) (mechanism.py:491-512) -- projections and 3D
# RoPE inside the reference -- plus the analysis calls the CLI makes on its
# trace (cli.py:432-433 gram_spectral(trace.o_lowrank[0]), cli.py:463-464
# gate_map(trace.g)).  They pin reference_api.forward end to end.
FORWARD_CASES = {
    "fwd_ref_lowrank": dict(seed=20, H=2, d=64, grid=(4, 8, 8), split=(16, 24, 24), r=16, block3=(1, 8, 8),
                            keep=0.5, compensator="lowrank", use_pe=True),
    "fwd_ref_linear_3d": dict(seed=21, H=2, d=64, grid=(4, 8, 8), split=(16, 24, 24), r=16, block3=(2, 4, 4),
                              keep=0.6, compensator="linear", use_pe=True),
}


def run_reference_forward(seed, H, d, grid, split, r, block3, keep, compensator, use_pe):
    M, GridShape, RopeConfig = _import_reference()
    import ropeslr.analysis as A  # noqa: E402
    g = GridShape(*grid)
    cfg = RopeConfig(*split)
    rng = np.random.default_rng(seed)
    D = H * d
    x = rng.standard_normal((g.size, D))
    backbone = M.random_backbone(H, d, seed + 1)
    params = M.init_params(H, d, r, seed + 2)
    params.w_g = rng.standard_normal(D) * 0.05  # non-zero so the gate path is exercised
    fs = M.ForwardSettings(sparse=M.SparseSettings(block=tuple(block3), keep=keep), compensator=compensator,
                           use_pe=use_pe)
    tr = M.forward(x, g, cfg, backbone, params, fs)
    spec = A.gram_spectral(tr.o_lowrank[0], g, 4)
    gmap = A.gate_map(tr.g, g)
    out = dict(x=x, w_q=backbone.w_q, w_k=backbone.w_k, w_v=backbone.w_v,
               **{f"p_{n}": np.asarray(getattr(params, n)) for n in (
                   "w_a", "w_b", "alpha", "w_g", "b_g", "rms_sparse", "rms_lowrank")},
               grid=np.array(grid), split=np.array(split), block3=np.array(block3), keep=np.float64(keep),
               compensator=np.array(compensator), use_pe=np.bool_(use_pe), source=np.array("reference_forward"))
    for f in ("x_hat", "o_sparse", "o_lowrank", "norm_sparse", "norm_lowrank", "g", "output", "sparsity"):
        out[f"ref_{f}"] = np.asarray(getattr(tr, f))
    out.update(ref_gram_sigma=spec.sigma, ref_gram_modes=spec.modes, ref_gate_values=gmap.values,
               ref_gate_frame_means=gmap.frame_means)
    return out


def main(only=None):
    os.makedirs(OUT_DIR, exist_ok=True)
    for name, spec in CASES.items():
        if only and name not in only:
            continue
        inp = make_inputs(**spec["inputs"])
        if "ref" in spec:
            outs = run_reference(inp, **spec["ref"])
            meta = dict(source=np.array("reference"), block3=np.array(spec["ref"]["block3"]),
                        keep=np.float64(spec["ref"]["keep"]), topk=np.int64(0),
                        compensator=np.array(spec["ref"]["compensator"]),
                        use_pe=np.bool_(spec["ref"].get("use_pe", True)))
        else:
            rs = spec["restated"]
            outs = run_restated(inp, **rs)
            meta = dict(source=np.array("restated"), block3=np.array((0, 0, rs["block"])),
                        keep=np.float64(0.0), topk=np.int64(rs["topk"]),
                        compensator=np.array(rs["compensator"]), use_pe=np.bool_(rs.get("use_pe", True)))
        if str(inp["dtype"]) == "bf16":
            for n in ("q", "k", "v", "x"):
                inp[n] = (np.ascontiguousarray(inp[n], np.float32).view(np.uint32) >> 16).astype(np.uint16)
        path = os.path.join(OUT_DIR, f"{name}.npz")
        np.savez_compressed(path, **inp, **meta, **{f"ref_{k}": v for k, v in outs.items()})
        print(f"{name}: {os.path.getsize(path) / 1024:.0f} KiB, source={meta['source']}, "
              f"sparsity={outs['sparsity']}")
    os.makedirs(os.path.join(OUT_DIR, "forward"), exist_ok=True)
    for name, spec in FORWARD_CASES.items():
        if only and name not in only:
            continue
        path = os.path.join(OUT_DIR, "forward", f"{name}.npz")
        out = run_reference_forward(**spec)
        np.savez_compressed(path, **out)
        print(f"{name}: {os.path.getsize(path) / 1024:.0f} KiB, source=reference_forward, "
              f"sparsity={out['ref_sparsity']}")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
