"""reference_api.forward: the reference-shaped drop-in for mechanism.forward
(mechanism.py:491-512), pinned by fixtures from the reference's own
mechanism.forward and analysis functions (oracle/make_golden.py
FORWARD_CASES).  The device tests feed the trace to the CLI's analysis
calls as cli.py:432-433 (gram_spectral(trace.o_lowrank[0])) and
cli.py:463-464 (gate_map(trace.g)) do; the analysis functions are restated
here (SVD, reshape), the reference's results are in the fixture."""

import os
from types import SimpleNamespace

import numpy as np
import pytest
import torch

import gpu_helpers as G

FWD_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "forward")
CASES = sorted(os.path.splitext(n)[0] for n in os.listdir(FWD_DIR))


def _load(name):
    with np.load(os.path.join(FWD_DIR, f"{name}.npz")) as z:
        g = {k: z[k] for k in z.files}
    grid_t = tuple(int(a) for a in g["grid"])
    split = tuple(int(a) for a in g["split"])
    # stand-ins with the reference dataclasses' attribute names (rope3d.py:25-99,
    # mechanism.py:47-133, 258-270, 387-396)
    grid = SimpleNamespace(t=grid_t[0], h=grid_t[1], w=grid_t[2], size=int(np.prod(grid_t)))
    cfg = SimpleNamespace(d_t=split[0], d_x=split[1], d_y=split[2], base=10000.0)
    backbone = SimpleNamespace(w_q=g["w_q"], w_k=g["w_k"], w_v=g["w_v"])
    params = SimpleNamespace(**{n: g[f"p_{n}"] for n in ("w_a", "w_b", "alpha", "w_g", "rms_sparse", "rms_lowrank")},
                             b_g=float(g["p_b_g"]))
    settings = SimpleNamespace(sparse=SimpleNamespace(block=tuple(int(b) for b in g["block3"]), keep=float(g["keep"])),
                               compensator=str(g["compensator"]), use_pe=bool(g["use_pe"]), rms_eps=1e-6)
    return g, grid, cfg, backbone, params, settings


def gram_sigma(o_lr):
    """analysis.gram_spectral's singular values (analysis.py:128-141)."""
    return np.linalg.svd(np.asarray(o_lr, np.float64), compute_uv=False)


def gate_frame_means(g, grid):
    """analysis.gate_map's frame means (analysis.py:153-159)."""
    return np.asarray(g, np.float64).reshape(grid.t, grid.h, grid.w).mean(axis=(1, 2))


def test_reference_errors_on_cpu():
    """Non-finite input and a wrong shape raise ValueError before any device
    work, like the reference (linalg.py:17-20, mechanism.py:495-496)."""
    from paper_2605_20659_b200 import reference_api as RA

    g, grid, cfg, backbone, params, settings = _load(CASES[0])
    x = g["x"].copy()
    x[3, 5] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        RA.forward(x, grid, cfg, backbone, params, settings)
    x[3, 5] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        RA.forward(x, grid, cfg, backbone, params, settings)
    with pytest.raises(ValueError, match="expected input shape"):
        RA.forward(g["x"][:-1], grid, cfg, backbone, params, settings)
    with pytest.raises(ValueError):
        RA.forward(g["x"][None], grid, cfg, backbone, params, settings)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_reference_forward_trace(name):
    from paper_2605_20659_b200 import reference_api as RA

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    g, grid, cfg, backbone, params, settings = _load(name)
    tr = RA.forward(g["x"], grid, cfg, backbone, params, settings)
    H, L, d = g["ref_o_sparse"].shape
    for f in ("o_sparse", "o_lowrank", "norm_sparse", "norm_lowrank"):
        assert getattr(tr, f).shape == (H, L, d), f
    assert tr.x_hat.shape == tr.output.shape == (L, H * d)
    assert tr.g.shape == (L,) and tr.sparsity.shape == (H,)
    np.testing.assert_allclose(tr.sparsity, g["ref_sparsity"], rtol=0, atol=1e-15)
    for f in ("x_hat", "o_sparse", "o_lowrank", "norm_sparse", "norm_lowrank", "g", "output"):
        G.assert_close(getattr(tr, f), g[f"ref_{f}"], "f32", f"{name} {f}", scale=10.0)
    # the CLI's consumers of the trace (cli.py:433, 464)
    np.testing.assert_allclose(gram_sigma(tr.o_lowrank[0]), g["ref_gram_sigma"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(gate_frame_means(tr.g, grid), g["ref_gate_frame_means"], rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(tr.g.reshape(grid.t, grid.h, grid.w), g["ref_gate_values"], rtol=1e-5, atol=1e-7)


@pytest.mark.gpu
def test_reference_forward_rejects_nonfinite_on_device_path():
    """The device forward flags non-finite Q/K (block means) and X (gate
    logits) when asked, and passes clean inputs."""
    import paper_2605_20659_b200 as P

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    q, k, v, x, params, pe, grid = G.make_full_inputs((2, 8, 16), 2, 128, (44, 42, 42), 64)
    st = P.ForwardSettings(P.SparseSettings(block=64, topk=2))
    P.forward(q, k, v, x, grid, params, st, pe, check_finite=True)
    for which, val in (("q", float("nan")), ("k", float("inf")), ("x", float("-inf"))):
        t = {"q": q, "k": k, "x": x}[which].clone()
        t.view(-1)[777] = val
        args = dict(q=q, k=k, x=x)
        args[which] = t
        with pytest.raises(ValueError, match="non-finite"):
            P.forward(args["q"], args["k"], v, args["x"], grid, params, st, pe, check_finite=True)
    # the host-buffer API always checks
    xh = x.cpu().clone()
    xh.view(-1)[5] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        P.forward_host(q.cpu(), k.cpu(), v.cpu(), xh, grid, params, st, pe)
