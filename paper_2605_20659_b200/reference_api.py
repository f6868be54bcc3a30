"""Reference-shaped drop-in for ``ropeslr.mechanism.forward``.

``forward(x, grid, cfg, backbone, params, settings)`` takes and returns what
the reference's ``mechanism.forward`` does (mechanism.py:491-512): NumPy
float64 arrays and the reference's own config / parameter objects (read by
attribute, so the reference's dataclasses work unchanged), and it returns a
``ForwardTrace`` with the reference's fields and per-head shapes
(mechanism.py:399-408):

    x_hat (L, D), o_sparse / o_lowrank / norm_sparse / norm_lowrank (H, L, d),
    g (L,), output (L, D), sparsity (H,)

so callers that index the trace -- ``trace.o_lowrank[0]`` into
``analysis.gram_spectral`` (cli.py:433), ``trace.g`` into
``analysis.gate_map`` (cli.py:464) -- get the same thing.

The compute runs on the device through the C ABI: the frozen projections and
the 3D RoPE are the caller-side step (``mechanism.forward_from_x``), then K1
(selection), K3 (compensator + gate), K2+K4 (sparse attention + fused
epilogue).  ``x_hat``, ``norm_sparse`` and ``norm_lowrank`` are trace-only
intermediates the op does not otherwise materialise; they are derived on the
device from the kernels' float32 branch outputs.

Errors follow the reference: non-finite input -> ValueError (linalg.py:17-20),
wrong input shape -> ValueError (mechanism.py:495-496), bad settings ->
ValueError.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import mechanism as M
from .rope3d import GridShape, RopeConfig


@dataclass(frozen=True)
class ForwardTrace:
    """mechanism.py:399-408, NumPy float64."""

    x_hat: np.ndarray
    o_sparse: np.ndarray  # (H, L, d_h)
    o_lowrank: np.ndarray  # (H, L, d_h) compensator outputs, pre-normalisation
    norm_sparse: np.ndarray
    norm_lowrank: np.ndarray
    g: np.ndarray  # (L,)
    output: np.ndarray  # (L, d_model)
    sparsity: np.ndarray  # (H,)


def as_matrix(x) -> np.ndarray:
    """float64 2-D array with finite entries (linalg.py:14-21)."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError("matrix contains non-finite values")
    return a


def _grid(g) -> GridShape:
    return g if isinstance(g, GridShape) else GridShape(int(g.t), int(g.h), int(g.w))


def _rope(c) -> RopeConfig:
    return c if isinstance(c, RopeConfig) else RopeConfig(int(c.d_t), int(c.d_x), int(c.d_y), float(c.base))


def _settings(s) -> M.ForwardSettings:
    sp = s.sparse
    block = tuple(int(b) for b in sp.block) if isinstance(sp.block, (tuple, list)) else int(sp.block)
    sparse = M.SparseSettings(block=block, keep=float(getattr(sp, "keep", 1.0)), topk=int(getattr(sp, "topk", 0)))
    return M.ForwardSettings(sparse, compensator=s.compensator, use_pe=bool(s.use_pe),
                             rms_eps=float(getattr(s, "rms_eps", M.RMS_EPS)))


def _rms(o: torch.Tensor, scale: torch.Tensor, eps: float) -> torch.Tensor:
    """rms_norm (mechanism.py:238-246) on the device, float64."""
    return o * torch.rsqrt(o.pow(2).mean(-1, keepdim=True) + eps) * scale


def forward(x, grid, cfg, backbone, params, settings, *, dtype: torch.dtype = torch.float32,
            device=None) -> ForwardTrace:
    """Drop-in for ``mechanism.forward`` (mechanism.py:491-512).

    dtype: storage dtype of the op's Q/K/V/X (float32 default; bfloat16 runs
    the tensor-core kernels for d_h = 128)."""
    x = as_matrix(x)
    g_ = _grid(grid)
    if x.shape != (g_.size, int(backbone.w_q.shape[1])):
        raise ValueError(f"expected input shape {(g_.size, int(backbone.w_q.shape[1]))}, got {x.shape}")
    rope = _rope(cfg)
    fs = _settings(settings)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    f64 = lambda a: torch.as_tensor(np.asarray(a, np.float64), device=dev)  # noqa: E731
    bb = M.Backbone(f64(backbone.w_q), f64(backbone.w_k), f64(backbone.w_v))
    p = M.MechanismParams.from_arrays(device=dev, **{n: np.asarray(getattr(params, n), np.float64) for n in (
        "w_a", "w_b", "alpha", "w_g", "rms_sparse", "rms_lowrank")}, b_g=float(params.b_g))
    pe = M.PETables.sinusoidal(g_, bb.d_model, rope, device=dev) if fs.use_pe else None
    xd = f64(x)
    tr = M.forward_from_x(xd, g_, rope, bb, p, fs, pe, dtype=dtype, trace=True)
    x_hat = xd
    if fs.use_pe:
        x_hat = xd + p.alpha.double()[None, :] * pe.dense(g_).double()
    o_sp = tr.o_sparse[0].double()
    o_lr = tr.o_lowrank[0].double()
    norm_sp = _rms(o_sp, p.rms_sparse.double(), fs.rms_eps)
    norm_lr = _rms(o_lr, p.rms_lowrank.double(), fs.rms_eps)
    np_ = lambda t: t.detach().to(torch.float64).cpu().numpy()  # noqa: E731
    return ForwardTrace(x_hat=np_(x_hat), o_sparse=np_(o_sp), o_lowrank=np_(o_lr), norm_sparse=np_(norm_sp),
                        norm_lowrank=np_(norm_lr), g=np_(tr.g[0]), output=np_(tr.output[0]),
                        sparsity=np_(tr.sparsity[0]))
