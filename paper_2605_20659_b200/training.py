"""Stage-I alignment training of the new parameters (SURVEY.md 8f "next" #3).

Mirrors the reference trainer (mechanism.py:519-614): the sparse branch reads
the frozen backbone, so it is computed once per sample -- by the B200 op (K1
selection + K2 tcgen05 attention, float32 o_sparse) -- and cached
(mechanism.py:536-549); each step then runs the fused forward / backward of
the low-rank compensator, the gate, the RMSNorms and the PE injection
(mechanism.py:426-488) against the cached branch and takes a plain
gradient-descent step on W_A, W_B, alpha, w_g, b_g, rms_sparse, rms_lowrank
(mechanism.py:582-614).  The per-step math is batched over heads and
samples' tokens as float32 device GEMMs (cuBLAS) and elementwise kernels;
the loss is the reference's mean squared error against fixed targets
(mechanism.py:519-526, 552-565).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from .mechanism import ForwardSettings, MechanismParams, PETables, forward
from .rope3d import GridShape

PARAM_NAMES = ("w_a", "w_b", "alpha", "w_g", "rms_sparse", "rms_lowrank")


@dataclass
class Stage1Sample:
    """One training sample: post-RoPE Q/K/V [1, H, L, d], token features
    X [1, L, H*d] and the target output [1, L, H*d] (e.g. full attention)."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    x: torch.Tensor
    target: torch.Tensor


@dataclass
class _Prepared:
    x: torch.Tensor          # [L, D] float32
    target: torch.Tensor     # [L, D] float32
    o_sparse: torch.Tensor   # [H, L, d] float32 (constant during training)


@dataclass
class TrainResult:
    losses: np.ndarray
    diverged: bool

    @property
    def initial_loss(self) -> float:
        return float(self.losses[0])

    @property
    def final_loss(self) -> float:
        return float(self.losses[-1])


def prepare(samples: Sequence[Stage1Sample], grid: GridShape, params: MechanismParams, settings: ForwardSettings,
            pe: Optional[PETables] = None) -> List[_Prepared]:
    """Cache the sparse branch of every sample through the op (mechanism.py:536-549)."""
    if settings.compensator != "lowrank":
        raise ValueError("Stage-I training is implemented for the low-rank compensator")
    out = []
    for s in samples:
        if s.q.shape[0] != 1:
            raise ValueError("samples are single sequences (B = 1)")
        tr = forward(s.q, s.k, s.v, s.x, grid, params, settings, pe, trace=True)
        out.append(_Prepared(x=s.x[0].float(), target=s.target[0].float(), o_sparse=tr.o_sparse[0].float()))
    return out


def _rms(o, scale, eps):
    inv = torch.rsqrt((o * o).mean(-1, keepdim=True) + eps)
    u = o * inv
    return u * scale, inv, u


def _rms_backward(d_y, o, inv, u, scale):
    """mechanism._rms_backward (mechanism.py:417-423), batched over leading dims."""
    d_scale = (d_y * u).reshape(-1, u.shape[-1]).sum(0)
    d_u = d_y * scale
    dot = (d_u * o).sum(-1, keepdim=True)
    d_o = d_u * inv - o * (inv ** 3 * dot / o.shape[-1])
    return d_o, d_scale


def loss_and_grads(prepared: Sequence[_Prepared], params: MechanismParams, settings: ForwardSettings,
                   pe_dense: Optional[torch.Tensor], want_grads: bool = True):
    """mechanism._loss_and_grads (mechanism.py:552-565) over the prepared
    samples; returns (loss, {name: gradient}) with float32 gradients."""
    eps = settings.rms_eps
    H, d, r = params.n_heads, params.d_h, params.rank
    w_a, w_b = params.w_a.float(), params.w_b.float()
    alpha, w_g = params.alpha.float(), params.w_g.float()
    rms_sp, rms_lr = params.rms_sparse.float(), params.rms_lowrank.float()
    grads = {n: torch.zeros_like(getattr(params, n), dtype=torch.float32) for n in PARAM_NAMES} if want_grads else None
    gb = torch.zeros((), dtype=torch.float64, device=w_a.device)
    total = 0.0
    n = len(prepared)
    for s in prepared:
        L, D = s.x.shape
        x_hat = s.x + alpha[None, :] * pe_dense if settings.use_pe else s.x
        g = torch.sigmoid(x_hat @ w_g + params.b_g)                          # [L]
        xh = x_hat.view(L, H, d).permute(1, 0, 2)                            # [H, L, d]
        h1 = torch.sigmoid(torch.bmm(xh, w_a))                               # [H, L, r]
        o_lr = torch.sigmoid(torch.bmm(h1, w_b))                             # [H, L, d]
        y_lr, inv_lr, u_lr = _rms(o_lr, rms_lr, eps)
        y_sp, inv_sp, u_sp = _rms(s.o_sparse, rms_sp, eps)
        out = (y_sp + g[None, :, None] * y_lr).permute(1, 0, 2).reshape(L, D)
        diff = out - s.target
        total += float((diff.double() ** 2).mean()) / n
        if not want_grads:
            continue
        gh = (2.0 * diff / (diff.numel() * n)).view(L, H, d).permute(1, 0, 2)  # [H, L, d]
        grads["rms_sparse"] += (gh * u_sp).reshape(-1, d).sum(0)
        d_g = (gh * y_lr).sum((0, 2))                                         # [L]
        d_o_lr, d_rl = _rms_backward(gh * g[None, :, None], o_lr, inv_lr, u_lr, rms_lr)
        grads["rms_lowrank"] += d_rl
        d_z2 = d_o_lr * o_lr * (1.0 - o_lr)
        grads["w_b"] += torch.bmm(h1.transpose(1, 2), d_z2)
        d_z1 = torch.bmm(d_z2, w_b.transpose(1, 2)) * h1 * (1.0 - h1)
        grads["w_a"] += torch.bmm(xh.transpose(1, 2), d_z1)
        d_xhat = torch.bmm(d_z1, w_a.transpose(1, 2)).permute(1, 0, 2).reshape(L, D)
        d_zg = d_g * g * (1.0 - g)
        grads["w_g"] += x_hat.t() @ d_zg
        gb += d_zg.double().sum()
        d_xhat = d_xhat + torch.outer(d_zg, w_g)
        if settings.use_pe:
            grads["alpha"] += (d_xhat * pe_dense).sum(0)
    if want_grads:
        grads["b_g"] = float(gb)
    return total, grads


def train_stage1(samples: Sequence[Stage1Sample], grid: GridShape, params: MechanismParams,
                 settings: ForwardSettings, pe: Optional[PETables], lr: float, steps: int) -> TrainResult:
    """Plain gradient descent on the new parameters against fixed targets
    (mechanism.py:582-614); mutates ``params`` in place, a non-finite loss
    aborts the run and reports it."""
    if not (np.isfinite(lr) and lr >= 0.0):
        raise ValueError(f"learning rate must be a non-negative real, got {lr}")
    if steps < 0:
        raise ValueError("step count must be non-negative")
    if not samples:
        raise ValueError("dataset must be non-empty")
    prepared = prepare(samples, grid, params, settings, pe)
    pe_dense = pe.dense(grid).float() if settings.use_pe else None
    losses = []
    for step in range(steps + 1):
        loss, grads = loss_and_grads(prepared, params, settings, pe_dense, want_grads=step < steps)
        losses.append(loss)
        if not np.isfinite(loss):
            return TrainResult(losses=np.asarray(losses), diverged=True)
        if step == steps:
            break
        with torch.no_grad():
            for name in PARAM_NAMES:
                getattr(params, name).sub_(lr * grads[name].to(getattr(params, name).dtype))
        params.b_g = float(params.b_g) - lr * grads["b_g"]
    return TrainResult(losses=np.asarray(losses), diverged=False)
