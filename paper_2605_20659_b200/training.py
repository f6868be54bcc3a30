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

from . import _lib
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
    x: torch.Tensor          # [H, L, d] float32, head-major (contiguous for the per-head GEMMs)
    target: torch.Tensor     # [H, L, d] float32, head-major
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
        H, d = s.q.shape[1], s.q.shape[3]
        out.append(_Prepared(x=_head_major(s.x[0].float(), H, d), target=_head_major(s.target[0].float(), H, d),
                             o_sparse=tr.o_sparse[0].float().contiguous()))
    return out


def _head_major(t: torch.Tensor, H: int, d: int) -> torch.Tensor:
    """[L, H*d] -> contiguous [H, L, d]."""
    return t.view(t.shape[0], H, d).transpose(0, 1).contiguous()


def _at_b(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Per head a^T b for a [H, L, m], b [H, L, n] -> [H, m, n], the long L
    reduction split into S segments (batched GEMMs, then a sum): cuBLAS picks
    a small-tile, single-split kernel for m, n << L otherwise."""
    H, L, m = a.shape
    S = next((c for c in range(32, 1, -1) if L % c == 0 and (L // c) % 4 == 0), 1)
    if S == 1:
        return torch.bmm(a.transpose(1, 2), b)
    a2 = a.reshape(H * S, L // S, m)
    b2 = b.reshape(H * S, L // S, b.shape[2])
    return torch.bmm(a2.transpose(1, 2), b2).view(H, S, m, b.shape[2]).sum(1)


def _tc_gemms(d: int, r: int) -> bool:
    """The tcgen05 float32-grade GEMMs (csrc/stage1_gemm.cu) cover d = 128
    with r in {64, 128}; other shapes use cuBLAS float32."""
    return d == 128 and r in (64, 128)


def _rows(A: torch.Tensor, B: torch.Tensor, *, b_trans: bool = False, epi: int = 0,
          aux: Optional[torch.Tensor] = None) -> torch.Tensor:
    """C[h] = epi(A[h] B[h]) on the tensor cores (ropeslr_stage1_gemm_rows)."""
    H, L, K = A.shape
    N = B.shape[1] if b_trans else B.shape[2]
    C = torch.empty((H, L, N), dtype=torch.float32, device=A.device)
    _lib.call("ropeslr_stage1_gemm_rows", H, L, K, N, A.data_ptr(), B.contiguous().data_ptr(), int(b_trans), epi,
              None if aux is None else aux.data_ptr(), C.data_ptr(), torch.cuda.current_stream(A.device).cuda_stream)
    return C


def _gram_into(out: torch.Tensor, A: torch.Tensor, B: torch.Tensor, transpose: bool) -> None:
    """out[h] += A[h]^T B[h] (or its transpose) on the tensor cores
    (ropeslr_stage1_gemm_gram)."""
    H, L, _ = A.shape
    N = B.shape[2]
    ws = torch.empty(max(16, _lib.lib().ropeslr_stage1_gram_workspace_bytes(H, L, N)), dtype=torch.uint8,
                     device=A.device)
    _lib.call("ropeslr_stage1_gemm_gram", H, L, N, A.data_ptr(), B.data_ptr(), out.data_ptr(), int(transpose), 1,
              ws.data_ptr(), ws.numel(), torch.cuda.current_stream(A.device).cuda_stream)


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
    samples; returns (loss, {name: gradient}) with float32 gradients.

    The per-row chains run as the fused kernels of csrc/stage1.cu between
    the float32 GEMMs (head dims 32 / 64 / 128); other head dims use
    the same math composed from torch ops (_loss_and_grads_composed)."""
    d = params.d_h
    if want_grads and prepared and prepared[0].x.is_cuda and _lib.lib().ropeslr_stage1_supported(d):
        return _loss_and_grads_fused(prepared, params, settings, pe_dense)
    return _loss_and_grads_composed(prepared, params, settings, pe_dense, want_grads)


def _loss_and_grads_fused(prepared, params, settings, pe_dense):
    acc, grads = _fused_device(prepared, params, settings, pe_dense)
    loss, gb = acc.tolist()  # the one host read of the step (the reference trainer reads the loss too)
    grads["b_g"] = float(gb)
    return float(loss), grads


def _fused_device(prepared, params, settings, pe_dense, b_g_dev: Optional[torch.Tensor] = None):
    """The fused loss and gradients with no host read: (acc = float64 [loss,
    d b_g] on the device, {name: float32 gradient} without b_g).  With
    ``b_g_dev`` (float64 [1]) the gate bias is read from the device, so the
    sequence can be captured in a CUDA graph and replayed (Stage1Step)."""
    eps = settings.rms_eps
    H, d, r = params.n_heads, params.d_h, params.rank
    dev = prepared[0].x.device
    st = torch.cuda.current_stream(dev).cuda_stream
    lib = _lib.lib()
    w_a, w_b = params.w_a.float().contiguous(), params.w_b.float().contiguous()
    alpha, w_g = params.alpha.float().contiguous(), params.w_g.float().contiguous()
    rms_sp, rms_lr = params.rms_sparse.float().contiguous(), params.rms_lowrank.float().contiguous()
    grads = {n: torch.zeros_like(getattr(params, n), dtype=torch.float32) for n in PARAM_NAMES}
    n = len(prepared)
    use_pe = settings.use_pe
    acc = torch.zeros(2, dtype=torch.float64, device=dev)  # loss, d b_g
    rms_acc = torch.zeros((2, d), dtype=torch.float32, device=dev)
    x_acc = torch.zeros((H, 2, d), dtype=torch.float32, device=dev)
    for s in prepared:
        _, L, _ = s.x.shape
        xh = torch.empty_like(s.x)
        gpart = torch.empty((H, L), dtype=torch.float32, device=dev)
        g = torch.empty((L,), dtype=torch.float32, device=dev)
        pe_ptr = pe_dense.data_ptr() if use_pe else None
        if b_g_dev is None:
            _lib.call("ropeslr_stage1_pre", H, L, d, s.x.data_ptr(), pe_ptr, alpha.data_ptr(), w_g.data_ptr(),
                      float(params.b_g), xh.data_ptr(), gpart.data_ptr(), g.data_ptr(), st)
        else:
            _lib.call("ropeslr_stage1_pre_dev", H, L, d, s.x.data_ptr(), pe_ptr, alpha.data_ptr(), w_g.data_ptr(),
                      b_g_dev.data_ptr(), xh.data_ptr(), gpart.data_ptr(), g.data_ptr(), st)
        tc = _tc_gemms(d, r)
        if tc:
            h1 = _rows(xh, w_a, epi=1)                                    # sigma(x_hat W_A) [H, L, r]
            dz2 = _rows(h1, w_b)                                          # z2 in, d z2 out (in place)
        else:
            h1 = torch.sigmoid_(torch.bmm(xh, w_a))
            dz2 = torch.bmm(h1, w_b)
        nb_rows = lib.ropeslr_stage1_rows_blocks(H, L)
        red = torch.empty((nb_rows, 2, d), dtype=torch.float32, device=dev)
        loss_part = torch.empty((nb_rows,), dtype=torch.float64, device=dev)
        dgpart = torch.empty((H, L), dtype=torch.float32, device=dev)
        _lib.call("ropeslr_stage1_rows", H, L, d, dz2.data_ptr(), s.o_sparse.data_ptr(), s.target.data_ptr(),
                  g.data_ptr(), rms_sp.data_ptr(), rms_lr.data_ptr(), float(eps), 2.0 / (H * L * d * n),
                  dgpart.data_ptr(), red.data_ptr(), loss_part.data_ptr(), st)
        _lib.call("ropeslr_stage1_reduce", red.data_ptr(), 1, nb_rows, 2, d, rms_acc.data_ptr(), st)
        dzg = torch.empty((L,), dtype=torch.float32, device=dev)
        bg_part = torch.empty((-(-L // 256),), dtype=torch.float64, device=dev)
        _lib.call("ropeslr_stage1_gate_bwd", H, L, dgpart.data_ptr(), g.data_ptr(), dzg.data_ptr(),
                  bg_part.data_ptr(), st)
        acc[0] += loss_part.sum() / (H * L * d * n)
        acc[1] += bg_part.sum()
        if tc:
            _gram_into(grads["w_b"], dz2, h1, transpose=True)            # (dz2^T h1)^T = h1^T dz2
            dz1 = _rows(dz2, w_b, b_trans=True, epi=2, aux=h1)            # (dz2 W_B^T) h1 (1 - h1)
            _gram_into(grads["w_a"], xh, dz1, transpose=False)            # x_hat^T dz1
            dxh = _rows(dz1, w_a, b_trans=True) if use_pe else xh         # dz1 W_A^T (read only with PE)
        else:
            grads["w_b"] += _at_b(h1, dz2)
            dz1 = torch.bmm(dz2, w_b.transpose(1, 2))
            _lib.call("ropeslr_stage1_dsig", dz1.data_ptr(), h1.data_ptr(), dz1.numel(), st)
            grads["w_a"] += _at_b(xh, dz1)
            dxh = torch.bmm(dz1, w_a.transpose(1, 2)) if use_pe else xh
        nb_x = lib.ropeslr_stage1_xgrad_blocks(H, L)
        xred = torch.empty((H, nb_x, 2, d), dtype=torch.float32, device=dev)
        _lib.call("ropeslr_stage1_xgrad", H, L, d, dxh.data_ptr(), xh.data_ptr(), pe_ptr, dzg.data_ptr(),
                  w_g.data_ptr(), xred.data_ptr(), st)
        _lib.call("ropeslr_stage1_reduce", xred.data_ptr(), H, nb_x, 2, d, x_acc.data_ptr(), st)
    grads["rms_sparse"] += rms_acc[0]
    grads["rms_lowrank"] += rms_acc[1]
    if use_pe:
        grads["alpha"] += x_acc[:, 0].reshape(-1)
    grads["w_g"] += x_acc[:, 1].reshape(-1)
    return acc, grads


class Stage1Step:
    """The fused Stage-I step (loss, gradients, the gradient-descent update)
    captured once in a CUDA graph per phase and replayed: no host work and
    no launch gaps between the kernels, one host read of the loss per step
    (mechanism.py:582-614 reads it too).  The update runs only when the step's
    loss is finite, on the device, so a diverging step leaves the parameters
    as the reference leaves them.  ``params`` are updated in place; b_g lives
    on the device during training and is written back by ``sync_bias``."""

    def __init__(self, prepared, params: MechanismParams, settings: ForwardSettings,
                 pe_dense: Optional[torch.Tensor], lr: float):
        if not (prepared and prepared[0].x.is_cuda and _lib.lib().ropeslr_stage1_supported(params.d_h)):
            raise ValueError("the captured Stage-I step needs CUDA samples with a fused head dim (32 / 64 / 128)")
        self.params = params
        dev = prepared[0].x.device
        self.b_g = torch.full((1,), float(params.b_g), dtype=torch.float64, device=dev)
        lr_t = torch.full((), lr, dtype=torch.float64, device=dev)
        zero_t = torch.zeros((), dtype=torch.float64, device=dev)
        names = [n for n in PARAM_NAMES if n != "b_g"]
        consts = {getattr(params, n).dtype: (lr_t.to(getattr(params, n).dtype), zero_t.to(getattr(params, n).dtype))
                  for n in names}
        # the graphs read these by address: they must live as long as the graphs
        self._keep = (lr_t, zero_t, consts, prepared, pe_dense)

        def body(update: bool):
            acc, grads = _fused_device(prepared, params, settings, pe_dense, self.b_g)
            if update:
                ok = torch.isfinite(acc[0])
                with torch.no_grad():
                    for name in names:
                        p = getattr(params, name)
                        lr_p, zero_p = consts[p.dtype]
                        p.sub_(torch.where(ok, grads[name].to(p.dtype) * lr_p, zero_p))
                    self.b_g.sub_(torch.where(ok, acc[1] * lr_t, zero_t))
            return acc

        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            body(False)  # warm-up outside the capture (workspaces, attributes)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.g_loss = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_loss):
            self.acc_loss = body(False)
        self.g_step = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_step, pool=self.g_loss.pool()):
            self.acc_step = body(True)

    def step(self) -> float:
        """Loss at the current parameters, then the update (if finite)."""
        self.g_step.replay()
        return float(self.acc_step[0].item())

    def loss(self) -> float:
        """Loss at the current parameters, no update."""
        self.g_loss.replay()
        return float(self.acc_loss[0].item())

    def sync_bias(self) -> None:
        self.params.b_g = float(self.b_g.item())


def _loss_and_grads_composed(prepared: Sequence[_Prepared], params: MechanismParams, settings: ForwardSettings,
                             pe_dense: Optional[torch.Tensor], want_grads: bool = True):
    eps = settings.rms_eps
    H, d, r = params.n_heads, params.d_h, params.rank
    w_a, w_b = params.w_a.float(), params.w_b.float()
    alpha, w_g = params.alpha.float(), params.w_g.float()
    rms_sp, rms_lr = params.rms_sparse.float(), params.rms_lowrank.float()
    grads = {n: torch.zeros_like(getattr(params, n), dtype=torch.float32) for n in PARAM_NAMES} if want_grads else None
    gb = torch.zeros((), dtype=torch.float64, device=w_a.device)
    total = 0.0
    n = len(prepared)
    w_g_h = w_g.view(H, d)
    alpha_h = alpha.view(H, d)
    for s in prepared:
        _, L, _ = s.x.shape
        # everything head-major [H, L, d]: contiguous operands for the batched
        # GEMMs and vectorised elementwise kernels (no strided permutes)
        xh = s.x + alpha_h[:, None, :] * pe_dense if settings.use_pe else s.x
        g = torch.sigmoid(torch.einsum("hld,hd->l", xh, w_g_h) + params.b_g)  # [L]
        h1 = torch.sigmoid(torch.bmm(xh, w_a))                               # [H, L, r]
        o_lr = torch.sigmoid(torch.bmm(h1, w_b))                             # [H, L, d]
        y_lr, inv_lr, u_lr = _rms(o_lr, rms_lr, eps)
        y_sp, inv_sp, u_sp = _rms(s.o_sparse, rms_sp, eps)
        diff = torch.addcmul(y_sp, g[None, :, None], y_lr) - s.target
        total += float((diff.double() ** 2).mean()) / n
        if not want_grads:
            continue
        gh = diff * (2.0 / (diff.numel() * n))                                # [H, L, d]
        grads["rms_sparse"] += (gh * u_sp).reshape(-1, d).sum(0)
        d_g = (gh * y_lr).sum((0, 2))                                         # [L]
        d_o_lr, d_rl = _rms_backward(gh * g[None, :, None], o_lr, inv_lr, u_lr, rms_lr)
        grads["rms_lowrank"] += d_rl
        d_z2 = d_o_lr * o_lr * (1.0 - o_lr)
        grads["w_b"] += _at_b(h1, d_z2)
        d_z1 = torch.bmm(d_z2, w_b.transpose(1, 2)) * h1 * (1.0 - h1)
        grads["w_a"] += _at_b(xh, d_z1)
        d_xh = torch.bmm(d_z1, w_a.transpose(1, 2))                          # [H, L, d]
        d_zg = d_g * g * (1.0 - g)
        grads["w_g"] += torch.einsum("hld,l->hd", xh, d_zg).reshape(-1)
        gb += d_zg.double().sum()
        if settings.use_pe:
            d_xh = d_xh + d_zg[None, :, None] * w_g_h[:, None, :]
            grads["alpha"] += (d_xh * pe_dense).sum(1).reshape(-1)
    if want_grads:
        grads["b_g"] = float(gb)
    return total, grads


def pe_head_major(pe: PETables, grid: GridShape, H: int, d: int) -> torch.Tensor:
    """The dense 3D PE [L, H*d] as the head-major float32 [H, L, d] that
    loss_and_grads takes."""
    return _head_major(pe.dense(grid).float(), H, d)


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
    pe_dense = pe_head_major(pe, grid, params.n_heads, params.d_h) if settings.use_pe else None
    losses = []
    if steps > 0 and prepared[0].x.is_cuda and _lib.lib().ropeslr_stage1_supported(params.d_h):
        # the captured step: loss, gradients and the guarded update per replay
        runner = Stage1Step(prepared, params, settings, pe_dense, lr)
        try:
            for step in range(steps + 1):
                loss = runner.step() if step < steps else runner.loss()
                losses.append(loss)
                if not np.isfinite(loss):
                    return TrainResult(losses=np.asarray(losses), diverged=True)
        finally:
            runner.sync_bias()
        return TrainResult(losses=np.asarray(losses), diverged=False)
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
