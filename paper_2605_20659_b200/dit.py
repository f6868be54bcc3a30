"""Wan2.1-1.3B-architecture DiT with RoPeSLR self-attention (BASELINE
config 4): the caller of the op in an end-to-end denoising step.

This is not the reference's code -- the reference has no model (SURVEY.md
8f "next" #2) -- but a random-init stand-in with the published shape:
30 blocks, hidden 1536, 12 heads of 128, FFN 8960, cross-attention to 512
text tokens of width 4096, a 16-channel latent patched 1x2x2.  Per block:

  adaLN-modulated LayerNorm -> Q/K/V projections (cuBLAS) with RMSNorm on
  Q and K -> RoPeSLR attention (the op; Q/K rotated by its fused RoPE +
  pooling pre-pass; X = the modulated hidden state feeds the low-rank
  compensator and gate) -> output projection, gated residual;
  cross-attention to the text tokens (torch SDPA); modulated FFN (GELU-tanh).

With a process group, the sequence is sharded across the ranks and the op
runs under ulysses_attention (all-to-all seq <-> head around it); every
other layer is token-wise and needs no communication.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import _lib
from .mechanism import ForwardSettings, MechanismParams, PETables, SparseSettings, forward
from .rope3d import GridShape, RopeConfig
from .ulysses import seq_slice, ulysses_attention


@dataclass(frozen=True)
class WanConfig:
    """Wan2.1-1.3B shape (BASELINE config 4)."""

    dim: int = 1536
    heads: int = 12
    ffn: int = 8960
    blocks: int = 30
    text_len: int = 512
    text_dim: int = 4096
    in_channels: int = 16
    patch: tuple = (1, 2, 2)
    freq_dim: int = 256
    rank: int = 64
    sparsity: float = 0.9
    block: int = 64
    rope_split: tuple = (44, 42, 42)
    eps: float = 1e-6

    @property
    def head_dim(self) -> int:
        return self.dim // self.heads


class RMSNorm(nn.Module):
    def __init__(self, dim, eps):
        super().__init__()
        self.eps = eps
        self.weight = nn.Parameter(torch.ones(dim))

    def forward(self, x):
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)).to(x.dtype) * self.weight


# ---- fused token-wise ops of the block (csrc/dit_ops.cu): one launch each
# where the PyTorch composition runs 5-8 elementwise kernels, bf16 rows.
# FUSED_OPS = False runs the plain PyTorch composition (tests compare both).
FUSED_OPS = True
def _stream(t):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def ln_modulate(x: torch.Tensor, shift: torch.Tensor, scale: torch.Tensor, eps: float) -> torch.Tensor:
    """bf16(LayerNorm(x) * (1 + scale) + shift); x [B, L, D] bf16, shift /
    scale broadcastable to [D] (float32)."""
    D = x.shape[-1]
    x = x.contiguous()
    sh = shift.reshape(-1)[-D:].float().contiguous()
    sc = scale.reshape(-1)[-D:].float().contiguous()
    y = torch.empty_like(x)
    _lib.call("ropeslr_dit_ln_modulate", x.data_ptr(), sh.data_ptr(), sc.data_ptr(), float(eps), x.numel() // D, D,
              y.data_ptr(), _stream(x))
    return y


def ln_affine(x: torch.Tensor, ln: nn.LayerNorm) -> torch.Tensor:
    """bf16(LayerNorm(x) * weight + bias) for an affine nn.LayerNorm; x
    [B, L, D] bf16."""
    D = x.shape[-1]
    x = x.contiguous()
    w = ln.weight.detach().float().contiguous()
    b = ln.bias.detach().float().contiguous()
    y = torch.empty_like(x)
    _lib.call("ropeslr_dit_ln_affine", x.data_ptr(), w.data_ptr(), b.data_ptr(), float(ln.eps), x.numel() // D, D,
              y.data_ptr(), _stream(x))
    return y


def rms_heads(x: torch.Tensor, weight: Optional[torch.Tensor], eps: float, H: int, head_major: bool = True):
    """RMSNorm over the last dim (weight None: none) of x [1, L, D] bf16; out
    [1, H, L, D/H] when head_major, else [1, L, H, D/H]."""
    B, L, D = x.shape
    if B != 1:
        raise ValueError("rms_heads: batch 1 (the DiT step)")
    if x.stride(-1) != 1 or x.stride(-2) % 8 or x.data_ptr() % 16:
        x = x.contiguous()
    out = torch.empty((1, H, L, D // H) if head_major else (1, L, H, D // H), dtype=x.dtype, device=x.device)
    w = None if weight is None else weight.to(x.dtype).contiguous()
    # a column slice of wider rows (the fused QKV projection) is read in place
    _lib.call("ropeslr_dit_rms_heads_strided", x.data_ptr(), x.stride(-2), None if w is None else w.data_ptr(),
              float(eps), L, D, H, int(head_major), out.data_ptr(), _stream(x))
    return out


def gated_residual_(x: torch.Tensor, y: torch.Tensor, gate: torch.Tensor) -> torch.Tensor:
    """x += bf16(y * gate) in place; x, y [B, L, D] bf16, gate -> [D] float32."""
    D = x.shape[-1]
    if not x.is_contiguous():
        raise ValueError("gated_residual_: x must be contiguous")
    y = y.contiguous()
    g = gate.reshape(-1)[-D:].float().contiguous()
    _lib.call("ropeslr_dit_gated_residual", x.data_ptr(), y.data_ptr(), g.data_ptr(), x.numel() // D, D, _stream(x))
    return x


def gated_add(x: torch.Tensor, y: torch.Tensor, gate: torch.Tensor) -> torch.Tensor:
    """x + bf16(y * gate) into a new tensor; x, y [B, L, D] bf16, gate -> [D] float32."""
    D = x.shape[-1]
    x = x.contiguous()
    y = y.contiguous()
    g = gate.reshape(-1)[-D:].float().contiguous()
    out = torch.empty_like(x)
    _lib.call("ropeslr_dit_gated_add", x.data_ptr(), y.data_ptr(), g.data_ptr(), x.numel() // D, D, out.data_ptr(),
              _stream(x))
    return out


def heads_to_tokens(a: torch.Tensor) -> torch.Tensor:
    """[B, H, L, dh] bf16 (contiguous) -> [B, L, H * dh]."""
    B, H, L, dh = a.shape
    a = a.contiguous()
    y = torch.empty((B, L, H * dh), dtype=a.dtype, device=a.device)
    _lib.call("ropeslr_dit_heads_to_tokens", a.data_ptr(), B, H, L, dh, y.data_ptr(), _stream(a))
    return y


def sinusoidal(t: torch.Tensor, dim: int) -> torch.Tensor:
    half = dim // 2
    freqs = torch.exp(-math.log(10000.0) * torch.arange(half, dtype=torch.float64, device=t.device) / half)
    a = t.double()[:, None] * freqs[None]
    return torch.cat([torch.cos(a), torch.sin(a)], dim=1).float()


class WanBlock(nn.Module):
    def __init__(self, cfg: WanConfig):
        super().__init__()
        D = cfg.dim
        self.cfg = cfg
        self.norm1 = nn.LayerNorm(D, eps=cfg.eps, elementwise_affine=False)
        self.q, self.k, self.v, self.o = (nn.Linear(D, D) for _ in range(4))
        self.norm_q, self.norm_k = RMSNorm(D, cfg.eps), RMSNorm(D, cfg.eps)
        self.norm3 = nn.LayerNorm(D, eps=cfg.eps, elementwise_affine=True)
        self.cq, self.ck, self.cv, self.co = (nn.Linear(D, D) for _ in range(4))
        self.norm_cq, self.norm_ck = RMSNorm(D, cfg.eps), RMSNorm(D, cfg.eps)
        self.norm2 = nn.LayerNorm(D, eps=cfg.eps, elementwise_affine=False)
        self.ffn1, self.ffn2 = nn.Linear(D, cfg.ffn), nn.Linear(cfg.ffn, D)
        self.modulation = nn.Parameter(torch.randn(1, 6, D) / math.sqrt(D))
        # the RoPeSLR parameter set of this layer (mechanism.py:100-133)
        H, d, r = cfg.heads, cfg.head_dim, cfg.rank
        self.w_a = nn.Parameter(torch.randn(H, d, r) / math.sqrt(d))
        self.w_b = nn.Parameter(torch.randn(H, r, d) / math.sqrt(r))
        self.alpha = nn.Parameter(torch.full((D,), 0.1))
        self.w_g = nn.Parameter(torch.randn(D) * 0.02)
        self.rms_sparse = nn.Parameter(torch.ones(d))
        self.rms_lowrank = nn.Parameter(torch.ones(d))

    def qkv_weights(self):
        """[W_q; W_k; W_v] and their biases concatenated for one projection
        GEMM, kept while the three layers' parameters are unchanged."""
        src = (self.q.weight, self.k.weight, self.v.weight, self.q.bias, self.k.bias, self.v.bias)
        key = tuple((p.data_ptr(), p._version) for p in src)
        if getattr(self, "_qkv_key", None) != key:
            with torch.no_grad():
                self._qkv = (torch.cat(src[:3], 0).contiguous(), torch.cat(src[3:], 0).contiguous())
            self._qkv_key = key
        return self._qkv

    def ropeslr_params(self) -> MechanismParams:
        """The layer's float32 RoPeSLR parameter set, converted once and kept
        while the parameters are unchanged (storage and version counters), so
        the op's parameter-only tables (mechanism.lowrank_tables) are built
        once per layer rather than on every step."""
        src = (self.w_a, self.w_b, self.alpha, self.w_g, self.rms_sparse, self.rms_lowrank)
        key = tuple((p.data_ptr(), p._version, p.dtype) for p in src)
        if getattr(self, "_mp_key", None) != key:
            f = lambda t: t.detach().float().contiguous()  # noqa: E731
            self._mp = MechanismParams(w_a=f(self.w_a), w_b=f(self.w_b), alpha=f(self.alpha), w_g=f(self.w_g),
                                       b_g=-2.0, rms_sparse=f(self.rms_sparse), rms_lowrank=f(self.rms_lowrank))
            self._mp_key = key
        return self._mp

    def forward(self, x, e, ctx, grid: GridShape, pe: PETables, settings: ForwardSettings, rope: RopeConfig,
                group=None):
        cfg = self.cfg
        B, Lr, D = x.shape
        H, d = cfg.heads, cfg.head_dim
        sh_a, sc_a, g_a, sh_f, sc_f, g_f = (self.modulation + e).chunk(6, dim=1)
        if FUSED_OPS and B == 1 and x.dtype == torch.bfloat16 and x.is_cuda:
            return self._forward_fused(x, (sh_a, sc_a, g_a, sh_f, sc_f, g_f), ctx, grid, pe, settings, rope, group)
        y = (self.norm1(x.float()) * (1 + sc_a) + sh_a).to(x.dtype)
        q = self.norm_q(self.q(y)).view(B, Lr, H, d)
        k = self.norm_k(self.k(y)).view(B, Lr, H, d)
        v = self.v(y).view(B, Lr, H, d)
        params = self.ropeslr_params()
        if group is not None:
            a = ulysses_attention(q, k, v, y, grid, params, settings, pe, group=group, rope=rope)
        else:
            qh, kh, vh = (t.permute(0, 2, 1, 3).contiguous() for t in (q, k, v))
            a = forward(qh, kh, vh, y.contiguous(), grid, params, settings, pe, rope=rope)
        x = x + (self.o(a).float() * g_a).to(x.dtype)
        # cross-attention to the text tokens
        c = self.norm3(x)
        cq = self.norm_cq(self.cq(c)).view(B, Lr, H, d).transpose(1, 2)
        ck = self.norm_ck(self.ck(ctx)).view(B, -1, H, d).transpose(1, 2)
        cv = self.cv(ctx).view(B, -1, H, d).transpose(1, 2)
        ca = F.scaled_dot_product_attention(cq, ck, cv).transpose(1, 2).reshape(B, Lr, D)
        x = x + self.co(ca)
        y = (self.norm2(x.float()) * (1 + sc_f) + sh_f).to(x.dtype)
        x = x + (self.ffn2(F.gelu(self.ffn1(y), approximate="tanh")).float() * g_f).to(x.dtype)
        return x

    def _forward_fused(self, x, mods, ctx, grid, pe, settings, rope, group):
        """The same block with the token-wise ops fused (csrc/dit_ops.cu):
        modulated and affine LayerNorms, Q/K RMSNorm written straight into
        the op's head-major layout, gated residuals (the first out of place,
        so the caller's x is left alone, the second in place), the
        cross-attention output back to token-major rows."""
        cfg = self.cfg
        B, Lr, D = x.shape
        H, d = cfg.heads, cfg.head_dim
        sh_a, sc_a, g_a, sh_f, sc_f, g_f = mods
        y = ln_modulate(x, sh_a, sc_a, cfg.eps)
        params = self.ropeslr_params()
        hm = group is None  # the Ulysses wrapper takes token-major [B, L_r, H, d]
        # Q, K, V in one GEMM (N = 3D), the RMSNorms read its column slices
        w_qkv, b_qkv = self.qkv_weights()
        qkv = F.linear(y, w_qkv, b_qkv)
        q = rms_heads(qkv[..., :D], self.norm_q.weight, self.norm_q.eps, H, head_major=hm)
        k = rms_heads(qkv[..., D:2 * D], self.norm_k.weight, self.norm_k.eps, H, head_major=hm)
        v = rms_heads(qkv[..., 2 * D:], None, 0.0, H, head_major=hm)
        if group is not None:
            a = ulysses_attention(q, k, v, y, grid, params, settings, pe, group=group, rope=rope)
        else:
            a = forward(q, k, v, y, grid, params, settings, pe, rope=rope)
        x = gated_add(x, self.o(a), g_a)  # a new tensor: the caller's x is not modified
        # cross-attention to the text tokens
        c = ln_affine(x, self.norm3)
        cq = rms_heads(self.cq(c), self.norm_cq.weight, self.norm_cq.eps, H)
        ck = self.norm_ck(self.ck(ctx)).view(B, -1, H, d).transpose(1, 2)
        cv = self.cv(ctx).view(B, -1, H, d).transpose(1, 2)
        ca = F.scaled_dot_product_attention(cq, ck, cv)
        ca = heads_to_tokens(ca) if ca.dtype == torch.bfloat16 else ca.transpose(1, 2).reshape(B, Lr, D)
        x += self.co(ca)
        y = ln_modulate(x, sh_f, sc_f, cfg.eps)
        # FFN up-projection with the tanh-GELU in the cuBLASLt epilogue
        h = torch._addmm_activation(self.ffn1.bias, y.view(-1, D), self.ffn1.weight.t(), use_gelu=True)
        gated_residual_(x, self.ffn2(h.view(B, Lr, -1)), g_f)
        return x


class WanDiT(nn.Module):
    """Patch embedding, text / time embeddings, the blocks, the output head."""

    def __init__(self, cfg: WanConfig):
        super().__init__()
        D = cfg.dim
        self.cfg = cfg
        pt, ph, pw = cfg.patch
        self.patch_embed = nn.Linear(cfg.in_channels * pt * ph * pw, D)
        self.text_embed = nn.Sequential(nn.Linear(cfg.text_dim, D), nn.GELU(approximate="tanh"), nn.Linear(D, D))
        self.time_embed = nn.Sequential(nn.Linear(cfg.freq_dim, D), nn.SiLU(), nn.Linear(D, D))
        self.time_proj = nn.Sequential(nn.SiLU(), nn.Linear(D, 6 * D))
        self.blocks = nn.ModuleList(WanBlock(cfg) for _ in range(cfg.blocks))
        self.head_norm = nn.LayerNorm(D, eps=cfg.eps, elementwise_affine=False)
        self.head_mod = nn.Parameter(torch.randn(1, 2, D) / math.sqrt(D))
        self.head = nn.Linear(D, cfg.in_channels * pt * ph * pw)
        d = cfg.head_dim
        self.rope = RopeConfig(*cfg.rope_split)
        # learnable 3D absolute PE of RoPeSLR, per-axis tables (shared by the blocks)
        self.pe_tables = None

    def patchify(self, latent: torch.Tensor):
        """[B, C, T, Hh, Ww] -> tokens [B, L, C*pt*ph*pw] and the token grid."""
        B, C, T, Hh, Ww = latent.shape
        pt, ph, pw = self.cfg.patch
        g = GridShape(T // pt, Hh // ph, Ww // pw)
        x = latent.view(B, C, g.t, pt, g.h, ph, g.w, pw).permute(0, 2, 4, 6, 1, 3, 5, 7)
        return x.reshape(B, g.size, C * pt * ph * pw), g

    def forward(self, latent, t, text, group=None):
        cfg = self.cfg
        tokens, grid = self.patchify(latent)
        world, rank = (torch.distributed.get_world_size(group), torch.distributed.get_rank(group)) if group else (1, 0)
        a, b = seq_slice(grid.size, world, rank)
        x = self.patch_embed(tokens[:, a:b])
        ctx = self.text_embed(text)
        e0 = self.time_embed(sinusoidal(t, cfg.freq_dim).to(x.dtype))
        e = self.time_proj(e0).view(-1, 6, cfg.dim).float()
        if self.pe_tables is None or self.pe_tables.pe_t.shape[0] != grid.t:
            gen = torch.Generator(device=x.device).manual_seed(1234)
            self.pe_tables = PETables(*(torch.randn((n, cfg.dim), generator=gen, device=x.device) * 0.02
                                        for n in grid.as_tuple()))
        nb = -(-grid.size // cfg.block)
        settings = ForwardSettings(SparseSettings(block=cfg.block, topk=SparseSettings.topk_for_sparsity(nb, cfg.sparsity)))
        for blk in self.blocks:
            x = blk(x, e, ctx, grid, self.pe_tables, settings, self.rope, group=group)
        sh, sc = (self.head_mod + e0.float()[:, None]).chunk(2, dim=1)
        return self.head((self.head_norm(x.float()) * (1 + sc) + sh).to(x.dtype))


def make_model(cfg: Optional[WanConfig] = None, device="cuda", dtype=torch.bfloat16, seed=0) -> WanDiT:
    torch.manual_seed(seed)
    m = WanDiT(cfg or WanConfig())
    for mod in m.modules():
        if isinstance(mod, nn.Linear):
            nn.init.normal_(mod.weight, std=0.02)
            nn.init.zeros_(mod.bias)
    return m.to(device=device, dtype=dtype).eval()
