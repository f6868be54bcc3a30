"""3D grid / rotary configuration types and the caller-side RoPE.

Mirrors the reference's ``rope3d.RopeConfig`` / ``rope3d.GridShape``
(rope3d.py:25-99) so reference users keep their config objects, and gives a
device-side ``rotate_rows`` (rope3d.py:122-143) for callers that hold
un-rotated projections.  The attention op itself consumes post-RoPE Q/K
(the drop-in boundary); rotation is the caller's step.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

import numpy as np
import torch

AXES = ("t", "x", "y")


@dataclass(frozen=True)
class RopeConfig:
    """Per-axis head-dimension split [t | x | y] (rope3d.py:25-62)."""

    d_t: int
    d_x: int
    d_y: int
    base: float = 10000.0

    def __post_init__(self):
        for name, d in (("d_t", self.d_t), ("d_x", self.d_x), ("d_y", self.d_y)):
            if d < 0 or d % 2 != 0:
                raise ValueError(f"{name} must be an even non-negative count, got {d}")
        if self.d_h < 2:
            raise ValueError("total head dimension must be at least 2")
        if not (np.isfinite(self.base) and self.base > 0.0):
            raise ValueError(f"frequency base must be a positive real, got {self.base}")

    @property
    def d_h(self) -> int:
        return self.d_t + self.d_x + self.d_y

    def axis_dim(self, axis: str) -> int:
        if axis not in AXES:
            raise ValueError(f"unknown axis {axis!r}, expected one of {AXES}")
        return {"t": self.d_t, "x": self.d_x, "y": self.d_y}[axis]

    @property
    def split(self) -> Tuple[int, int, int]:
        return (self.d_t, self.d_x, self.d_y)


@dataclass(frozen=True)
class GridShape:
    """T frames of H x W tokens, flattened p = t*H*W + x*W + y (rope3d.py:65-99)."""

    t: int
    h: int
    w: int

    def __post_init__(self):
        if min(self.t, self.h, self.w) < 1:
            raise ValueError(f"grid dimensions must be positive, got {(self.t, self.h, self.w)}")

    @property
    def size(self) -> int:
        return self.t * self.h * self.w

    def coords(self, device=None) -> torch.Tensor:
        """(L, 3) int64 (t, x, y) of every flat index (rope3d.py:82-88)."""
        p = torch.arange(self.size, device=device)
        frame = self.h * self.w
        return torch.stack([p // frame, (p % frame) // self.w, p % self.w], dim=1)

    def as_tuple(self) -> Tuple[int, int, int]:
        return (self.t, self.h, self.w)


def pair_angles(grid: GridShape, cfg: RopeConfig, device=None) -> torch.Tensor:
    """(L, d_h/2) float64 angle coord_axis * base^(-2(m-1)/d_axis) per pair,
    pairs in (axis, m) order (rope3d.py:102-124)."""
    thetas, axis_idx = [], []
    for ai, axis in enumerate(AXES):
        d_k = cfg.axis_dim(axis)
        for m in range(1, d_k // 2 + 1):
            thetas.append(float(cfg.base ** (-2.0 * (m - 1) / d_k)))
            axis_idx.append(ai)
    th = torch.tensor(thetas, dtype=torch.float64, device=device)
    ax = torch.tensor(axis_idx, dtype=torch.long, device=device)
    return grid.coords(device).to(torch.float64)[:, ax] * th[None, :]


def rotate_rows(m: torch.Tensor, grid: GridShape, cfg: RopeConfig) -> torch.Tensor:
    """Rotate row p of a (..., L, d_h) tensor by the composite rotation at p,
    pairs (2j, 2j+1), in float64 (rope3d.py:127-143).  Returns float64."""
    if m.shape[-2:] != (grid.size, cfg.d_h):
        raise ValueError(f"expected trailing shape {(grid.size, cfg.d_h)}, got {tuple(m.shape[-2:])}")
    ang = pair_angles(grid, cfg, m.device)
    c, s = torch.cos(ang), torch.sin(ang)
    m64 = m.to(torch.float64)
    even, odd = m64[..., 0::2], m64[..., 1::2]
    out = torch.empty_like(m64)
    out[..., 0::2] = c * even - s * odd
    out[..., 1::2] = s * even + c * odd
    return out
