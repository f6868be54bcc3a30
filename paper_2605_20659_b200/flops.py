"""Cost model of the fused attention (flops.py:14-63 of the reference), with
the sparse term taken from the measured attended-pair count."""

from __future__ import annotations


def c_sparse_from_pairs(attended_pairs: float, d_h: int) -> float:
    """4 * d_h * attended pairs == flops.c_sparse at S = 1 - pairs / L^2."""
    return 4.0 * d_h * attended_pairs


def c_full(b: int, h: int, l: int, d_h: int) -> float:
    return 4.0 * b * h * l ** 2 * d_h                     # flops.py:34-36


def c_lowrank(b: int, h: int, l: int, d_h: int, r: int) -> float:
    return 4.0 * b * h * l * d_h * r                      # flops.py:39-40


def c_fusion(b: int, h: int, l: int, d_h: int) -> float:
    return 2.0 * b * h * l * d_h                          # flops.py:43-44


def c_linear_branch(b: int, h: int, l: int, d_h: int) -> float:
    return 4.0 * b * h * l * d_h ** 2                     # flops.py:47-48


def overhead_eta(l: int, s: float, r: int) -> float:
    return (r + 0.5) / (l * (1.0 - s))                    # flops.py:56-59


def total_ropeslr(attended_pairs: float, b: int, h: int, l: int, d_h: int, r: int,
                  compensator: str = "lowrank") -> float:
    """flops.total_ropeslr (flops.py:62-63) with the measured sparse count."""
    comp = c_lowrank(b, h, l, d_h, r) if compensator == "lowrank" else c_linear_branch(b, h, l, d_h)
    return c_sparse_from_pairs(attended_pairs, d_h) + comp + c_fusion(b, h, l, d_h)
