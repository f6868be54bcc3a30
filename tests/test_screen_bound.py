"""The error bound the K1 screening path assumes (csrc/select.cu, kScreenBound
and its derivation), checked on the CPU: with every operand split into bf16
hi + lo and the three products hi.hi + hi.lo + lo.hi summed in float32, the
screening score differs from the float64 dot product by at most
2^-12 |q| |k|.  The derivation allows the tensor cores a float32 adder with
twice the rounding error of round-to-nearest; here the float32 sums run in
three orders (sequential, pairwise, reversed) on random, large-dynamic-range
and cancelling vectors, and the worst case must sit far inside the bound."""

import numpy as np
import torch

BOUND = 2.0 ** -12
D = 128


def _split(x: np.ndarray):
    t = torch.from_numpy(x)
    hi = t.to(torch.bfloat16).double()
    lo = (t - hi).to(torch.bfloat16).double()
    return hi.numpy(), lo.numpy()


def _approx(q: np.ndarray, k: np.ndarray, order: str) -> float:
    qh, ql = _split(q)
    kh, kl = _split(k)
    terms = np.concatenate([ql * kh, qh * kl, qh * kh]).astype(np.float64)  # bf16 x bf16: exact in float32
    terms32 = terms.astype(np.float32)
    assert np.array_equal(terms32.astype(np.float64), terms)
    if order == "reversed":
        terms32 = terms32[::-1]
    if order == "pairwise":
        v = terms32.copy()
        while len(v) > 1:
            if len(v) % 2:
                v = np.append(v, np.float32(0))
            v = (v[0::2] + v[1::2]).astype(np.float32)
        return float(v[0])
    acc = np.float32(0)
    for t in terms32:
        acc = np.float32(acc + t)
    return float(acc)


def _cases(rng):
    yield "normal", rng.standard_normal(D), rng.standard_normal(D)
    yield "pooled", rng.standard_normal(D) / np.sqrt(128), rng.standard_normal(D) / np.sqrt(128)
    yield "dynamic", rng.standard_normal(D) * np.exp(rng.uniform(-20, 20, D)), rng.standard_normal(D)
    base = rng.standard_normal(D)
    yield "cancel", base, np.concatenate([base[:64], -base[:64]]) + 1e-6 * rng.standard_normal(D)
    yield "aligned", np.abs(rng.standard_normal(D)), np.abs(rng.standard_normal(D))


def test_screen_bound_holds_with_margin():
    rng = np.random.default_rng(0)
    worst = 0.0
    for _ in range(40):
        for name, q, k in _cases(rng):
            exact = float(np.dot(q, k))
            scale = np.linalg.norm(q) * np.linalg.norm(k)
            for order in ("sequential", "pairwise", "reversed"):
                err = abs(_approx(q, k, order) - exact) / scale
                worst = max(worst, err)
                assert err <= BOUND, (name, order, err)
    # the kernel's bound is 2^-12; float32-grade sums sit orders of magnitude inside it
    assert worst < BOUND / 64, worst
