"""CPU oracle for the RoPeSLR attention forward -- TEST INFRASTRUCTURE ONLY.

This module is a float64 NumPy restatement of the reference package's hot
path (``/root/reference/pkg/src/ropeslr``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it, and only as the checker or as the timed CPU reference -- the
product path (``paper_2605_20659_b200``) never calls into it.

Every function cites the reference lines it follows.  Three deliberate,
documented extensions let it cover the
BASELINE configs that the reference's 3-D tiling cannot express:

  (i)   flat contiguous blocks of ``block`` tokens with a ragged last block;
        padding tokens never exist (L is not padded), so they are excluded
        from pooling, keys and outputs by construction;
  (ii)  the inputs are the already-rotated (post-RoPE, post-cast) Q/K, so
        the rotation inside ``block_sparse_attention`` is not repeated;
  (iii) a fixed ``topk`` rule ``order[:k]`` as an alternative to the
        cumulative-mass ``keep`` rule (``count_for_mass``).

Pinning: ``tests/test_oracle.py`` checks this module against golden vectors
produced by the unmodified reference functions (``oracle/make_golden.py``)
and, when ``/root/reference`` is present, against the live reference.
"""

from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

RMS_EPS = 1e-6            # mechanism.py:24
MASS_SLACK = 1e-12        # decomposition.py:102
LINEAR_FLOOR = 1e-8       # mechanism.py:347


# ---------------------------------------------------------------------------
# elementwise helpers


def sigmoid(x):
    """Stable logistic; mechanism.py:27-30."""
    x = np.asarray(x, dtype=np.float64)
    t = np.exp(-np.abs(x))
    return np.where(x >= 0.0, 1.0 / (1.0 + t), t / (1.0 + t))


def elu_plus_one(x):
    """phi(x) = elu(x) + 1; mechanism.py:33-36."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x > 0.0, x + 1.0, np.exp(np.minimum(x, 0.0)))


def count_for_mass(sorted_desc: np.ndarray, target: float) -> int:
    """Smallest leading count whose cumulative sum reaches target - 1e-12,
    never fewer than one; decomposition.py:105-111."""
    csum = np.cumsum(sorted_desc)
    reached = csum >= target - MASS_SLACK
    if not np.any(reached):
        return int(sorted_desc.size)
    return int(np.argmax(reached)) + 1


def topk_for_sparsity(n_blocks: int, sparsity: float) -> int:
    """k = floor((1 - S) * nb + 1/2), at least 1 (SURVEY.md section 8 table:
    reproduces top-51 of 512 at S = 0.9)."""
    return max(1, int(math.floor((1.0 - sparsity) * n_blocks + 0.5)))


# ---------------------------------------------------------------------------
# 3D grid / RoPE (used to build inputs; the op consumes post-RoPE tensors)


def grid_coords(t: int, h: int, w: int) -> np.ndarray:
    """(L, 3) coordinates of flat index p = t*H*W + x*W + y; rope3d.py:82-88."""
    p = np.arange(t * h * w)
    frame = h * w
    return np.stack([p // frame, (p % frame) // w, p % w], axis=1)


def rope_slots(split: Sequence[int], base: float = 10000.0) -> Tuple[np.ndarray, np.ndarray]:
    """Pair frequencies and axis index in (axis, m) order; rope3d.py:102-119."""
    thetas, axis_idx = [], []
    for ai, d_k in enumerate(split):
        for m in range(1, d_k // 2 + 1):
            thetas.append(float(base ** (-2.0 * (m - 1) / d_k)))
            axis_idx.append(ai)
    return np.asarray(thetas), np.asarray(axis_idx, dtype=np.int64)


def rotate_rows(m: np.ndarray, grid: Sequence[int], split: Sequence[int],
                base: float = 10000.0) -> np.ndarray:
    """Rotate row p by the composite rotation at position p, pairs at columns
    (2j, 2j+1); rope3d.py:122-143."""
    m = np.asarray(m, dtype=np.float64)
    thetas, axis_idx = rope_slots(split, base)
    ang = grid_coords(*grid)[:, axis_idx] * thetas[None, :]
    c, s = np.cos(ang), np.sin(ang)
    even, odd = m[..., 0::2], m[..., 1::2]
    out = np.empty_like(m)
    out[..., 0::2] = c * even - s * odd
    out[..., 1::2] = s * even + c * odd
    return out


# ---------------------------------------------------------------------------
# block partitions


def flat_block_members(L: int, block: int) -> List[np.ndarray]:
    """Extension (i): contiguous blocks of `block` tokens, last one ragged.
    Equals mechanism._block_ids (mechanism.py:280-287) whenever a 3D tile
    (1, b_x, b_y) spans whole rows of the grid."""
    nb = (L + block - 1) // block
    return [np.arange(b * block, min(L, (b + 1) * block)) for b in range(nb)]


def tile_block_members(grid: Sequence[int], block: Sequence[int]) -> List[np.ndarray]:
    """3D tile blocks exactly as mechanism._block_ids (mechanism.py:280-287)
    and the member lists of mechanism.py:306."""
    t, h, w = grid
    b_t, b_x, b_y = block
    if t % b_t or h % b_x or w % b_y:
        raise ValueError(f"block dims {tuple(block)} do not divide grid {tuple(grid)}")
    n_x, n_y = h // b_x, w // b_y
    c = grid_coords(t, h, w)
    ids = (c[:, 0] // b_t) * (n_x * n_y) + (c[:, 1] // b_x) * n_y + (c[:, 2] // b_y)
    nb = (t // b_t) * n_x * n_y
    return [np.flatnonzero(ids == b) for b in range(nb)]


# ---------------------------------------------------------------------------
# block-sparse branch (mechanism.py:290-328)


def block_scores(rq: np.ndarray, rk: np.ndarray, members: List[np.ndarray]) -> np.ndarray:
    """Mean-pooled block scores / sqrt(d); mechanism.py:306-309."""
    rq = np.asarray(rq, dtype=np.float64)
    rk = np.asarray(rk, dtype=np.float64)
    d = rq.shape[1]
    pooled_q = np.stack([rq[m].mean(axis=0) for m in members])
    pooled_k = np.stack([rk[m].mean(axis=0) for m in members])
    return (pooled_q @ pooled_k.T) / math.sqrt(d)


def block_probs(scores: np.ndarray) -> np.ndarray:
    """Row softmax of the block scores; mechanism.py:310-311."""
    probs = np.exp(scores - scores.max(axis=1, keepdims=True))
    probs /= probs.sum(axis=1, keepdims=True)
    return probs


def select_blocks(scores: np.ndarray, keep: Optional[float] = None,
                  topk: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """Selection mask (nb, nb) bool and per-row counts.

    keep mode follows mechanism.py:316-320 (stable argsort of -probs, then
    count_for_mass); topk mode (extension iii) keeps order[:k] of the same
    stable ordering (ties to the lower block index)."""
    if (keep is None) == (topk is None):
        raise ValueError("exactly one of keep / topk must be given")
    probs = block_probs(scores)
    nb = scores.shape[0]
    selected = np.zeros((nb, nb), dtype=bool)
    counts = np.zeros(nb, dtype=np.int64)
    for qb in range(nb):
        order = np.argsort(-probs[qb], kind="stable")
        if topk is not None:
            n_keep = min(int(topk), nb)
        else:
            n_keep = count_for_mass(probs[qb][order], keep)
        selected[qb, order[:n_keep]] = True
        counts[qb] = n_keep
    return selected, counts


def decision_margin(scores: np.ndarray, counts: np.ndarray) -> np.ndarray:
    """Per-row gap between the last kept and the first dropped block score
    (inf when every block is kept).  A mask flip between two fp
    implementations needs a score error larger than this gap."""
    nb = scores.shape[0]
    out = np.full(nb, np.inf)
    for qb in range(nb):
        k = int(counts[qb])
        if k >= nb:
            continue
        srt = np.sort(scores[qb])[::-1]
        out[qb] = srt[k - 1] - srt[k]
    return out


def attend_selected(rq: np.ndarray, rk: np.ndarray, v: np.ndarray, members: List[np.ndarray],
                    selected: np.ndarray, qblocks: Optional[Sequence[int]] = None,
                    out: Optional[np.ndarray] = None) -> Tuple[np.ndarray, int]:
    """Exact softmax attention of each query block over the concatenated
    tokens of its selected key blocks in ascending block order;
    mechanism.py:321-326.  Returns (output (L, d), attended pairs)."""
    rq = np.asarray(rq, dtype=np.float64)
    rk = np.asarray(rk, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    L, d = rq.shape
    if out is None:
        out = np.zeros((L, v.shape[1]))
    scale = math.sqrt(d)
    attended = 0
    nb = len(members)
    for qb in (range(nb) if qblocks is None else qblocks):
        chosen = np.flatnonzero(selected[qb])
        keys = np.concatenate([members[b] for b in chosen])
        qtok = members[qb]
        s = (rq[qtok] @ rk[keys].T) / scale
        e = np.exp(s - s.max(axis=1, keepdims=True))
        out[qtok] = (e / e.sum(axis=1, keepdims=True)) @ v[keys]
        attended += qtok.size * keys.size
    return out, attended


def block_sparse_attention(rq, rk, v, members, keep=None, topk=None):
    """Whole sparse branch for one head: (output (L,d), selected, sparsity,
    scores, counts); mechanism.py:290-328 with extensions (i)-(iii)."""
    scores = block_scores(rq, rk, members)
    selected, counts = select_blocks(scores, keep=keep, topk=topk)
    out, attended = attend_selected(rq, rk, v, members, selected)
    L = rq.shape[0]
    return out, selected, 1.0 - attended / float(L) ** 2, scores, counts


def attended_pairs(members: List[np.ndarray], selected: np.ndarray) -> int:
    """sum_qb |qtok| * |keys| without running attention; mechanism.py:326."""
    sizes = np.array([m.size for m in members], dtype=np.int64)
    return int((sizes[:, None] * (selected.astype(np.int64) * sizes[None, :])).sum())


# ---------------------------------------------------------------------------
# PE, compensators, gate, RMSNorm, fusion (mechanism.py:183-255, 350-362, 411-453)


def pe_from_axis_tables(grid: Sequence[int], pe_t, pe_x, pe_y) -> np.ndarray:
    """PE[p] = P_t[t] + P_x[x] + P_y[y] (the kernel's parameterisation; the
    reference's build_pe3d table is the special case of
    sinusoidal_axis_tables)."""
    c = grid_coords(*grid)
    return (np.asarray(pe_t, np.float64)[c[:, 0]] + np.asarray(pe_x, np.float64)[c[:, 1]]
            + np.asarray(pe_y, np.float64)[c[:, 2]])


def sinusoidal_axis_tables(grid: Sequence[int], d_model: int, split: Sequence[int],
                           base: float = 10000.0):
    """Per-axis decomposition of build_pe3d (mechanism.py:183-209): each axis
    table is non-zero only on its own column block, interleaved (sin, cos)
    of theta_m * coord with theta_m = base^(-2(m-1)/width)."""
    d_h = sum(split)
    if d_model % d_h:
        raise ValueError(f"d_model={d_model} is not a multiple of the head dim {d_h}")
    sizes = tuple(grid)
    tables = []
    col = 0
    for ai, d_k in enumerate(split):
        numer = d_model * d_k
        if numer % d_h:
            raise ValueError(f"axis block width {numer}/{d_h} is not an integer")
        width = numer // d_h
        if width % 2:
            raise ValueError(f"axis block width {width} must be even")
        tab = np.zeros((sizes[ai], d_model))
        c = np.arange(sizes[ai], dtype=np.float64)
        for m in range(1, width // 2 + 1):
            theta = base ** (-2.0 * (m - 1) / width)
            tab[:, col] = np.sin(theta * c)
            tab[:, col + 1] = np.cos(theta * c)
            col += 2
        tables.append(tab)
    return tuple(tables)


def rms_norm(o, scale, eps: float = RMS_EPS) -> np.ndarray:
    """o / sqrt(mean(o^2) + eps) * scale; mechanism.py:238-246, 411-414."""
    o = np.asarray(o, dtype=np.float64)
    inv = 1.0 / np.sqrt(np.mean(o * o, axis=1, keepdims=True) + eps)
    return o * inv * np.asarray(scale, np.float64)[None, :]


def gate(x_hat, w_g, b_g) -> np.ndarray:
    """g = sigmoid(x_hat @ w_g + b_g); mechanism.py:249-255, 434-435."""
    return sigmoid(np.asarray(x_hat, np.float64) @ np.asarray(w_g, np.float64) + b_g)


def lowrank_compensator(x_hat, w_a, w_b, head: int) -> np.ndarray:
    """sigmoid(sigmoid(x_hat_h @ W_A[h]) @ W_B[h]); mechanism.py:225-235, 441-446."""
    d = w_a.shape[1]
    xh = np.asarray(x_hat, np.float64)[:, head * d:(head + 1) * d]
    return sigmoid(sigmoid(xh @ np.asarray(w_a[head], np.float64)) @ np.asarray(w_b[head], np.float64))


def linear_state(k_lin, v_lin) -> Tuple[np.ndarray, np.ndarray]:
    """S = phi(k)^T v, z = sum phi(k); mechanism.py:354-357."""
    pk = elu_plus_one(k_lin)
    return pk.T @ np.asarray(v_lin, np.float64), pk.sum(axis=0)


def linear_apply(q_lin, smat, svec) -> np.ndarray:
    """phi(q) S / max(phi(q) . z, 1e-8); mechanism.py:354-361."""
    pq = elu_plus_one(q_lin)
    denom = np.maximum(pq @ svec, LINEAR_FLOOR)
    return (pq @ smat) / denom[:, None]


def linear_compensator(x_hat, w_q, w_k, w_v, head: int) -> np.ndarray:
    """Linear-attention compensator of one head from the backbone projections
    of x_hat (no RoPE); mechanism.py:350-362."""
    x_hat = np.asarray(x_hat, np.float64)
    q = x_hat @ np.asarray(w_q[head], np.float64)
    k = x_hat @ np.asarray(w_k[head], np.float64)
    v = x_hat @ np.asarray(w_v[head], np.float64)
    smat, svec = linear_state(k, v)
    return linear_apply(q, smat, svec)


def fused_forward(x, sparse_out, pe, params: dict, compensator: str = "lowrank",
                  use_pe: bool = True, eps: float = RMS_EPS, backbone: Optional[dict] = None,
                  lin_proj: Optional[Sequence[Tuple[np.ndarray, np.ndarray, np.ndarray]]] = None):
    """mechanism._fused_forward (mechanism.py:426-453).

    params: dict with w_a (H,d,r), w_b (H,r,d), alpha (D,), w_g (D,), b_g,
    rms_sparse (d,), rms_lowrank (d,).  For compensator == "linear" either
    `backbone` (w_q, w_k, w_v of shape (H, D, d)) or precomputed per-head
    projections `lin_proj` [(q, k, v)] must be given.
    Returns dict(x_hat, g, o_lowrank (H,L,d), norm_sparse, norm_lowrank, output (L,D))."""
    x = np.asarray(x, np.float64)
    H = len(sparse_out)
    d = sparse_out[0].shape[1]
    alpha = np.asarray(params["alpha"], np.float64)
    x_hat = x + alpha[None, :] * np.asarray(pe, np.float64) if use_pe else x
    g = sigmoid(x_hat @ np.asarray(params["w_g"], np.float64) + float(params["b_g"]))
    out = np.empty((x.shape[0], H * d))
    o_lr_all, ysp_all, ylr_all = [], [], []
    for h in range(H):
        y_sp = rms_norm(sparse_out[h], params["rms_sparse"], eps)
        if compensator == "lowrank":
            o_lr = lowrank_compensator(x_hat, params["w_a"], params["w_b"], h)
        elif compensator == "linear":
            if lin_proj is not None:
                q, k, v = lin_proj[h]
                smat, svec = linear_state(k, v)
                o_lr = linear_apply(q, smat, svec)
            else:
                o_lr = linear_compensator(x_hat, backbone["w_q"], backbone["w_k"], backbone["w_v"], h)
        else:
            raise ValueError(f"unknown compensator {compensator!r}")
        y_lr = rms_norm(o_lr, params["rms_lowrank"], eps)
        out[:, h * d:(h + 1) * d] = y_sp + g[:, None] * y_lr
        o_lr_all.append(o_lr)
        ysp_all.append(y_sp)
        ylr_all.append(y_lr)
    return dict(x_hat=x_hat, g=g, o_lowrank=np.stack(o_lr_all), norm_sparse=np.stack(ysp_all),
                norm_lowrank=np.stack(ylr_all), output=out)


# ---------------------------------------------------------------------------
# Stage-I backward (mechanism.py:411-423, 456-488, 519-565): gradients of the
# alignment loss w.r.t. the new parameter set, the sparse branch constant.


def rms_backward(d_y, o, scale, eps: float = RMS_EPS):
    """mechanism._rms_backward (mechanism.py:417-423) with the cache of
    mechanism._rms_cache (mechanism.py:411-414) recomputed from o."""
    o = np.asarray(o, np.float64)
    inv = 1.0 / np.sqrt(np.mean(o * o, axis=1, keepdims=True) + eps)
    u = o * inv
    d_scale = np.sum(d_y * u, axis=0)
    d_u = d_y * np.asarray(scale, np.float64)[None, :]
    dot = np.sum(d_u * o, axis=1, keepdims=True)
    d_o = d_u * inv - o * (inv ** 3 * dot / o.shape[1])
    return d_o, d_scale


def fused_backward(g_out, x, sparse_out, pe, params: dict, use_pe: bool = True, eps: float = RMS_EPS) -> dict:
    """mechanism._fused_backward (mechanism.py:456-488), low-rank compensator:
    d loss / d output = g_out (L, D) -> gradients of w_a, w_b, alpha, w_g, b_g,
    rms_sparse, rms_lowrank (same names and shapes as the parameters)."""
    x = np.asarray(x, np.float64)
    H = len(sparse_out)
    d = sparse_out[0].shape[1]
    w_a = np.asarray(params["w_a"], np.float64)
    w_b = np.asarray(params["w_b"], np.float64)
    w_g = np.asarray(params["w_g"], np.float64)
    alpha = np.asarray(params["alpha"], np.float64)
    x_hat = x + alpha[None, :] * np.asarray(pe, np.float64) if use_pe else x
    g = sigmoid(x_hat @ w_g + float(params["b_g"]))
    grads = {n: np.zeros_like(np.asarray(params[n], np.float64)) for n in
             ("w_a", "w_b", "alpha", "w_g", "rms_sparse", "rms_lowrank")}
    grads["b_g"] = 0.0
    d_g = np.zeros(x.shape[0])
    d_xhat = np.zeros_like(x_hat)
    for h in range(H):
        gh = np.asarray(g_out, np.float64)[:, h * d:(h + 1) * d]
        _, d_rs = rms_backward(gh, sparse_out[h], params["rms_sparse"], eps)
        grads["rms_sparse"] += d_rs
        xh = x_hat[:, h * d:(h + 1) * d]
        h1 = sigmoid(xh @ w_a[h])
        o_lr = sigmoid(h1 @ w_b[h])
        y_lr = rms_norm(o_lr, params["rms_lowrank"], eps)
        d_g += np.sum(gh * y_lr, axis=1)
        d_o_lr, d_rl = rms_backward(gh * g[:, None], o_lr, params["rms_lowrank"], eps)
        grads["rms_lowrank"] += d_rl
        d_z2 = d_o_lr * o_lr * (1.0 - o_lr)
        grads["w_b"][h] += h1.T @ d_z2
        d_z1 = (d_z2 @ w_b[h].T) * h1 * (1.0 - h1)
        grads["w_a"][h] += xh.T @ d_z1
        d_xhat[:, h * d:(h + 1) * d] += d_z1 @ w_a[h].T
    d_zg = d_g * g * (1.0 - g)
    grads["w_g"] += x_hat.T @ d_zg
    grads["b_g"] += float(d_zg.sum())
    d_xhat += np.outer(d_zg, w_g)
    if use_pe:
        grads["alpha"] += np.sum(d_xhat * np.asarray(pe, np.float64), axis=0)
    return grads


def align_loss_and_grads(x, sparse_out, pe, target, params: dict, use_pe: bool = True, eps: float = RMS_EPS):
    """One sample of mechanism._loss_and_grads (mechanism.py:552-565): mean
    squared error against the target and its parameter gradients."""
    out = fused_forward(x, sparse_out, pe, params, use_pe=use_pe, eps=eps)["output"]
    diff = out - np.asarray(target, np.float64)
    loss = float(np.mean(diff * diff))
    return loss, fused_backward(2.0 * diff / diff.size, x, sparse_out, pe, params, use_pe, eps)


# ---------------------------------------------------------------------------
# flops accounting (flops.py:30-63)


def flops_sparse(attended_total: float, d: int) -> float:
    """4 * d * attended pairs == flops.c_sparse at S = 1 - attended/L^2."""
    return 4.0 * d * attended_total


def flops_lowrank(B: int, H: int, L: int, d: int, r: int) -> float:
    return 4.0 * B * H * L * d * r        # flops.py:39-40


def flops_fusion(B: int, H: int, L: int, d: int) -> float:
    return 2.0 * B * H * L * d            # flops.py:43-44


def flops_linear_branch(B: int, H: int, L: int, d: int) -> float:
    return 4.0 * B * H * L * d * d        # flops.py:47-48
