"""Error anatomy of the sparse branch at the config-1 shape: o_sparse (float32
out of K2) against the float64 oracle on sampled query blocks, split into
the tcgen05 fixed-exponent kernel, the running-max kernel and the CUDA-core
kernel; quantiles of |err| / rms(o) per row."""
import sys
sys.path[:0] = ['.', 'tests', 'oracle']
import numpy as np
import torch
import paper_2605_20659_b200 as P
import gpu_helpers as G
import restated as R

q, k, v, x, params, pe, grid = G.make_full_inputs((21, 30, 52), 12, 128, (44, 42, 42), 64, seed=0)
L = grid.size
st = P.ForwardSettings(P.SparseSettings.for_sparsity(64, L, 0.9))
members = R.flat_block_members(L, 64)
rng = np.random.default_rng(3)
res = {}
for mode in ("fixed", "online", "simt"):
    opt = P._lib.option("k2_online", 1 if mode == "online" else 0)
    with opt:
        tr = P.forward(q, k, v, x, grid, params, st, pe, trace=True, impl="simt" if mode == "simt" else "auto")
    torch.cuda.synchronize()
    res[mode] = tr.o_sparse[0].cpu().numpy()
for h in (0, 7):
    qh, kh, vh = (t[0, h].double().cpu().numpy() for t in (q, k, v))
    sel, _ = R.select_blocks(R.block_scores(qh, kh, members), topk=st.sparse.topk)
    qbs = sorted(rng.choice(len(members), size=6, replace=False).tolist())
    rows = np.concatenate([members[b] for b in qbs])
    ref = G.oracle_rows(qh, kh, vh, members, sel, qbs)[rows]
    rms = np.sqrt((ref ** 2).mean(-1, keepdims=True))
    for mode, o in res.items():
        e = np.abs(o[h][rows] - ref) / rms
        qs = np.quantile(e, [0.5, 0.9, 0.99, 0.999, 1.0])
        big = np.abs(ref / rms) > 3
        print(f"h{h} {mode:6s} |err|/rms quantiles 50/90/99/99.9/max {np.array2string(qs, precision=5)}  "
              f"std {e.std():.5f}  max at |y|>3: {e[big].max() if big.any() else 0:.5f}", flush=True)
