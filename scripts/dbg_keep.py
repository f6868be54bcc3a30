import sys; sys.path[:0]=['.','tests','oracle']
import numpy as np, torch
import paper_2605_20659_b200 as P
from paper_2605_20659_b200 import _lib
import restated as R
nb, block, ragged = 300, 32, 5
g = torch.Generator(device="cuda").manual_seed(nb)
L = nb * block - ragged
q = torch.randn((1, 3, L, 128), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((1, 3, L, 128), generator=g, device="cuda").to(torch.bfloat16)
for keep in (1e-9, 0.3, 0.9, 0.999, 1.0):
    sp = P.SparseSettings(block=block, keep=keep)
    with _lib.option("keep_bitonic", 0):
        a = P.select_blocks(q, k, sp, want_scores=True)
    with _lib.option("keep_bitonic", 1):
        b = P.select_blocks(q, k, sp, want_scores=True)
    torch.cuda.synchronize()
    bad = (a.cnt != b.cnt).nonzero()
    mbad = (a.mask != b.mask).any(-1).nonzero()
    print("keep", keep, "cnt diffs", bad.shape[0], "mask-diff rows", mbad.shape[0], "att", a.attended.tolist(), b.attended.tolist())
    for r in mbad[:3].tolist():
        h, qb = r[1], r[2]
        s = a.scores[0, h, qb].double().cpu().numpy()
        p = np.exp(s - s.max()); p /= p.sum()
        order = np.argsort(-p, kind="stable"); cs = np.cumsum(p[order])
        ca, cb = int(a.cnt[0, h, qb]), int(b.cnt[0, h, qb])
        print("  row", h, qb, "cnt new", ca, "bitonic", cb, "oracle", R.count_for_mass(p[order], keep))
        for j in range(min(ca, cb) - 2, max(ca, cb) + 1):
            if 0 <= j < nb: print("    pos", j, "p", p[order[j]], "cum", cs[j], "cum-target", cs[j] - (keep - 1e-12))
        ma = a.mask[0, h, qb].cpu().numpy(); mb = b.mask[0, h, qb].cpu().numpy()
        print("    only-new", np.nonzero(ma & ~mb)[0][:10], "only-bitonic", np.nonzero(mb & ~ma)[0][:10])
