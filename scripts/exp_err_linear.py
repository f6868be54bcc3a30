"""Error anatomy of the linear compensator (tcgen05, PE in the kernels) at
the config-1 shape: y_lr against the float64 oracle on the kernel's own
bf16 projections, with and without the PE injection."""
import math
import sys
sys.path[:0] = ['.', 'tests', 'oracle']
import numpy as np
import torch
import paper_2605_20659_b200 as P
import gpu_helpers as G
import restated as R
from test_gpu_compensator import _linear_oracle

q, k, v, x, params, pe, grid = G.make_full_inputs((21, 30, 52), 12, 128, (44, 42, 42), 64, seed=4)
H, d, L = 12, 128, grid.size
D = H * d
gen = torch.Generator(device="cuda").manual_seed(9)
W = [torch.randn((H, D, d), generator=gen, device="cuda") / math.sqrt(D) for _ in range(3)]
lin = tuple(torch.einsum("bld,hde->bhle", x.double(), w.double()).to(torch.bfloat16).contiguous() for w in W)
rms = params.rms_lowrank.double().cpu().numpy()
for use_pe in (True, False):
    st = P.ForwardSettings(P.SparseSettings.for_sparsity(64, L, 0.9), compensator="linear", use_pe=use_pe)
    y_lr, o_lr, g, state = P.compensator_branch(x, grid, params, st, pe, lin_proj=lin, lin_weights=W, want_o_lr=True,
                                                want_state=True)
    torch.cuda.synchronize()
    for h in (0, 11):
        o, smat, svec, g_ref = _linear_oracle(x, params, pe, (21, 30, 52), W, lin, use_pe, 0, h)
        y = o / np.sqrt((o ** 2).mean(-1, keepdims=True) + st.rms_eps) * rms
        e = np.abs(y_lr[0, :, h].double().cpu().numpy() - y)
        e32 = np.abs(o_lr[0, h].double().cpu().numpy() - o) / np.sqrt((o ** 2).mean(-1, keepdims=True))
        sd = state[h].double().cpu().numpy()
        es = np.abs(sd[:, :128] - smat).max() / np.abs(smat).max()
        ez = np.abs(sd[:, 128] - svec).max() / np.abs(svec).max()
        print(f"use_pe={use_pe} h{h}: y_lr |err| q50/99/99.9/max {np.quantile(e, [0.5, 0.99, 0.999, 1.0])}; "
              f"o_lr/rms max {e32.max():.4f}; S rel {es:.2e}, z rel {ez:.2e}; |o| rms {np.sqrt((o**2).mean()):.4f}",
              flush=True)
