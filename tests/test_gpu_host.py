"""The forward from host buffers (C ABI ropeslr_forward_host): chunked,
pipelined H2D / compute / D2H must give exactly the device-resident
forward's output and attended counts, and match the reference fixtures."""

import numpy as np
import pytest
import torch

import golden_io
import gpu_helpers as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _host(t, pinned=True):
    h = t.cpu()
    return h.pin_memory() if pinned else h


@pytest.mark.parametrize("name", ["bf16_d128_b128", "bf16_d128_keep", "ragged_topk_bf16", "ragged_topk_f32", "cfg0_lowrank"])
def test_host_forward_matches_reference(name):
    import paper_2605_20659_b200 as P

    g = golden_io.load(name)
    q, k, v, x, params, pe, st, grid, _ = G.golden_to_device(g)
    block, perm = P.block_layout(grid.size, st.sparse, grid, q.device)
    if st.compensator != "lowrank" or perm is not None:
        pytest.skip("host path takes flat blocks and the low-rank compensator")
    st = P.ForwardSettings(P.SparseSettings(block=block, keep=st.sparse.keep, topk=st.sparse.topk), use_pe=st.use_pe)
    out, att = P.forward_host(_host(q), _host(k), _host(v), _host(x), grid, params, st, pe, want_attended=True)
    ref_dev = P.forward(q, k, v, x, grid, params, st, pe, trace=True)
    torch.cuda.synchronize()
    assert torch.equal(out, ref_dev.output.cpu()), "host path differs from the device path"
    assert torch.equal(att, ref_dev.attended.cpu())
    G.assert_close(out[0].float().numpy(), g["ref_output"], g["dtype"], f"{name} host output")


@pytest.mark.parametrize("chunk", [0, 1, 3, 5])
@pytest.mark.parametrize("pinned", [True, False])
def test_host_forward_chunks_bit_identical(chunk, pinned):
    """Any head chunking (including a ragged last chunk) gives the device result bit for bit."""
    import paper_2605_20659_b200 as P

    q, k, v, x, params, pe, grid = G.make_full_inputs((3, 8, 40), 7, 128, (16, 56, 56), 64, seed=3)
    L = grid.size
    st = P.ForwardSettings(P.SparseSettings.for_sparsity(128, L, 0.75))
    want = P.forward(q, k, v, x, grid, params, st, pe, trace=True)
    out, att = P.forward_host(_host(q, pinned), _host(k, pinned), _host(v, pinned), _host(x, pinned), grid, params,
                              st, pe, chunk_heads=chunk, want_attended=True)
    assert torch.equal(out, want.output.cpu())
    assert torch.equal(att, want.attended.cpu())


def test_host_forward_column_slice_and_gate_hook():
    """A head-parallel rank: X and out are column slices of wider host
    matrices, and the gate hook sees the partial logits on the call's stream."""
    import paper_2605_20659_b200 as P

    H, d = 6, 128
    q, k, v, x, params, pe, grid = G.make_full_inputs((2, 8, 32), H, d, (16, 56, 56), 64, seed=5)
    L = grid.size
    st = P.ForwardSettings(P.SparseSettings.for_sparsity(64, L, 0.8))
    h0, h1 = 2, 5
    sl = params.heads(h0, h1)
    xs = x[:, :, h0 * d:h1 * d]
    want = P.forward(q[:, h0:h1].contiguous(), k[:, h0:h1].contiguous(), v[:, h0:h1].contiguous(),
                     xs.contiguous(), grid, sl, st, pe, head_offset=h0)
    seen = []

    def hook(g):
        seen.append(g.clone())
    wide_x = _host(x)
    wide_out = torch.zeros((1, L, H * d), dtype=x.dtype).pin_memory()
    P.forward_host(_host(q[:, h0:h1].contiguous()), _host(k[:, h0:h1].contiguous()), _host(v[:, h0:h1].contiguous()),
                   wide_x[:, :, h0 * d:h1 * d], grid, sl, st, pe, head_offset=h0, gate_reduce=hook,
                   out=wide_out[:, :, h0 * d:h1 * d], chunk_heads=1)
    torch.cuda.synchronize()
    assert torch.equal(wide_out[:, :, h0 * d:h1 * d], want.cpu())
    assert torch.count_nonzero(wide_out[:, :, :h0 * d]) == 0 and torch.count_nonzero(wide_out[:, :, h1 * d:]) == 0
    assert len(seen) == 1 and seen[0].shape == (1, L)


def test_host_forward_rejects_device_tensors():
    import paper_2605_20659_b200 as P

    g = golden_io.load("bf16_d128_b128")
    q, k, v, x, params, pe, st, grid, _ = G.golden_to_device(g)
    with pytest.raises(ValueError):
        P.forward_host(q, k, v, x, grid, params, st, pe)
