"""CPU-side checks of the C ABI and the host layer (no kernel launches)."""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "ropeslr_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ropeslr_[a-z_0-9]+)\s*\(", src)))


def test_library_loads_and_exports_every_header_symbol():
    import paper_2605_20659_b200 as P

    lib = P.lib()
    names = header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), f"{n} declared in the header but not exported"
    assert set(names) == set(P.EXPORTED), "ctypes signature table out of sync with the header"


def test_nvcc_target_is_sm100a():
    """The library carries sm_100a SASS (tcgen05 / TMA instructions present)."""
    import shutil
    import subprocess

    import paper_2605_20659_b200._lib as L

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-sass", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in out, f"{mnem} missing from the SASS"


def test_host_functions():
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import _lib

    lib = P.lib()
    assert lib.ropeslr_abi_version() == 3
    assert lib.ropeslr_num_blocks(118800, 128) == 929
    assert lib.ropeslr_num_blocks(32760, 64) == 512
    assert lib.ropeslr_num_blocks(0, 64) == 0
    assert lib.ropeslr_status_string(-1).decode().startswith("inconsistent")
    shp = _lib.Shape(1, 24, 118800, 128, 128, _lib.BF16)
    ws = lib.ropeslr_select_workspace_bytes(ctypes.byref(shp))
    assert ws >= (2 * 24 * 929 * 128 + 24 * 929 * 929) * 8
    # tcgen05: unit schedule, fallback flags / count / list (256-byte rounded)
    up = lambda n: (n + 255) // 256 * 256  # noqa: E731
    assert lib.ropeslr_attend_workspace_bytes(ctypes.byref(shp), 0) == up((3 * 24 * 929 + 1) * 4)
    assert lib.ropeslr_attend_workspace_bytes(ctypes.byref(shp), 1) == 24 * 118800 * 128 * 4
    # block 64 adds the query-block pairs' union lists: counts, indices, bits
    shp64 = _lib.Shape(1, 12, 32760, 128, 64, _lib.BF16)
    units = 12 * 256
    assert lib.ropeslr_attend_workspace_bytes(ctypes.byref(shp64), 0) == \
        up((3 * 12 * 512 + 1) * 4) + units * 4 + units * 512 * 4 + units * 512


def test_abi_rejects_bad_arguments_without_a_gpu():
    """Validation happens before any launch; NULL / ranges give a status."""
    import paper_2605_20659_b200 as P
    from paper_2605_20659_b200 import _lib

    lib = P.lib()
    shp = _lib.Shape(1, 1, 100, 128, 64, _lib.BF16)
    sel = _lib.SelectParams(0, 1.5)  # keep outside (0, 1]
    st = lib.ropeslr_select_blocks(ctypes.byref(shp), ctypes.byref(sel), 16, 16, 16, 2, 16, None, 16, None,
                                   16, 1 << 30, None)
    assert st == -6
    bad = _lib.Shape(1, 1, 100, 128, 64, 7)
    sel = _lib.SelectParams(1, 0.0)
    st = lib.ropeslr_select_blocks(ctypes.byref(bad), ctypes.byref(sel), 16, 16, 16, 2, 16, None, 16, None,
                                   16, 1 << 30, None)
    assert st == -2
    st = lib.ropeslr_select_blocks(ctypes.byref(shp), ctypes.byref(sel), None, 16, 16, 2, 16, None, 16, None,
                                   16, 1 << 30, None)
    assert st == -9


def test_dit_ops_reject_bad_arguments_without_a_gpu():
    """The config-4 caller helpers validate before launching."""
    import paper_2605_20659_b200 as P

    lib = P.lib()
    # NULL input, D not a multiple of 8, D beyond 2048, heads not dividing D,
    # a misaligned pointer
    assert lib.ropeslr_dit_ln_modulate(None, 16, 16, ctypes.c_float(1e-6), 4, 64, 16, None) == -9
    assert lib.ropeslr_dit_ln_modulate(16, 16, 16, ctypes.c_float(1e-6), 4, 60, 16, None) == -1
    assert lib.ropeslr_dit_ln_modulate(16, 16, 16, ctypes.c_float(1e-6), 4, 4096, 16, None) == -1
    assert lib.ropeslr_dit_rms_heads(16, None, ctypes.c_float(0.0), 4, 1536, 7, 1, 16, None) == -1
    assert lib.ropeslr_dit_rms_heads(18, None, ctypes.c_float(0.0), 4, 1536, 12, 1, 16, None) == -3
    assert lib.ropeslr_dit_gated_residual(16, 16, None, 4, 1536, None) == -9


def test_settings_validation_mirrors_reference():
    import paper_2605_20659_b200 as P

    with pytest.raises(ValueError):
        P.SparseSettings(block=(1, 2))
    with pytest.raises(ValueError):
        P.SparseSettings(block=(0, 2, 2))
    with pytest.raises(ValueError):
        P.SparseSettings(block=64, keep=0.0)
    with pytest.raises(ValueError):
        P.SparseSettings(block=64, keep=1.5)
    with pytest.raises(ValueError):
        P.SparseSettings(block=64, topk=-1)
    with pytest.raises(ValueError):
        P.ForwardSettings(P.SparseSettings(64, topk=1), compensator="favor")
    with pytest.raises(ValueError):
        P.RopeConfig(3, 4, 4)
    with pytest.raises(ValueError):
        P.GridShape(0, 1, 1)
    assert P.SparseSettings.topk_for_sparsity(929, 0.9) == 93
    assert P.SparseSettings.for_sparsity(64, 32760, 0.9).topk == 51


def test_block_layout_3d_permutation():
    """3D tiles -> stable tile-major permutation whose flat blocks carry the
    reference's block ids (mechanism.py:280-287)."""
    import numpy as np
    import torch

    import paper_2605_20659_b200 as P
    import restated as R

    grid = P.GridShape(4, 8, 8)
    block, perm = P.block_layout(grid.size, P.SparseSettings((2, 4, 4)), grid, "cpu")
    assert block == 32
    members = R.tile_block_members((4, 8, 8), (2, 4, 4))
    p = perm.numpy()
    for b, m in enumerate(members):
        np.testing.assert_array_equal(np.sort(p[b * 32:(b + 1) * 32]), m)
    block, perm = P.block_layout(grid.size, P.SparseSettings((1, 8, 8)), grid, "cpu")
    assert block == 64 and perm is None
    with pytest.raises(ValueError):
        P.block_layout(grid.size, P.SparseSettings((3, 8, 8)), grid, "cpu")


def test_rotate_rows_matches_oracle():
    import numpy as np
    import torch

    import paper_2605_20659_b200 as P
    import restated as R

    rng = np.random.default_rng(0)
    grid, split = (3, 4, 5), (44, 42, 42)
    m = rng.standard_normal((60, 128))
    got = P.rotate_rows(torch.from_numpy(m), P.GridShape(*grid), P.RopeConfig(*split)).numpy()
    np.testing.assert_allclose(got, R.rotate_rows(m, grid, split), rtol=0, atol=1e-13)


def test_sinusoidal_tables_match_oracle():
    import numpy as np

    import paper_2605_20659_b200 as P
    import restated as R

    pe = P.PETables.sinusoidal(P.GridShape(4, 8, 8), 128, P.RopeConfig(16, 24, 24), device="cpu")
    want = R.sinusoidal_axis_tables((4, 8, 8), 128, (16, 24, 24))
    for a, b in zip((pe.pe_t, pe.pe_x, pe.pe_y), want):
        np.testing.assert_allclose(a.numpy(), b, rtol=0, atol=1e-7)


def test_flops_model():
    from paper_2605_20659_b200 import flops

    assert flops.c_full(1, 24, 118800, 128) == pytest.approx(1.734e14, rel=1e-3)
    assert flops.c_lowrank(1, 24, 118800, 128, 64) == pytest.approx(9.34e10, rel=1e-3)
    assert flops.overhead_eta(118800, 0.9, 64) == pytest.approx(5.43e-3, rel=1e-3)


def test_stage1_ops_reject_bad_arguments_without_a_gpu():
    """The Stage-I row kernels validate before launching (no device needed)."""
    import paper_2605_20659_b200 as P

    lib = P.lib()
    assert [lib.ropeslr_stage1_supported(d) for d in (32, 48, 64, 128, 256, 512)] == [1, 0, 1, 1, 0, 0]
    f = ctypes.c_float
    # unsupported head dim, NULL output, PE without alpha
    assert lib.ropeslr_stage1_pre(2, 8, 48, 16, None, None, 16, f(0.0), 16, 16, 16, None) == -1
    assert lib.ropeslr_stage1_pre(2, 8, 64, 16, None, None, 16, f(0.0), None, 16, 16, None) == -9
    assert lib.ropeslr_stage1_pre(2, 8, 64, 16, 16, None, 16, f(0.0), 16, 16, 16, None) == -9
    assert lib.ropeslr_stage1_rows(2, 0, 64, 16, 16, 16, 16, 16, 16, f(1e-6), f(1.0), 16, 16, 16, None) == -1
    assert lib.ropeslr_stage1_dsig(18, 16, 8, None) == -3
    assert lib.ropeslr_stage1_reduce(16, 1, 0, 2, 64, 16, None) == -1


def test_row_segment_struct_layout():
    """ulysses.Segments packs ropeslr_row_segment as seven int64 words: the
    header's struct is 56 bytes with row_bytes in the low half of word 6."""
    import ctypes

    class Seg(ctypes.Structure):
        _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("src_stride", ctypes.c_int64),
                    ("dst_stride", ctypes.c_int64), ("rows", ctypes.c_int64), ("row0", ctypes.c_int64),
                    ("row_bytes", ctypes.c_int32), ("pad", ctypes.c_int32)]

    assert ctypes.sizeof(Seg) == 56 and Seg.row_bytes.offset == 48
    src = open(os.path.join(REPO, "paper_2605_20659_b200", "ulysses.py")).read()
    assert "dtype=torch.int64)  # ropeslr_row_segment: 56 bytes" in src and "(len(self.views), 7)" in src
