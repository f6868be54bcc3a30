"""ctypes binding of the C ABI in include/ropeslr_b200.h.

The library is built in-tree (``build.py``) and loaded from this package
directory.  There is no fallback: if the shared library is missing or was
built for another architecture, every op raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# ROPESLR_LIBRARY points at an alternative build of the same library (kernel
# variant experiments); the default is the in-tree build.
LIB_PATH = os.environ.get("ROPESLR_LIBRARY") or os.path.join(PKG, "libropeslr_b200.so")

ABI_VERSION = 3  # include/ropeslr_b200.h ROPESLR_ABI_VERSION
F32, BF16 = 0, 1
LOWRANK, LINEAR = 0, 1
NONFINITE_QK, NONFINITE_X = 1, 2
IMPL = {"auto": 0, "simt": 1, "tcgen05": 2}

c_i32, c_i64, c_f32, c_f64, c_sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double, ctypes.c_size_t
c_vp = ctypes.c_void_p


class Shape(ctypes.Structure):
    _fields_ = [("B", c_i64), ("H", c_i64), ("L", c_i64), ("d", c_i64), ("block", c_i32), ("dtype", c_i32),
                ("qb_begin", c_i32), ("qb_end", c_i32)]


class SelectParams(ctypes.Structure):
    _fields_ = [("topk", c_i32), ("keep", c_f64), ("nonfinite", c_vp)]


class TokenArgs(ctypes.Structure):
    _fields_ = [("x", c_vp), ("x_row_stride", c_i64), ("head_offset", c_i64), ("d_model", c_i64),
                ("grid_t", c_i32), ("grid_h", c_i32), ("grid_w", c_i32), ("use_pe", c_i32),
                ("pe_t", c_vp), ("pe_x", c_vp), ("pe_y", c_vp), ("alpha", c_vp), ("w_g", c_vp), ("nonfinite", c_vp),
                ("token_offset", c_i64)]


class RopeArgs(ctypes.Structure):
    _fields_ = [("d_t", c_i32), ("d_x", c_i32), ("d_y", c_i32), ("grid_t", c_i32), ("grid_h", c_i32),
                ("grid_w", c_i32), ("base", c_f64)]


GateHook = ctypes.CFUNCTYPE(None, c_vp, c_i64, c_vp, c_vp)


class HostForward(ctypes.Structure):
    _fields_ = [("shape", Shape), ("sel", SelectParams), ("q", c_vp), ("k", c_vp), ("v", c_vp), ("tok", TokenArgs),
                ("w_a", c_vp), ("w_b", c_vp), ("rank", c_i32), ("rms_sparse", c_vp), ("rms_lowrank", c_vp),
                ("b_g", c_f32), ("eps", c_f32), ("out", c_vp), ("out_row_stride", c_i64), ("attended", c_vp),
                ("chunk_heads", c_i32), ("gate_hook", GateHook), ("gate_hook_user", c_vp)]


P = ctypes.POINTER
_SIGNATURES = {
    "ropeslr_abi_version": (c_i32, []),
    "ropeslr_status_string": (ctypes.c_char_p, [c_i32]),
    "ropeslr_last_cuda_error": (ctypes.c_char_p, []),
    "ropeslr_device_check": (c_i32, [c_i32]),
    "ropeslr_num_blocks": (c_i64, [c_i64, c_i32]),
    "ropeslr_set_option": (c_i32, [ctypes.c_char_p, c_i32]),
    "ropeslr_get_option": (c_i32, [ctypes.c_char_p]),
    "ropeslr_select_workspace_bytes": (c_sz, [P(Shape)]),
    "ropeslr_select_blocks": (c_i32, [P(Shape), P(SelectParams), c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp,
                                      c_vp, c_sz, c_vp]),
    "ropeslr_sparse_attention": (c_i32, [P(Shape), c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "ropeslr_lowrank_workspace_bytes": (c_sz, [P(Shape), P(TokenArgs), c_i32]),
    "ropeslr_lowrank_tables_bytes": (c_sz, [P(Shape), P(TokenArgs), c_i32]),
    "ropeslr_lowrank_tables": (c_i32, [P(Shape), P(TokenArgs), c_vp, c_vp, c_i32, c_vp, c_sz, c_vp]),
    "ropeslr_lowrank_branch_folded": (c_i32, [P(Shape), P(TokenArgs), c_i32, c_vp, c_sz, c_vp, c_f32, c_vp, c_vp,
                                              c_vp, c_vp, c_sz, c_vp]),
    "ropeslr_lowrank_branch": (c_i32, [P(Shape), P(TokenArgs), c_vp, c_vp, c_i32, c_vp, c_f32, c_vp, c_vp, c_vp,
                                       c_vp, c_sz, c_vp]),
    "ropeslr_gate_logits": (c_i32, [P(Shape), P(TokenArgs), c_vp, c_vp]),
    "ropeslr_linear_workspace_bytes": (c_sz, [P(Shape)]),
    "ropeslr_linear_branch": (c_i32, [P(Shape), c_vp, c_vp, c_vp, c_vp, c_f32, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "ropeslr_linear_tables_bytes": (c_sz, [P(Shape), P(TokenArgs)]),
    "ropeslr_linear_tables": (c_i32, [P(Shape), P(TokenArgs), c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "ropeslr_linear_pe_workspace_bytes": (c_sz, [P(Shape), P(TokenArgs)]),
    "ropeslr_linear_branch_pe": (c_i32, [P(Shape), P(TokenArgs), c_vp, c_vp, c_vp, c_vp, c_vp, c_f32, c_vp, c_vp,
                                         c_vp, c_vp, c_vp, c_sz, c_vp]),
    "ropeslr_fuse_output": (c_i32, [P(Shape), c_vp, c_vp, c_vp, c_f32, c_vp, c_f32, c_vp, c_vp]),
    "ropeslr_attend_fused": (c_i32, [P(Shape), c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_f32, c_vp,
                                     c_f32, c_vp, c_i32, c_vp, c_i32, c_vp, c_sz, c_vp]),
    "ropeslr_attend_workspace_bytes": (c_sz, [P(Shape), c_i32]),
    "ropeslr_select_pooled_workspace_bytes": (c_sz, [P(Shape)]),
    "ropeslr_select_screen_offsets": (c_i32, [P(Shape), c_i32, P(c_sz), P(c_sz), P(c_sz)]),
    "ropeslr_select_from_pooled": (c_i32, [P(Shape), P(SelectParams), c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp,
                                           c_vp, c_sz, c_vp]),
    "ropeslr_copy_rows": (c_i32, [c_vp, c_i32, c_i64, c_vp]),
    "ropeslr_dit_ln_modulate": (c_i32, [c_vp, c_vp, c_vp, c_f32, c_i64, c_i32, c_vp, c_vp]),
    "ropeslr_dit_ln_affine": (c_i32, [c_vp, c_vp, c_vp, c_f32, c_i64, c_i32, c_vp, c_vp]),
    "ropeslr_dit_gated_add": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "ropeslr_dit_rms_heads_strided": (c_i32, [c_vp, c_i64, c_vp, c_f32, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "ropeslr_dit_heads_to_tokens": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_i32, c_vp, c_vp]),
    "ropeslr_dit_rms_heads": (c_i32, [c_vp, c_vp, c_f32, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "ropeslr_dit_gated_residual": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "ropeslr_stage1_supported": (c_i32, [c_i64]),
    "ropeslr_stage1_rows_blocks": (c_i32, [c_i64, c_i64]),
    "ropeslr_stage1_xgrad_blocks": (c_i32, [c_i64, c_i64]),
    "ropeslr_stage1_pre": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_f32, c_vp, c_vp, c_vp, c_vp]),
    "ropeslr_stage1_pre_dev": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ropeslr_stage1_rows": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_f32, c_f32, c_vp,
                                    c_vp, c_vp, c_vp]),
    "ropeslr_stage1_gate_bwd": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ropeslr_stage1_dsig": (c_i32, [c_vp, c_vp, c_i64, c_vp]),
    "ropeslr_stage1_xgrad": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ropeslr_stage1_reduce": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "ropeslr_stage1_gemm_rows": (c_i32, [c_i64, c_i64, c_i32, c_i32, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "ropeslr_stage1_gram_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "ropeslr_stage1_gemm_gram": (c_i32, [c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_sz, c_vp]),
    "ropeslr_rope_pool_workspace_bytes": (c_sz, [P(RopeArgs)]),
    "ropeslr_rope_pool": (c_i32, [P(Shape), P(RopeArgs), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "ropeslr_forward_host_workspace_bytes": (c_sz, [P(HostForward)]),
    "ropeslr_forward_host": (c_i32, [P(HostForward), c_vp, c_sz, c_vp]),
}
EXPORTED = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


class RopeSLRError(ValueError):
    """Nonzero status from the C ABI (a ValueError, like the reference's)."""

    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn}: {msg} (status {status})")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libropeslr_b200.so once; raise if it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2605_20659_b200.build` "
                    "(there is no CPU fallback for the RoPeSLR op)")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            if handle.ropeslr_abi_version() != ABI_VERSION:
                raise RuntimeError("libropeslr_b200.so ABI version mismatch")
            _lib = handle
    return _lib


def check(fn: str, status: int) -> None:
    if status != 0:
        msg = lib().ropeslr_status_string(status).decode()
        if status == -5:  # ROPESLR_ERR_LAUNCH: add the CUDA runtime's message
            msg += f" [{lib().ropeslr_last_cuda_error().decode()}]"
        raise RopeSLRError(fn, status, msg)


def call(fn: str, *args) -> None:
    check(fn, getattr(lib(), fn)(*args))


def set_option(name: str, value) -> None:
    """Process-wide kernel-variant switch (include/ropeslr_b200.h
    ropeslr_set_option); ``value`` may be a one-character string ('f', 'd')."""
    v = ord(value) if isinstance(value, str) else int(value)
    check("ropeslr_set_option", lib().ropeslr_set_option(name.encode(), v))


def get_option(name: str) -> int:
    v = lib().ropeslr_get_option(name.encode())
    if v < 0:
        check("ropeslr_get_option", v)
    return v


class option:
    """Context manager: ``with option("k2_online", 1): ...`` restores the
    previous value on exit."""

    def __init__(self, name: str, value):
        self.name, self.value = name, value

    def __enter__(self):
        self.prev = get_option(self.name)
        set_option(self.name, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.name, self.prev)
