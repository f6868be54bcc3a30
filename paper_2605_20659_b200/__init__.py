"""B200-native (sm_100a) RoPeSLR sparse-low-rank attention forward.

Host-side mirror of the reference's ``ropeslr.mechanism`` API over hand-written
CUDA kernels in ``libropeslr_b200.so`` (C ABI: include/ropeslr_b200.h).
"""

from . import flops
from ._lib import EXPORTED, RopeSLRError, lib
from .mechanism import (RMS_EPS, Backbone, BlockSparseResult, ForwardSettings, ForwardTrace, MechanismParams,
                        PETables, Prepared, Selection, attend, attend_workspace, fallback_units, prepare, SparseSettings, block_layout, block_sparse_attention,
                        compensator_branch, forward, forward_from_x, forward_host, gate, init_params, lowrank_compensator,
                        project_and_rotate, rope_pool, select_blocks)
from .rope3d import GridShape, RopeConfig, rotate_rows

__all__ = [
    "RMS_EPS", "Backbone", "BlockSparseResult", "ForwardSettings", "ForwardTrace", "MechanismParams", "PETables",
    "Selection", "SparseSettings", "Prepared", "prepare", "attend", "attend_workspace", "fallback_units", "GridShape", "RopeConfig", "block_layout", "block_sparse_attention",
    "compensator_branch", "forward", "forward_from_x", "forward_host", "gate", "init_params", "lowrank_compensator",
    "project_and_rotate", "rope_pool", "rotate_rows", "select_blocks", "flops", "lib", "EXPORTED", "RopeSLRError",
]
