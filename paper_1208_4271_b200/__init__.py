"""B200-native MINE score engine (MIC/MAS/MEV/MCN + MIC_e/TIC).

The hot path -- per-pair rank/sort, EquipartitionYAxis, GetClumps /
GetSuperclumpsPartition, the OptimizeXAxis DP and the statistic reductions of
the reference (/root/reference/proj/src) -- runs as hand-written sm_100a CUDA
kernels in libmine_b200.so behind the C ABI of include/mine_b200.h.
"""
from .engine import (  # noqa: F401
    ALL_STATS, MIC_APPROX, MIC_E, STATS, CharacteristicMatrix, Engine, MineError, Parameters,
    cell_shapes, compute_score, compute_statistics, default_engine, grid_bound,
    load_library, read_dataset, validate_parameters,
)

__all__ = [
    "ALL_STATS", "MIC_APPROX", "MIC_E", "STATS", "CharacteristicMatrix", "Engine", "MineError", "Parameters",
    "cell_shapes", "compute_score", "compute_statistics", "default_engine", "grid_bound",
    "load_library", "read_dataset", "validate_parameters",
]
