"""gf2ple-b200: B200-native block-iterative PLE over F2 (arXiv 1111.6549).

The hot path of the reference library gf2elim
(``gf2::block_iterative_ple``, proj/include/gf2/ple.hpp:166) rebuilt as
hand-written sm_100a CUDA behind a C ABI (include/gf2cu.h). This package is
the Python mirror of the reference interface over that ABI.
"""
from ._lib import build, load  # noqa: F401
from .ple import (  # noqa: F401
    BitMatrix,
    ColSwap,
    DeviceMatrix,
    MatrixView,
    PleConfig,
    PleOutcome,
    RowPermutation,
    addmul,
    block_iterative_ple,
    device_count,
    echelonize_strategy,
    mul,
    mul_into,
    partial_ple,
    litmus,
    undo_column_swaps,
    recursive_ple,
    echelonize,
    extract_e,
    extract_l,
    fill_ctr,
    fill_random,
    fill_random_rows,
    host_checksum,
    rref_from_ple,
    trsm_upper_left_unit,
    words_per_row,
)

__all__ = [
    "BitMatrix", "ColSwap", "DeviceMatrix", "MatrixView", "PleConfig", "PleOutcome",
    "RowPermutation", "block_iterative_ple", "device_count", "fill_ctr", "fill_random",
    "host_checksum", "words_per_row", "build", "load", "echelonize", "extract_e", "extract_l",
    "rref_from_ple", "trsm_upper_left_unit", "fill_random_rows", "addmul", "mul", "mul_into", "recursive_ple",
    "echelonize_strategy", "partial_ple", "undo_column_swaps", "litmus",
]
