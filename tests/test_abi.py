"""CPU: the C-ABI library builds, loads and exports every symbol
include/gf2cu.h declares; argument validation and the host-side helpers
work without a GPU; with no sm_100 device the calls fail loudly (no CPU
fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1111_6549_b200 as G
from paper_1111_6549_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "gf2cu.h")).read()
    return sorted(set(re.findall(r"\b(gf2cu_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    decl = declared_functions()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(_lib.SYMBOLS), set(decl) ^ set(_lib.SYMBOLS)


def test_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.SO} 2>/dev/null").read()
    assert "sm_100a" in out


def test_version_and_defaults():
    L = _lib.load()
    assert b"sm_100a" in L.gf2cu_version()
    cfg = _lib.gf2cu_cfg()
    L.gf2cu_default_config(C.byref(cfg))
    assert cfg.k == 0 and abs(cfg.k_scale - 0.75) < 1e-12 and cfg.table_count == 4


def test_host_generators_match_oracle():
    for (m, n, d, seed) in [(17, 130, 0.5, 7), (8, 64, 1 / 64, 3), (3, 5, 1.0, 1), (4, 70, 0.0, 9)]:
        a = G.BitMatrix(m, n)
        G.fill_random(a, d, seed)
        assert np.array_equal(a.words, O.fill_random(m, n, d, seed))
    for (m, n, seed) in [(40, 300, 1), (3, 64, 11), (5, 1, 2)]:
        a = G.BitMatrix(m, n)
        G.fill_ctr(a, seed)
        assert np.array_equal(a.words, O.fill_ctr(m, n, seed))


def test_argument_validation_maps_to_reference_exceptions():
    a = G.BitMatrix(4, 4)
    with pytest.raises(ValueError):
        G.fill_random(a, 1.5, 1)  # std::invalid_argument (bit_matrix.hpp:460)
    with pytest.raises(IndexError):  # window past the row stride
        G.block_iterative_ple(G.MatrixView(a.words, 1, 10, 4, 60))
    with pytest.raises(IndexError):  # more rows than the array holds
        G.MatrixView(a.words, 1, 0, 5, 4)
    with pytest.raises(IndexError):  # a stride that walks off the array
        G.MatrixView(np.zeros(10, dtype=np.uint64), 3, 0, 5, 64)
    ok = G.MatrixView(np.zeros(10, dtype=np.uint64), 3, 0, 4, 63)  # (4-1)*3 + 1 = 10 words
    assert ok.nrows() == 4
    with pytest.raises(IndexError):
        a.view().sub(1, 0, 4, 4)  # std::out_of_range (bit_matrix.hpp:218-221)


def test_empty_inputs_do_not_touch_a_device():
    for m, n in [(0, 5), (5, 0), (0, 0)]:
        out = G.block_iterative_ple(G.BitMatrix(m, n))
        assert out.rank == 0 and out.processed == m and len(out.q) == 0


@pytest.mark.skipif(G.device_count() > 0, reason="a GPU is visible")
def test_no_device_fails_loudly():
    with pytest.raises(_lib.Gf2cuError):
        G.block_iterative_ple(G.BitMatrix.identity(8))
    with pytest.raises(_lib.Gf2cuError):
        G.DeviceMatrix(8, 8)
