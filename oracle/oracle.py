"""ctypes front-end for the test-only checkers (see oracle/__init__.py).

Matrices are numpy ``uint64`` arrays of shape ``(m, stride)`` in the
reference layout (bit_matrix.hpp:15-22): column c at bit c & 63 of word
c >> 6, padding bits zero.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(HERE, "liboracle.so")
_REF_SO = os.path.join(HERE, "_ref", "libgf2ref.so")

_sz = C.c_size_t
_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref/libgf2ref.so when the reference is present)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE_SO):
            build()
        L = C.CDLL(_ORACLE_SO)
        L.orc_fill_random.argtypes = [_u64p, _sz, _sz, _sz, C.c_double, C.c_uint64]
        L.orc_fill_random.restype = C.c_int
        L.orc_fill_random_rows.argtypes = [_u64p, _sz, _sz, _sz, _sz, C.c_uint64]
        L.orc_fill_random_rows.restype = C.c_int
        L.orc_fill_ctr.argtypes = [_u64p, _sz, _sz, _sz, C.c_uint64]
        L.orc_fill_ctr.restype = None
        L.orc_ple.argtypes = [_u64p, _sz, _sz, _sz, _szp, _szp]
        L.orc_ple.restype = _sz
        L.orc_canonical_col_swaps.argtypes = [_szp, _sz, _szp]
        L.orc_canonical_col_swaps.restype = _sz
        L.orc_partial_ple.argtypes = [_u64p, _sz, _sz, _sz, _szp, _szp, _szp]
        L.orc_partial_ple.restype = _sz
        L.orc_undo_col_swaps.argtypes = [_u64p, _sz, _sz, _szp, _sz]
        L.orc_undo_col_swaps.restype = None
        L.orc_mul.argtypes = [_u64p, _sz, _sz, _sz, _u64p, _sz, _sz, _u64p, _sz]
        L.orc_mul.restype = None
        L.orc_echelonize.argtypes = [_u64p, _sz, _sz, _sz, C.c_int]
        L.orc_echelonize.restype = _sz
        L.orc_trsm_upper.argtypes = [_u64p, _sz, _sz, _u64p, _sz, _sz]
        L.orc_trsm_upper.restype = None
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def ref():
    """The compiled reference (oracle/_ref/libgf2ref.so)."""
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            raise RuntimeError("oracle/_ref/libgf2ref.so missing (build it where /root/reference exists)")
        R = C.CDLL(_REF_SO)
        R.ref_block_iterative_ple.argtypes = [_u64p, _sz, _sz, _sz, C.c_uint, C.c_uint, _szp, _szp,
                                              _szp, _szp, _sz, _szp]
        R.ref_block_iterative_ple.restype = C.c_double
        R.ref_recursive_ple.argtypes = [_u64p, _sz, _sz, _sz, _sz, _sz, C.c_uint, _szp, _szp, _szp]
        R.ref_recursive_ple.restype = C.c_double
        R.ref_partial_ple.argtypes = [_u64p, _sz, _sz, _sz, _szp, _szp, _szp]
        R.ref_partial_ple.restype = _sz
        R.ref_fill_random.argtypes = [_u64p, _sz, _sz, _sz, C.c_double, C.c_uint64]
        R.ref_fill_random.restype = C.c_int
        R.ref_fill_random_rows.argtypes = [_u64p, _sz, _sz, _sz, _sz, C.c_uint64]
        R.ref_fill_random_rows.restype = C.c_int
        R.ref_mul.argtypes = [_u64p, _sz, _sz, _sz, _u64p, _sz, _sz, _u64p, _sz]
        R.ref_mul.restype = C.c_int
        R.ref_extract_e.argtypes = [_u64p, _sz, _sz, _sz, _sz, _szp, _szp, _szp, _sz, _u64p, _sz]
        R.ref_extract_e.restype = C.c_int
        R.ref_rref_from_ple.argtypes = [_u64p, _sz, _sz, _sz, _sz, _szp, _szp, _szp, _sz, C.c_int]
        R.ref_rref_from_ple.restype = C.c_int
        R.ref_reconstructs.argtypes = [_u64p, _u64p, _sz, _sz, _sz, _sz, _szp, _szp, _szp, _sz]
        R.ref_reconstructs.restype = C.c_int
        R.ref_save_matrix.argtypes = [_u64p, _sz, _sz, _sz, C.c_int, C.c_char_p, _sz]
        R.ref_save_matrix.restype = C.c_longlong
        R.ref_load_matrix.argtypes = [C.c_char_p, _sz, _u64p, _sz, _szp, _szp, C.c_char_p, _sz]
        R.ref_load_matrix.restype = C.c_int
        R.ref_echelonize.argtypes = [_u64p, _sz, _sz, _sz, C.c_int, C.c_int]
        R.ref_echelonize.restype = C.c_longlong
        R.ref_trsm_upper_left_unit.argtypes = [_u64p, _sz, _sz, _u64p, _sz, _sz]
        R.ref_trsm_upper_left_unit.restype = C.c_int
        _ref = R
    return _ref


def _u64(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u64p)


def _szarr(a: np.ndarray):
    assert a.dtype == np.uintp and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_szp)


def words_per_row(n: int) -> int:
    return (n + 63) // 64


def zeros(m: int, n: int, stride: int | None = None) -> np.ndarray:
    return np.zeros((m, stride or max(1, words_per_row(n))), dtype=np.uint64)


# ---------------------------------------------------------------- generators
def fill_random(m: int, n: int, density: float, seed: int, stride: int | None = None) -> np.ndarray:
    a = zeros(m, n, stride)
    if lib().orc_fill_random(_u64(a), m, n, a.shape[1], density, seed & (2**64 - 1)) != 0:
        raise ValueError("density outside [0,1]")
    return a


def fill_random_rows(m: int, n: int, nnz: int, seed: int, stride: int | None = None) -> np.ndarray:
    a = zeros(m, n, stride)
    if lib().orc_fill_random_rows(_u64(a), m, n, a.shape[1], nnz, seed & (2**64 - 1)) != 0:
        raise ValueError("nnz exceeds column count")
    return a


def fill_ctr(m: int, n: int, seed: int, stride: int | None = None) -> np.ndarray:
    a = zeros(m, n, stride)
    lib().orc_fill_ctr(_u64(a), m, n, a.shape[1], seed & (2**64 - 1))
    return a


def mul(a: np.ndarray, l: int, b: np.ndarray, n: int) -> np.ndarray:
    """A (m x l) * B (l x n) over F2 with the restatement."""
    m = a.shape[0]
    c = zeros(m, n)
    lib().orc_mul(_u64(a), m, l, a.shape[1], _u64(b), n, b.shape[1], _u64(c), c.shape[1])
    return c


# ---------------------------------------------------------------------- PLE
@dataclass
class Outcome:
    rank: int
    swaps: np.ndarray  # uintp[rank]
    q: np.ndarray  # uintp[rank]
    col_swaps: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), dtype=np.uintp))


def canonical_col_swaps(q: np.ndarray) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.uintp)
    out = np.zeros((max(1, len(q)), 3), dtype=np.uintp)
    k = lib().orc_canonical_col_swaps(_szarr(q), len(q), _szarr(out))
    return out[:k].copy()


def ple(a: np.ndarray, m: int, n: int) -> Outcome:
    """The C restatement, in place on ``a``."""
    cap = max(1, min(m, n))
    swaps = np.zeros(cap, dtype=np.uintp)
    q = np.zeros(cap, dtype=np.uintp)
    rank = lib().orc_ple(_u64(a), m, n, a.shape[1], _szarr(swaps), _szarr(q))
    q = q[:rank].copy()
    return Outcome(rank, swaps[:rank].copy(), q, canonical_col_swaps(q))


def partial_ple(a: np.ndarray, m: int, n: int):
    """The C restatement of partial_ple (ple.hpp:57-130), in place on ``a``.
    Returns (Outcome, processed)."""
    cap = max(1, min(m, n))
    swaps = np.zeros(cap, dtype=np.uintp)
    q = np.zeros(cap, dtype=np.uintp)
    rank = np.zeros(1, dtype=np.uintp)
    processed = lib().orc_partial_ple(_u64(a), m, n, a.shape[1], _szarr(swaps), _szarr(q), _szarr(rank))
    r = int(rank[0])
    q = q[:r].copy()
    return Outcome(r, swaps[:r].copy(), q, canonical_col_swaps(q)), int(processed)


def ref_partial_ple(a: np.ndarray, m: int, n: int):
    """The compiled reference's partial_ple, in place. Returns (Outcome, processed)."""
    cap = max(1, min(m, n))
    swaps = np.zeros(cap, dtype=np.uintp)
    q = np.zeros(cap, dtype=np.uintp)
    rank = np.zeros(1, dtype=np.uintp)
    processed = ref().ref_partial_ple(_u64(a), m, n, a.shape[1], _szarr(swaps), _szarr(q), _szarr(rank))
    r = int(rank[0])
    q = q[:r].copy()
    return Outcome(r, swaps[:r].copy(), q, canonical_col_swaps(q)), int(processed)


def undo_col_swaps(a: np.ndarray, m: int, cs: np.ndarray) -> None:
    cs = np.ascontiguousarray(cs, dtype=np.uintp).reshape(-1, 3)
    lib().orc_undo_col_swaps(_u64(a), m, a.shape[1], _szarr(cs), cs.shape[0])


def ref_ple(a: np.ndarray, m: int, n: int, k: int = 0, table_count: int = 0):
    """The compiled reference's block_iterative_ple, in place. Returns (Outcome, seconds)."""
    cap = max(1, min(m, n))
    swaps = np.zeros(cap, dtype=np.uintp)
    q = np.zeros(cap, dtype=np.uintp)
    rank = np.zeros(1, dtype=np.uintp)
    ccap = 2 * cap + 2
    cs = np.zeros((ccap, 3), dtype=np.uintp)
    ncs = np.zeros(1, dtype=np.uintp)
    secs = ref().ref_block_iterative_ple(_u64(a), m, n, a.shape[1], k, table_count, _szarr(swaps),
                                         _szarr(q), _szarr(rank), _szarr(cs), ccap, _szarr(ncs))
    if secs < 0:
        raise RuntimeError("reference block_iterative_ple threw")
    r = int(rank[0])
    return Outcome(r, swaps[:r].copy(), q[:r].copy(), cs[: int(ncs[0])].copy()), secs


def ref_recursive_ple(a: np.ndarray, m: int, n: int, base_bytes=0, base_ncols=0, base_k=0) -> Outcome:
    cap = max(1, min(m, n))
    swaps = np.zeros(cap, dtype=np.uintp)
    q = np.zeros(cap, dtype=np.uintp)
    rank = np.zeros(1, dtype=np.uintp)
    ref().ref_recursive_ple(_u64(a), m, n, a.shape[1], base_bytes, base_ncols, base_k,
                            _szarr(swaps), _szarr(q), _szarr(rank))
    r = int(rank[0])
    return Outcome(r, swaps[:r].copy(), q[:r].copy())


def ref_fill_random(m, n, density, seed, stride=None) -> np.ndarray:
    a = zeros(m, n, stride)
    if ref().ref_fill_random(_u64(a), m, n, a.shape[1], density, seed & (2**64 - 1)) != 0:
        raise ValueError("density outside [0,1]")
    return a


def ref_fill_random_rows(m, n, nnz, seed, stride=None) -> np.ndarray:
    a = zeros(m, n, stride)
    if ref().ref_fill_random_rows(_u64(a), m, n, a.shape[1], nnz, seed & (2**64 - 1)) != 0:
        raise ValueError("nnz exceeds column count")
    return a


def ref_mul(a: np.ndarray, l: int, b: np.ndarray, n: int) -> np.ndarray:
    m = a.shape[0]
    c = zeros(m, n)
    if ref().ref_mul(_u64(a), m, l, a.shape[1], _u64(b), n, b.shape[1], _u64(c), c.shape[1]) != 0:
        raise RuntimeError("reference mul threw")
    return c


def ref_extract_e(a: np.ndarray, m: int, n: int, out: Outcome) -> np.ndarray:
    e = zeros(max(out.rank, 1), n)
    cs = np.ascontiguousarray(out.col_swaps, dtype=np.uintp).reshape(-1, 3)
    sw = np.ascontiguousarray(out.swaps, dtype=np.uintp)
    q = np.ascontiguousarray(out.q, dtype=np.uintp)
    if ref().ref_extract_e(_u64(a), m, n, a.shape[1], out.rank, _szarr(sw), _szarr(q), _szarr(cs),
                           cs.shape[0], _u64(e), e.shape[1]) != 0:
        raise RuntimeError("reference extract_e threw")
    return e[: out.rank]


def ref_rref_from_ple(a: np.ndarray, m: int, n: int, out: Outcome, full: bool = True) -> None:
    cs = np.ascontiguousarray(out.col_swaps, dtype=np.uintp).reshape(-1, 3)
    sw = np.ascontiguousarray(out.swaps, dtype=np.uintp)
    q = np.ascontiguousarray(out.q, dtype=np.uintp)
    if ref().ref_rref_from_ple(_u64(a), m, n, a.shape[1], out.rank, _szarr(sw), _szarr(q), _szarr(cs),
                               cs.shape[0], int(full)) != 0:
        raise RuntimeError("reference rref_from_ple threw")


def ref_reconstructs(orig: np.ndarray, dec: np.ndarray, m: int, n: int, out: Outcome) -> bool:
    cs = np.ascontiguousarray(out.col_swaps, dtype=np.uintp).reshape(-1, 3)
    sw = np.ascontiguousarray(out.swaps, dtype=np.uintp)
    q = np.ascontiguousarray(out.q, dtype=np.uintp)
    assert orig.shape == dec.shape
    rc = ref().ref_reconstructs(_u64(orig), _u64(dec), m, n, orig.shape[1], out.rank, _szarr(sw),
                                _szarr(q), _szarr(cs), cs.shape[0])
    if rc < 0:
        raise RuntimeError("reference reconstruction threw")
    return rc == 1


def echelonize(a: np.ndarray, m: int, n: int, full: bool = True) -> int:
    """orc_echelonize: naive_echelonize restated (ple.hpp:362-380), in place."""
    return int(lib().orc_echelonize(_u64(a), m, n, a.shape[1], int(full)))


def trsm_upper(u: np.ndarray, r: int, b: np.ndarray, n: int) -> None:
    """orc_trsm_upper: b <- u^-1 b (multiply.hpp:314-335 restated), in place."""
    lib().orc_trsm_upper(_u64(u), r, u.shape[1], _u64(b), n, b.shape[1])


STRATEGIES = {"naive": 0, "m4ri": 1, "ple_iterative": 2, "ple_recursive": 3}


def ref_echelonize(a: np.ndarray, m: int, n: int, strategy: str = "ple_iterative",
                   full: bool = True) -> int:
    rc = ref().ref_echelonize(_u64(a), m, n, a.shape[1], STRATEGIES[strategy], int(full))
    if rc < 0:
        raise RuntimeError("reference echelonize threw")
    return int(rc)


def ref_trsm_upper_left_unit(u: np.ndarray, r: int, b: np.ndarray, n: int) -> None:
    if ref().ref_trsm_upper_left_unit(_u64(u), r, u.shape[1], _u64(b), n, b.shape[1]) != 0:
        raise RuntimeError("reference trsm_upper_left_unit threw")


def ref_save_matrix(a: np.ndarray, m: int, n: int, ascii: bool = False) -> bytes:
    """The reference's save_gf2b / save_ascii output bytes."""
    cap = 64 + m * (n + 1) + 8 * a.size + 64
    buf = C.create_string_buffer(cap)
    got = ref().ref_save_matrix(_u64(a), m, n, a.shape[1] if a.ndim == 2 else 1, int(ascii), buf, cap)
    if got < 0:
        raise RuntimeError("reference save threw")
    return buf.raw[:got]


def ref_load_matrix(data: bytes):
    """The reference's load_matrix: (m, n, words) or ('io_error', message)."""
    cap = max(1, len(data) // 8 + 16)
    words = np.zeros(cap, dtype=np.uint64)
    m, n = C.c_size_t(), C.c_size_t()
    err = C.create_string_buffer(256)
    rc = ref().ref_load_matrix(data, len(data), _u64(words), cap, C.byref(m), C.byref(n), err, 256)
    if rc != 0:
        return ("io_error" if rc == 1 else "error", err.value.decode())
    W = max(1, (n.value + 63) // 64)
    return m.value, n.value, words[: m.value * W].reshape(m.value, W) if m.value else np.zeros((0, W), np.uint64)
