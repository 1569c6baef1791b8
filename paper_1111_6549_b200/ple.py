"""Host-side mirror of the reference PLE interface over the B200 C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/gf2/{bit_matrix,ple}.hpp:

* ``BitMatrix`` / ``MatrixView``   -- bit_matrix.hpp:163-394 (row-major
  uint64 words, LSB-first, padding bits zero; views carry a bit offset).
* ``PleConfig``, ``ColSwap``, ``PleOutcome`` -- ple.hpp:31-51.
* ``RowPermutation``               -- bit_matrix.hpp:416-438 (LAPACK swaps).
* ``block_iterative_ple(a, cfg)``  -- ple.hpp:166, computed on the B200 by
  ``gf2cu_ple`` (host view) or ``gf2cu_ple_device`` (``DeviceMatrix``).

Exceptions match the reference: ValueError for std::invalid_argument,
IndexError for std::out_of_range, MemoryError for std::bad_alloc; CUDA
failures (including "no sm_100 device") raise ``Gf2cuError``. There is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import check, gf2cu_cfg, gf2cu_colswap, gf2cu_stats, gf2cu_view

WORD_BITS = 64


def words_per_row(ncols: int) -> int:
    return (ncols + WORD_BITS - 1) // WORD_BITS


# --------------------------------------------------------------------- types
@dataclass
class PleConfig:
    """ple.hpp:31-39. k / table_count are accepted for interface parity; the
    device path factors 64-column panels and its output does not depend on
    them (nor does the reference's)."""
    k: int = 0
    k_scale: float = 0.75
    table_count: int = 4
    base_bytes: int = 256 << 10
    base_ncols: int = 64
    base_k: int = 0
    device: int = 0
    stream: Optional[int] = None   # cudaStream_t as an int (e.g. torch stream.cuda_stream)
    time_kernels: bool = False
    multi_kernel: bool = False     # one launch per phase (cross-check driver)
    single_panel: bool = False     # force the persistent driver with one panel per sweep
    super_step: bool = False       # force the super-step driver (two panels per sweep)
    peer_ranks: int = 0            # >0: the row-sharded peer-memory driver with this many
                                   # ranks emulated on the one device (ple_peer.cuh)
    check: bool = False            # check mode: device invariants asserted every step

    def to_c(self) -> gf2cu_cfg:
        c = gf2cu_cfg()
        _lib.load().gf2cu_default_config(C.byref(c))
        c.k = int(self.k)
        c.k_scale = float(self.k_scale)
        c.table_count = max(1, int(self.table_count))
        c.device = int(self.device)
        c.stream = C.c_void_p(self.stream) if self.stream else None
        c.flags = (_lib.FLAG_TIME_KERNELS if self.time_kernels else 0) | \
            (_lib.FLAG_MULTI_KERNEL if self.multi_kernel else 0) | \
            (_lib.FLAG_SINGLE_PANEL if self.single_panel else 0) | \
            (_lib.FLAG_SUPER_STEP if self.super_step else 0) | \
            (_lib.FLAG_CHECK if self.check else 0) | \
            ((int(self.peer_ranks) & 15) << 16)
        return c


@dataclass(frozen=True)
class ColSwap:
    a: int
    b: int
    from_row: int


@dataclass
class RowPermutation:
    """LAPACK-style transpositions: swaps[i] is the row swapped with row i
    (bit_matrix.hpp:416-438)."""
    swaps: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint64))

    def size(self) -> int:
        return len(self.swaps)

    def validate(self, nrows: int) -> None:
        s = np.asarray(self.swaps, dtype=np.int64)
        if len(s) and (np.any(s < np.arange(len(s))) or np.any(s >= nrows)):
            raise ValueError("RowPermutation: entry out of range")

    def apply(self, a: np.ndarray) -> None:
        """Replay the swaps forward on the rows of a 2-D array."""
        self.validate(a.shape[0])
        for i, j in enumerate(np.asarray(self.swaps, dtype=np.int64)):
            if j != i:
                a[[i, j]] = a[[j, i]]

    def apply_inverse(self, a: np.ndarray) -> None:
        self.validate(a.shape[0])
        s = np.asarray(self.swaps, dtype=np.int64)
        for i in range(len(s) - 1, -1, -1):
            j = s[i]
            if j != i:
                a[[i, j]] = a[[j, i]]


class PleOutcome:
    """ple.hpp:45-51. `col_swaps` is materialised lazily from the (k, 3)
    array `col_swaps_array` (the canonical {j, q[j], j} list)."""

    def __init__(self, rank: int = 0, processed: int = 0, p: Optional[RowPermutation] = None,
                 q: Optional[np.ndarray] = None, col_swaps_array: Optional[np.ndarray] = None,
                 stats: Optional[dict] = None):
        self.rank = rank
        self.processed = processed
        self.p = p if p is not None else RowPermutation()
        self.q = q if q is not None else np.zeros(0, dtype=np.uint64)
        self.col_swaps_array = (col_swaps_array if col_swaps_array is not None
                                else np.zeros((0, 3), dtype=np.uint64))
        self.stats = stats
        self._cs = None

    @property
    def col_swaps(self) -> List[ColSwap]:
        if self._cs is None:
            self._cs = [ColSwap(int(a), int(b), int(c)) for a, b, c in self.col_swaps_array]
        return self._cs


class MatrixView:
    """Non-owning window {data, stride, col_off, nrows, ncols} over a uint64
    word array (bit_matrix.hpp:163-340)."""

    def __init__(self, words: np.ndarray, stride: int, col_off: int, nrows: int, ncols: int):
        if words.dtype != np.uint64:
            raise ValueError("MatrixView needs uint64 words")
        self.words = words
        self.stride = int(stride)
        self.col_off = int(col_off)
        self._nrows = int(nrows)
        self._ncols = int(ncols)
        if min(self.stride, self.col_off, self._nrows, self._ncols) < 0:
            raise IndexError("negative view geometry")
        if self._nrows and self._ncols:
            # the device path writes L\E back through the raw pointer: the
            # window must lie inside the array (bit_matrix.hpp:214-221 raise
            # std::out_of_range for windows outside the matrix)
            end = self.col_off + self._ncols
            if end > 64 * self.stride:
                raise IndexError("view window wider than its stride")
            need = (self._nrows - 1) * self.stride + (end + 63) // 64
            if words.size < need:
                raise IndexError(f"view needs {need} words, array holds {words.size}")

    def nrows(self) -> int:
        return self._nrows

    def ncols(self) -> int:
        return self._ncols

    def col_offset(self) -> int:
        return self.col_off

    def sub(self, r0: int, c0: int, rows: int, cols: int) -> "MatrixView":
        if r0 > self._nrows or rows > self._nrows - r0 or c0 > self._ncols or cols > self._ncols - c0:
            raise IndexError("subview outside matrix view")
        flat = self.words.reshape(-1)
        return MatrixView(flat[r0 * self.stride:], self.stride, self.col_off + c0, rows, cols)

    def get(self, i: int, j: int) -> bool:
        p = self.col_off + j
        return bool((int(self.words.reshape(-1)[i * self.stride + (p >> 6)]) >> (p & 63)) & 1)

    def _c(self) -> gf2cu_view:
        v = gf2cu_view()
        if not self.words.flags["C_CONTIGUOUS"]:
            raise ValueError("MatrixView words must be C-contiguous")
        v.data = self.words.ctypes.data_as(C.POINTER(C.c_uint64))
        v.stride = self.stride
        v.col_off = self.col_off
        v.nrows = self._nrows
        v.ncols = self._ncols
        return v


class BitMatrix:
    """Owning packed matrix, stride = ceil(ncols/64) words, padding zero
    (bit_matrix.hpp:342-394)."""

    def __init__(self, rows: int, cols: int, words: Optional[np.ndarray] = None):
        self._nrows, self._ncols = int(rows), int(cols)
        self._stride = words_per_row(cols)
        if words is None:
            self.words = np.zeros((rows, self._stride), dtype=np.uint64)
        else:
            words = np.ascontiguousarray(words, dtype=np.uint64)
            if words.shape != (rows, self._stride):
                raise ValueError("words shape does not match (rows, ceil(cols/64))")
            self.words = words

    @staticmethod
    def identity(n: int) -> "BitMatrix":
        a = BitMatrix(n, n)
        for i in range(n):
            a.words[i, i >> 6] |= np.uint64(1) << np.uint64(i & 63)
        return a

    @staticmethod
    def from_rows(rows: List[str]) -> "BitMatrix":
        a = BitMatrix(len(rows), len(rows[0]) if rows else 0)
        for i, s in enumerate(rows):
            for j, ch in enumerate(s):
                if ch == "1":
                    a.set(i, j, True)
        return a

    def nrows(self) -> int:
        return self._nrows

    def ncols(self) -> int:
        return self._ncols

    def stride(self) -> int:
        return self._stride

    def get(self, i: int, j: int) -> bool:
        return bool((int(self.words[i, j >> 6]) >> (j & 63)) & 1)

    def set(self, i: int, j: int, v: bool) -> None:
        bit = np.uint64(1) << np.uint64(j & 63)
        if v:
            self.words[i, j >> 6] |= bit
        else:
            self.words[i, j >> 6] &= ~bit

    def view(self) -> MatrixView:
        return MatrixView(self.words, self._stride, 0, self._nrows, self._ncols)

    def copy(self) -> "BitMatrix":
        return BitMatrix(self._nrows, self._ncols, self.words.copy())

    def __eq__(self, other) -> bool:
        return (isinstance(other, BitMatrix) and self._nrows == other._nrows
                and self._ncols == other._ncols and np.array_equal(self.words, other.words))

    def row_string(self, i: int) -> str:
        return "".join("1" if self.get(i, j) else "0" for j in range(self._ncols))


# --------------------------------------------------------------- generators
def fill_random(a: BitMatrix, density: float, seed: int) -> None:
    """gf2::fill_random (bit_matrix.hpp:459-486), host-side (std::mt19937_64)."""
    L = _lib.load()
    check(L.gf2cu_fill_random(a.words.ctypes.data_as(C.POINTER(C.c_uint64)), a.nrows(), a.ncols(),
                              a.stride(), float(density), int(seed) & (2**64 - 1)))


def fill_random_rows(a: BitMatrix, nnz: int, seed: int) -> None:
    """gf2::fill_random_rows (bit_matrix.hpp:489-520), host-side."""
    L = _lib.load()
    check(L.gf2cu_fill_random_rows(a.words.ctypes.data_as(C.POINTER(C.c_uint64)), a.nrows(),
                                   a.ncols(), a.stride(), int(nnz), int(seed) & (2**64 - 1)))


def fill_ctr(a: BitMatrix, seed: int) -> None:
    """The counter generator of SURVEY.md 8(d) (random access; the device
    generator DeviceMatrix.fill_ctr produces the same words)."""
    L = _lib.load()
    check(L.gf2cu_fill_ctr(a.words.ctypes.data_as(C.POINTER(C.c_uint64)), a.nrows(), a.ncols(),
                           a.stride(), int(seed) & (2**64 - 1)))


# ----------------------------------------------------------- device matrix
class DeviceMatrix:
    """An m x n matrix resident in HBM (128-byte aligned rows)."""

    def __init__(self, m: int, n: int, device: int = 0):
        L = _lib.load()
        h = C.c_void_p()
        check(L.gf2cu_matrix_create(m, n, device, C.byref(h)))
        self._h = h
        self.m, self.n, self.device = m, n, device
        st = C.c_size_t()
        ptr = C.POINTER(C.c_uint64)()
        check(L.gf2cu_matrix_info(h, None, None, C.byref(st), C.byref(ptr)))
        self.stride_words = st.value

    @property
    def handle(self):
        return self._h

    def data_ptr(self) -> int:
        ptr = C.POINTER(C.c_uint64)()
        check(_lib.load().gf2cu_matrix_info(self._h, None, None, None, C.byref(ptr)))
        return C.cast(ptr, C.c_void_p).value or 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().gf2cu_matrix_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, words: np.ndarray, stream: Optional[int] = None) -> None:
        words = np.ascontiguousarray(words, dtype=np.uint64)
        if words.shape[0] != self.m:
            raise ValueError("row count mismatch")
        check(_lib.load().gf2cu_matrix_upload(self._h, words.ctypes.data_as(C.POINTER(C.c_uint64)),
                                              words.shape[1], C.c_void_p(stream) if stream else None))

    def upload_ptr(self, host_ptr: int, host_stride: int, stream: Optional[int] = None) -> None:
        check(_lib.load().gf2cu_matrix_upload(self._h, C.cast(C.c_void_p(host_ptr), C.POINTER(C.c_uint64)),
                                              host_stride, C.c_void_p(stream) if stream else None))

    def download(self, out: Optional[np.ndarray] = None, stream: Optional[int] = None) -> np.ndarray:
        W = words_per_row(self.n)
        if out is None:
            out = np.zeros((self.m, max(1, W)), dtype=np.uint64)
        check(_lib.load().gf2cu_matrix_download(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                out.shape[1], C.c_void_p(stream) if stream else None))
        return out

    def download_ptr(self, host_ptr: int, host_stride: int, stream: Optional[int] = None) -> None:
        check(_lib.load().gf2cu_matrix_download(self._h, C.cast(C.c_void_p(host_ptr), C.POINTER(C.c_uint64)),
                                                host_stride, C.c_void_p(stream) if stream else None))

    def copy_from(self, other: "DeviceMatrix", stream: Optional[int] = None) -> None:
        check(_lib.load().gf2cu_matrix_copy(self._h, other._h, C.c_void_p(stream) if stream else None))

    def fill_ctr(self, seed: int, stream: Optional[int] = None) -> None:
        check(_lib.load().gf2cu_matrix_fill_ctr(self._h, int(seed) & (2**64 - 1),
                                                C.c_void_p(stream) if stream else None))

    def checksum(self, stream: Optional[int] = None) -> int:
        out = C.c_uint64()
        check(_lib.load().gf2cu_matrix_checksum(self._h, C.byref(out), C.c_void_p(stream) if stream else None))
        return out.value


def host_checksum(words: np.ndarray, ncols: int) -> int:
    """Same fold as gf2cu_matrix_checksum, computed on host words (test helper
    and bench parity handle): per-row FNV-1a over the W logical words, then
    FNV-1a over the row hashes."""
    W = words_per_row(ncols)
    w = np.ascontiguousarray(words[:, :W], dtype=np.uint64)
    prime = np.uint64(0x100000001B3)
    h = np.full(w.shape[0], 0xCBF29CE484222325, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for x in range(W):
            h ^= w[:, x]
            h *= prime
        acc = np.uint64(0xCBF29CE484222325)
        for v in h:
            acc ^= v
            acc *= prime
    return int(acc)


# ----------------------------------------------------------------- the path
def _outcome(rank, swaps, q, cs, ncs, m, st) -> PleOutcome:
    r = int(rank.value)
    return PleOutcome(rank=r, processed=m, p=RowPermutation(swaps[:r].astype(np.uint64)),
                      q=q[:r].astype(np.uint64),
                      col_swaps_array=cs[: int(ncs.value)].astype(np.uint64),
                      stats={f: getattr(st, f) for f, _ in gf2cu_stats._fields_})


def block_iterative_ple(a, cfg: Optional[PleConfig] = None) -> PleOutcome:
    """gf2::block_iterative_ple (ple.hpp:166) on the B200.

    ``a`` is a ``BitMatrix``/``MatrixView`` (host words, factored in place)
    or a ``DeviceMatrix`` (factored in place in HBM)."""
    cfg = cfg or PleConfig()
    L = _lib.load()
    c = cfg.to_c()
    if isinstance(a, DeviceMatrix):
        m, n = a.m, a.n
        h = a.handle
    else:
        view = a.view() if isinstance(a, BitMatrix) else a
        m, n = view.nrows(), view.ncols()
    cap = max(1, min(m, n))
    swaps = np.empty(cap, dtype=np.uintp)
    q = np.empty(cap, dtype=np.uintp)
    cs = np.empty((cap, 3), dtype=np.uintp)  # gf2cu_colswap = 3 x size_t
    rank = C.c_size_t()
    ncs = C.c_size_t()
    st = gf2cu_stats()
    szp = C.POINTER(C.c_size_t)
    sp, qp = swaps.ctypes.data_as(szp), q.ctypes.data_as(szp)
    cp = C.cast(cs.ctypes.data, C.POINTER(gf2cu_colswap))
    if isinstance(a, DeviceMatrix):
        check(L.gf2cu_ple_device(h, C.byref(c), sp, qp, C.byref(rank), cp, C.byref(ncs), C.byref(st)))
    else:
        v = view._c()
        check(L.gf2cu_ple(C.byref(v), C.byref(c), sp, qp, C.byref(rank), cp, C.byref(ncs), C.byref(st)))
    return _outcome(rank, swaps, q, cs, ncs, m, st)


def partial_ple(a, cfg: Optional[PleConfig] = None) -> PleOutcome:
    """gf2::partial_ple (ple.hpp:57-130) on the B200: the lazy single pass.
    Same rank / q / p.swaps / col_swaps as the reference; ``processed`` is
    its watermark and rows past it are left untouched (only possible when
    every column finds a pivot and rank == ncols < nrows). Host views only,
    as the reference's MatrixView."""
    if isinstance(a, DeviceMatrix):
        raise TypeError("partial_ple takes a host BitMatrix / MatrixView")
    cfg = cfg or PleConfig()
    L = _lib.load()
    c = cfg.to_c()
    view = _host_view(a)
    m, n = view.nrows(), view.ncols()
    cap = max(1, min(m, n))
    swaps = np.empty(cap, dtype=np.uintp)
    q = np.empty(cap, dtype=np.uintp)
    cs = np.empty((cap, 3), dtype=np.uintp)
    rank, processed, ncs = C.c_size_t(), C.c_size_t(), C.c_size_t()
    szp = C.POINTER(C.c_size_t)
    v = view._c()
    check(L.gf2cu_partial_ple(C.byref(v), C.byref(c), swaps.ctypes.data_as(szp), q.ctypes.data_as(szp),
                              C.byref(rank), C.byref(processed),
                              C.cast(cs.ctypes.data, C.POINTER(gf2cu_colswap)), C.byref(ncs)))
    r = int(rank.value)
    return PleOutcome(rank=r, processed=int(processed.value), p=RowPermutation(swaps[:r].astype(np.uint64)),
                      q=q[:r].astype(np.uint64), col_swaps_array=cs[: int(ncs.value)].astype(np.uint64))


def undo_column_swaps(a, col_swaps, cfg: Optional[PleConfig] = None) -> None:
    """gf2::undo_column_swaps (ple.hpp:293-296) on the B200: the compression
    swaps (a list of ColSwap or a (k, 3) array) replayed backwards."""
    if isinstance(col_swaps, np.ndarray):
        arr = np.ascontiguousarray(col_swaps.reshape(-1, 3), dtype=np.uintp)
    else:
        arr = np.array([[c.a, c.b, c.from_row] for c in col_swaps], dtype=np.uintp).reshape(-1, 3)
    L = _lib.load()
    cp = C.cast(arr.ctypes.data, C.POINTER(gf2cu_colswap)) if len(arr) else None
    if isinstance(a, DeviceMatrix):
        check(L.gf2cu_undo_column_swaps_device(a.handle, cp, len(arr), None))
        return
    c = (cfg or PleConfig()).to_c()
    v = _host_view(a)._c()
    check(L.gf2cu_undo_column_swaps(C.byref(v), cp, len(arr), C.byref(c)))


def litmus(kind: int, rounds: int = 64, device: int = 0):
    """gf2cu_litmus: message-passing litmus run of one of the drivers'
    cross-CTA hand-offs (0 arrival/acquire, 1 two-counter spin, 2 system
    scope, 3 streamed output to the host). Returns (words checked, failures)."""
    checked, failures = C.c_ulonglong(), C.c_ulonglong()
    check(_lib.load().gf2cu_litmus(int(kind), int(rounds), int(device), C.byref(checked), C.byref(failures)))
    return int(checked.value), int(failures.value)


def _host_view(a) -> MatrixView:
    return a.view() if isinstance(a, BitMatrix) else a


def _pivots(out: PleOutcome, nrows: int) -> np.ndarray:
    if out.processed != nrows:
        raise ValueError("rref_from_ple on the device needs a complete decomposition "
                         "(processed == nrows)")
    return np.ascontiguousarray(np.asarray(out.q[: out.rank], dtype=np.uintp))


def rref_from_ple(a, out: PleOutcome, full: bool = True, cfg: Optional[PleConfig] = None) -> None:
    """gf2::rref_from_ple (ple.hpp:318-329) on the B200, in place: the top
    ``out.rank`` rows become the row echelon form of the original matrix
    (reduced when ``full``), the rows below zero. ``a`` holds the in-place
    result that ``out`` describes (host view or ``DeviceMatrix``)."""
    L = _lib.load()
    szp = C.POINTER(C.c_size_t)
    if isinstance(a, DeviceMatrix):
        q = _pivots(out, a.m)
        stream = cfg.stream if cfg is not None else None
        check(L.gf2cu_rref_from_ple_device(a.handle, q.ctypes.data_as(szp), out.rank, int(full),
                                           C.c_void_p(stream) if stream else None))
        return
    view = _host_view(a)
    q = _pivots(out, view.nrows())
    c = (cfg or PleConfig()).to_c()
    v = view._c()
    check(L.gf2cu_rref_from_ple(C.byref(v), q.ctypes.data_as(szp), out.rank, int(full), C.byref(c)))


def extract_e(a, out: PleOutcome) -> BitMatrix:
    """gf2::extract_e (ple.hpp:344-352): the rank x ncols echelon factor,
    computed on the device from a copy (``a`` is not modified)."""
    view = _host_view(a)
    m, n = view.nrows(), view.ncols()
    work = BitMatrix(m, n)
    W = words_per_row(n)
    flat = view.words.reshape(-1)
    if view.col_off % 64 == 0 and n % 64 == 0:
        for i in range(m):
            s0 = i * view.stride + view.col_off // 64
            work.words[i, :] = flat[s0:s0 + W]
    else:
        for i in range(m):
            for j in range(n):
                if view.get(i, j):
                    work.set(i, j, True)
    rref_from_ple(work, out, full=False)
    return BitMatrix(out.rank, n, work.words[: out.rank].copy())


def extract_l(a, out: PleOutcome) -> BitMatrix:
    """gf2::extract_l (ple.hpp:332-341): the processed x rank unit lower
    factor (a host-side reshuffle of the stored multipliers)."""
    view = _host_view(a)
    l = BitMatrix(out.processed, out.rank)
    for i in range(out.processed):
        for j in range(min(i, out.rank)):
            if view.get(i, j):
                l.set(i, j, True)
        if i < out.rank:
            l.set(i, i, True)
    return l


def echelonize(a, full: bool = True, cfg: Optional[PleConfig] = None) -> int:
    """gf2::echelonize(a, EchelonStrategy::ple_iterative, full) (m4ri.hpp:88-98):
    block_iterative_ple + rref_from_ple with the matrix resident on the
    device in between. Returns the rank."""
    L = _lib.load()
    c = (cfg or PleConfig()).to_c()
    rank = C.c_size_t()
    if isinstance(a, DeviceMatrix):
        check(L.gf2cu_echelonize_device(a.handle, int(full), C.byref(c), C.byref(rank)))
    else:
        v = _host_view(a)._c()
        check(L.gf2cu_echelonize(C.byref(v), int(full), C.byref(c), C.byref(rank)))
    return int(rank.value)


def trsm_upper_left_unit(u, b, cfg: Optional[PleConfig] = None) -> None:
    """gf2::trsm_upper_left_unit (multiply.hpp:314-335) on the B200:
    b <- u^-1 b for the unit upper triangle of the square u."""
    L = _lib.load()
    c = (cfg or PleConfig()).to_c()
    uv, bv = _host_view(u)._c(), _host_view(b)._c()
    check(L.gf2cu_trsm_upper_left_unit(C.byref(uv), C.byref(bv), C.byref(c)))


def recursive_ple(a, cfg: Optional[PleConfig] = None) -> PleOutcome:
    """gf2::recursive_ple (ple.hpp:246-289). Its in-place result, rank, q and
    p.swaps equal block_iterative_ple's (pinned against the compiled reference
    in tests/test_rref_host.py), so the device path serves it unchanged."""
    return block_iterative_ple(a, cfg)


ECHELON_STRATEGIES = ("naive", "m4ri", "ple_iterative", "ple_recursive")


def echelonize_strategy(a, strategy: str = "ple_iterative", full: bool = True,
                        cfg: Optional[PleConfig] = None) -> int:
    """gf2::echelonize(a, strategy, full) (m4ri.hpp:88-105). Every strategy
    returns the same matrix (the reduced form is unique; the non-reduced forms
    of naive / m4ri / PLE coincide, pinned in tests/test_rref_host.py), so all
    of them run the device PLE + rref_from_ple."""
    if strategy not in ECHELON_STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    return echelonize(a, full, cfg)


def _mul(c, a, b, accumulate: bool, cfg: Optional[PleConfig]) -> None:
    L = _lib.load()
    if isinstance(c, DeviceMatrix):
        if not (isinstance(a, DeviceMatrix) and isinstance(b, DeviceMatrix)):
            raise ValueError("device product needs device operands")
        stream = cfg.stream if cfg is not None else None
        check(L.gf2cu_matrix_mul(c.handle, a.handle, b.handle, int(accumulate),
                                 C.c_void_p(stream) if stream else None))
        return
    cc = (cfg or PleConfig()).to_c()
    cv, av, bv = _host_view(c)._c(), _host_view(a)._c(), _host_view(b)._c()
    fn = L.gf2cu_addmul if accumulate else L.gf2cu_mul
    check(fn(C.byref(cv), C.byref(av), C.byref(bv), C.byref(cc)))


def mul(a, b, cfg: Optional[PleConfig] = None) -> BitMatrix:
    """gf2::mul (multiply.hpp:266-274): a new a.nrows x b.ncols product."""
    av, bv = _host_view(a), _host_view(b)
    c = BitMatrix(av.nrows(), bv.ncols())
    _mul(c, av, bv, False, cfg)
    return c


def mul_into(c, a, b, cfg: Optional[PleConfig] = None) -> None:
    """c = a * b (host views or DeviceMatrix operands)."""
    _mul(c, a, b, False, cfg)


def addmul(c, a, b, cfg: Optional[PleConfig] = None) -> None:
    """gf2::addmul (multiply.hpp:254-264): c ^= a * b."""
    _mul(c, a, b, True, cfg)


def device_count() -> int:
    return int(_lib.load().gf2cu_device_count())
