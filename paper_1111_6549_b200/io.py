"""gf2b / ASCII matrix files, the host-side mirror of
gf2/io.hpp (io.hpp:14-124).

Binary "gf2b" (io.hpp:16-24): bytes 0..4 magic 'G' 'F' '2' 'B' 0x01; bytes
5..12 nrows and 13..20 ncols as little-endian u64; then nrows * ceil(ncols/64)
little-endian words. Loads reject bad magic, truncated headers or data,
implausible dimensions (> 2^32), dirty padding bits past ncols and trailing
bytes (io.hpp:75-90). Text "ascii" (io.hpp:26-27): "nrows ncols\\n" then one
line of '0'/'1' per row (io.hpp:92-110). load_matrix autodetects by magic
(io.hpp:113-122). Every failure raises IoError (io.hpp:32-34).

This is file I/O, not compute: numpy does the packing. load_gf2b_device reads
a gf2b file straight into HBM.
"""
from __future__ import annotations

import io as _io
import os
from typing import BinaryIO, Union

import numpy as np

from .ple import BitMatrix, DeviceMatrix, words_per_row

MAGIC = b"GF2B\x01"
PathOrFile = Union[str, os.PathLike, BinaryIO]


class IoError(RuntimeError):
    """gf2::io_error (io.hpp:32-34)."""


def _open(f: PathOrFile, mode: str):
    if isinstance(f, (str, os.PathLike)):
        return open(f, mode), True
    return f, False


def _padding_clean(words: np.ndarray, ncols: int) -> bool:
    """BitMatrix::padding_clean: no bits past ncols in the last word of a row."""
    if ncols % 64 == 0 or words.shape[0] == 0:
        return True
    mask = np.uint64(~((1 << (ncols % 64)) - 1) & 0xFFFFFFFFFFFFFFFF)
    return not np.any(words[:, -1] & mask)


def save_gf2b(f: PathOrFile, a: BitMatrix) -> None:
    """gf2::save_gf2b (io.hpp:59-66)."""
    fh, own = _open(f, "wb")
    try:
        fh.write(MAGIC)
        fh.write(np.array([a.nrows(), a.ncols()], dtype="<u8").tobytes())
        fh.write(np.ascontiguousarray(a.words, dtype="<u8").tobytes())
    except OSError as e:
        raise IoError("write failed") from e
    finally:
        if own:
            fh.close()


def _read_gf2b_words(fh) -> tuple[int, int, np.ndarray]:
    if fh.read(5) != MAGIC:
        raise IoError("bad magic")
    hdr = fh.read(16)
    if len(hdr) != 16:
        raise IoError("truncated header")
    rows, cols = (int(x) for x in np.frombuffer(hdr, dtype="<u8"))
    if rows > (1 << 32) or cols > (1 << 32):
        raise IoError("header dimensions implausibly large")
    W = words_per_row(cols)
    nbytes = rows * W * 8
    data = fh.read(nbytes)
    if len(data) != nbytes:
        raise IoError("truncated header")  # the reference's get_u64_le message
    words = np.frombuffer(data, dtype="<u8").astype(np.uint64).reshape(rows, W)
    if not _padding_clean(words, cols):
        raise IoError("nonzero bits in row padding")
    if fh.read(1):
        raise IoError("trailing bytes after matrix data")
    return rows, cols, words


def load_gf2b(f: PathOrFile) -> BitMatrix:
    """gf2::load_gf2b (io.hpp:75-90)."""
    fh, own = _open(f, "rb")
    try:
        rows, cols, words = _read_gf2b_words(fh)
    finally:
        if own:
            fh.close()
    return BitMatrix(rows, cols, words.copy())


def load_gf2b_device(f: PathOrFile, device: int = 0) -> DeviceMatrix:
    """A gf2b file straight into a DeviceMatrix (HBM)."""
    fh, own = _open(f, "rb")
    try:
        rows, cols, words = _read_gf2b_words(fh)
    finally:
        if own:
            fh.close()
    d = DeviceMatrix(rows, cols, device)
    if rows and cols:
        d.upload(np.ascontiguousarray(words))
    return d


def save_ascii(f: PathOrFile, a: BitMatrix) -> None:
    """gf2::save_ascii (io.hpp:68-76)."""
    fh, own = _open(f, "wb")
    try:
        m, n = a.nrows(), a.ncols()
        fh.write(f"{m} {n}\n".encode())
        if m and n:
            bits = np.unpackbits(a.words.view(np.uint8), axis=1, bitorder="little")[:, :n]
            chars = (bits + ord("0")).astype(np.uint8)
            out = np.concatenate([chars, np.full((m, 1), ord("\n"), np.uint8)], axis=1)
            fh.write(out.tobytes())
        elif m:
            fh.write(b"\n" * m)
    except OSError as e:
        raise IoError("write failed") from e
    finally:
        if own:
            fh.close()


def load_ascii(f: PathOrFile) -> BitMatrix:
    """gf2::load_ascii (io.hpp:92-110)."""
    fh, own = _open(f, "rb")
    try:
        text = fh.read()
    finally:
        if own:
            fh.close()
    return _parse_ascii(text)


def _parse_ascii(text: bytes) -> BitMatrix:
    """Stream semantics of load_ascii: `in >> rows >> cols` (whitespace
    skipped), ignore to the end of that line, then std::getline per row
    (fails only at end of input with nothing read; a trailing '\r' dropped)."""
    pos, n = 0, len(text)

    def number() -> int:
        nonlocal pos
        while pos < n and text[pos:pos + 1].isspace():
            pos += 1
        start = pos
        while pos < n and 48 <= text[pos] <= 57:
            pos += 1
        if pos == start:
            raise IoError("bad text header")
        return int(text[start:pos])

    rows = number()
    cols = number()
    nl = text.find(b"\n", pos)
    pos = n if nl < 0 else nl + 1
    a = BitMatrix(rows, cols)
    for i in range(rows):
        if pos >= n:
            raise IoError("truncated text matrix")
        nl = text.find(b"\n", pos)
        line = text[pos:] if nl < 0 else text[pos:nl]
        pos = n if nl < 0 else nl + 1
        if line.endswith(b"\r"):
            line = line[:-1]
        if len(line) != cols:
            raise IoError("row length mismatch")
        arr = np.frombuffer(line, dtype=np.uint8)
        if np.any((arr != ord("0")) & (arr != ord("1"))):
            raise IoError("row contains characters other than 0/1")
        if cols:
            packed = np.packbits((arr == ord("1")).astype(np.uint8), bitorder="little")
            buf = np.zeros(a.stride() * 8, dtype=np.uint8)
            buf[: packed.size] = packed
            a.words[i] = buf.view(np.uint64)
    return a


def load_matrix(f: PathOrFile) -> BitMatrix:
    """gf2::load_matrix (io.hpp:113-122): gf2b by magic, else ASCII."""
    fh, own = _open(f, "rb")
    try:
        data = fh.read()
    finally:
        if own:
            fh.close()
    if data[:5] == MAGIC:
        return load_gf2b(_io.BytesIO(data))
    return _parse_ascii(data)
