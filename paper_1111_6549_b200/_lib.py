"""Loader and builder for the in-tree CUDA library ``libgf2cu.so``.

The library is the product: hand-written sm_100a kernels behind the C ABI of
``include/gf2cu.h``. It is built in-tree (nvcc, ``-gencode
arch=compute_100a,code=sm_100a``) so the built ``.so`` travels with the repo
to the GPU box. There is no CPU fallback: if the library is missing or no
sm_100 device is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO = os.path.join(PKG, "libgf2cu.so")
SRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp", "-lgomp", "-cudart", "static",
]


def sources():
    return [os.path.join(SRC, f) for f in sorted(os.listdir(SRC)) if f.endswith(".cu")]


def _deps():
    return [os.path.join(SRC, f) for f in os.listdir(SRC)] + [os.path.join(INCLUDE, "gf2cu.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libgf2cu.so for sm_100a (cross-compiles without a GPU)."""
    if not force and not needs_build():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    cmd = [nvcc, *NVCC_FLAGS, "-I" + INCLUDE, "-o", SO + ".tmp", *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out.stdout + out.stderr)
    os.replace(SO + ".tmp", SO)
    if verbose:
        print(out.stdout + out.stderr)
    return SO


class gf2cu_view(C.Structure):
    _fields_ = [("data", C.POINTER(C.c_uint64)), ("stride", C.c_size_t), ("col_off", C.c_size_t),
                ("nrows", C.c_size_t), ("ncols", C.c_size_t)]


class gf2cu_cfg(C.Structure):
    _fields_ = [("k", C.c_uint), ("k_scale", C.c_double), ("table_count", C.c_uint),
                ("device", C.c_int), ("stream", C.c_void_p), ("flags", C.c_uint)]


class gf2cu_colswap(C.Structure):
    _fields_ = [("a", C.c_size_t), ("b", C.c_size_t), ("from_row", C.c_size_t)]


class gf2cu_stats(C.Structure):
    _fields_ = [("steps", C.c_size_t), ("trailing_launches", C.c_size_t),
                ("trailing_ms", C.c_double), ("panel_ms", C.c_double), ("coef_ms", C.c_double),
                ("alg_bytes", C.c_double), ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double),
                ("kernel_ms", C.c_double), ("driver", C.c_int), ("sweep_bytes", C.c_double),
                ("input_first_rows", C.c_size_t), ("input_first_steps", C.c_size_t),
                ("input_blocks", C.c_size_t)]


FLAG_TIME_KERNELS = 1
FLAG_MULTI_KERNEL = 2
FLAG_SINGLE_PANEL = 4
FLAG_SUPER_STEP = 8
FLAG_CHECK = 32
PEER_HANDLE_BYTES = 64  # GF2CU_PEER_HANDLE_BYTES


def FLAG_PEER_RANKS(g: int) -> int:
    return (int(g) & 15) << 16

# name -> (restype, argtypes): every symbol include/gf2cu.h declares.
_sz, _szp = C.c_size_t, C.POINTER(C.c_size_t)
_u64p = C.POINTER(C.c_uint64)
_mp = C.c_void_p
SYMBOLS = {
    "gf2cu_default_config": (None, [C.POINTER(gf2cu_cfg)]),
    "gf2cu_ple": (C.c_int, [C.POINTER(gf2cu_view), C.POINTER(gf2cu_cfg), _szp, _szp, _szp,
                            C.POINTER(gf2cu_colswap), _szp, C.POINTER(gf2cu_stats)]),
    "gf2cu_partial_ple": (C.c_int, [C.POINTER(gf2cu_view), C.POINTER(gf2cu_cfg), _szp, _szp, _szp, _szp,
                                    C.POINTER(gf2cu_colswap), _szp]),
    "gf2cu_undo_column_swaps": (C.c_int, [C.POINTER(gf2cu_view), C.POINTER(gf2cu_colswap), _sz,
                                          C.POINTER(gf2cu_cfg)]),
    "gf2cu_undo_column_swaps_device": (C.c_int, [_mp, C.POINTER(gf2cu_colswap), _sz, C.c_void_p]),
    "gf2cu_last_error": (C.c_char_p, []),
    "gf2cu_device_count": (C.c_int, []),
    "gf2cu_version": (C.c_char_p, []),
    "gf2cu_matrix_create": (C.c_int, [_sz, _sz, C.c_int, C.POINTER(_mp)]),
    "gf2cu_matrix_destroy": (C.c_int, [_mp]),
    "gf2cu_matrix_info": (C.c_int, [_mp, _szp, _szp, _szp, C.POINTER(_u64p)]),
    "gf2cu_matrix_upload": (C.c_int, [_mp, _u64p, _sz, C.c_void_p]),
    "gf2cu_matrix_download": (C.c_int, [_mp, _u64p, _sz, C.c_void_p]),
    "gf2cu_matrix_copy": (C.c_int, [_mp, _mp, C.c_void_p]),
    "gf2cu_matrix_fill_ctr": (C.c_int, [_mp, C.c_uint64, C.c_void_p]),
    "gf2cu_matrix_checksum": (C.c_int, [_mp, _u64p, C.c_void_p]),
    "gf2cu_ple_device": (C.c_int, [_mp, C.POINTER(gf2cu_cfg), _szp, _szp, _szp,
                                   C.POINTER(gf2cu_colswap), _szp, C.POINTER(gf2cu_stats)]),
    "gf2cu_rref_from_ple": (C.c_int, [C.POINTER(gf2cu_view), _szp, _sz, C.c_int, C.POINTER(gf2cu_cfg)]),
    "gf2cu_rref_from_ple_device": (C.c_int, [_mp, _szp, _sz, C.c_int, C.c_void_p]),
    "gf2cu_echelonize": (C.c_int, [C.POINTER(gf2cu_view), C.c_int, C.POINTER(gf2cu_cfg), _szp]),
    "gf2cu_echelonize_device": (C.c_int, [_mp, C.c_int, C.POINTER(gf2cu_cfg), _szp]),
    "gf2cu_trsm_upper_left_unit": (C.c_int, [C.POINTER(gf2cu_view), C.POINTER(gf2cu_view),
                                             C.POINTER(gf2cu_cfg)]),
    "gf2cu_mul": (C.c_int, [C.POINTER(gf2cu_view)] * 3 + [C.POINTER(gf2cu_cfg)]),
    "gf2cu_addmul": (C.c_int, [C.POINTER(gf2cu_view)] * 3 + [C.POINTER(gf2cu_cfg)]),
    "gf2cu_matrix_mul": (C.c_int, [_mp, _mp, _mp, C.c_int, C.c_void_p]),
    "gf2cu_shard_create": (C.c_int, [_sz, _sz, C.c_int, C.c_int, _sz, C.c_int, C.POINTER(_mp)]),
    "gf2cu_shard_destroy": (C.c_int, [_mp]),
    "gf2cu_shard_info": (C.c_int, [_mp, _szp, _szp]),
    "gf2cu_shard_upload": (C.c_int, [_mp, _u64p, _sz, C.c_void_p]),
    "gf2cu_shard_download": (C.c_int, [_mp, _u64p, _sz, C.c_void_p]),
    "gf2cu_shard_begin": (C.c_int, [_mp, C.c_void_p]),
    "gf2cu_shard_fill_ctr": (C.c_int, [_mp, C.c_uint64, C.c_void_p]),
    "gf2cu_shard_gather": (C.c_int, [_mp, _u64p, _sz, _sz, C.c_void_p]),
    "gf2cu_shard_panel": (C.c_int, [_mp, _sz, _u64p, C.c_int, C.POINTER(C.c_uint32), C.c_void_p]),
    "gf2cu_shard_apply": (C.c_int, [_mp, _sz, _u64p, C.c_void_p]),
    "gf2cu_shard_pack_stage": (C.c_int, [_mp, _sz, C.c_void_p]),
    "gf2cu_shard_step_gather": (C.c_int, [_mp, _sz, _u64p, C.c_void_p]),
    "gf2cu_shard_step_panel": (C.c_int, [_mp, _sz, _u64p, C.c_void_p]),
    "gf2cu_shard_step_update": (C.c_int, [_mp, _sz, C.c_void_p]),
    "gf2cu_shard_set_stage": (C.c_int, [_mp, _u64p]),
    "gf2cu_shard_pivots": (C.c_int, [_mp, _szp, C.c_void_p]),
    "gf2cu_shard_unpack": (C.c_int, [_mp, _sz, C.c_uint64, _u64p, C.c_void_p]),
    "gf2cu_shard_trailing": (C.c_int, [_mp, _sz, C.c_void_p]),
    "gf2cu_shard_finish": (C.c_int, [_mp, _szp, _szp, _szp, C.POINTER(C.c_uint32), C.c_void_p]),
    "gf2cu_peer_create": (C.c_int, [_sz, _sz, C.c_int, C.c_int, _sz, C.c_int, C.POINTER(_mp)]),
    "gf2cu_peer_destroy": (C.c_int, [_mp]),
    "gf2cu_peer_info": (C.c_int, [_mp, _szp]),
    "gf2cu_peer_export": (C.c_int, [_mp, C.c_void_p]),
    "gf2cu_peer_connect": (C.c_int, [_mp, C.c_void_p]),
    "gf2cu_peer_upload": (C.c_int, [_mp, _u64p, _sz, C.c_void_p]),
    "gf2cu_peer_download": (C.c_int, [_mp, _u64p, _sz, C.c_void_p]),
    "gf2cu_peer_fill_ctr": (C.c_int, [_mp, C.c_uint64, C.c_void_p]),
    "gf2cu_peer_reset": (C.c_int, [_mp, C.c_void_p]),
    "gf2cu_peer_ping": (C.c_int, [_mp, C.c_uint32, C.POINTER(C.c_uint32)]),
    "gf2cu_peer_run": (C.c_int, [_mp, C.c_void_p, C.POINTER(gf2cu_stats)]),
    "gf2cu_peer_finish": (C.c_int, [_mp, _szp, _szp, _szp, C.POINTER(C.c_uint32), C.c_void_p]),
    "gf2cu_litmus": (C.c_int, [C.c_int, C.c_uint, C.c_int, C.POINTER(C.c_ulonglong),
                               C.POINTER(C.c_ulonglong)]),
    "gf2cu_stream_in_plan": (C.c_int, [_sz, _sz, C.c_int, _szp, C.POINTER(C.c_uint), _szp]),
    "gf2cu_fill_random": (C.c_int, [_u64p, _sz, _sz, _sz, C.c_double, C.c_uint64]),
    "gf2cu_fill_ctr": (C.c_int, [_u64p, _sz, _sz, _sz, C.c_uint64]),
    "gf2cu_fill_random_rows": (C.c_int, [_u64p, _sz, _sz, _sz, _sz, C.c_uint64]),
}

_lib = None


def load(build_if_missing: bool = True):
    """Load libgf2cu.so (building it first if it is missing and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO):
        if not build_if_missing:
            raise RuntimeError(f"{SO} is missing; run __graft_entry__.build()")
        build()
    L = C.CDLL(SO)
    for name, (res, args) in SYMBOLS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class Gf2cuError(RuntimeError):
    pass


class Gf2cuCheckError(Gf2cuError):
    """GF2CU_ECHECK: check mode found a violated device invariant."""


def check(status: int) -> None:
    """Map a gf2cu_status to the exception the reference would raise."""
    if status == 0:
        return
    msg = load().gf2cu_last_error().decode(errors="replace")
    if status == 1:
        raise ValueError(msg)          # std::invalid_argument
    if status == 2:
        raise IndexError(msg)          # std::out_of_range
    if status == 3:
        raise MemoryError(msg)         # std::bad_alloc
    if status == 6:
        raise Gf2cuCheckError(msg)
    raise Gf2cuError(f"gf2cu status {status}: {msg}")
