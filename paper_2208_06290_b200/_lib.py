"""ctypes binding of the sm_100a C ABI (include/hodlr_b200.h).

The library is built in-tree (``make`` / ``__graft_entry__.build()``) into
``paper_2208_06290_b200/lib/libhodlr_b200.so``.  There is deliberately no CPU
fallback: if the library is missing or no CUDA device is present, every
compute entry point raises :class:`HodlrNativeError`.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libhodlr_b200.so"

OK, ERR_ARG, ERR_SHAPE, ERR_SINGULAR, ERR_CUDA, ERR_NCCL = range(6)
PHASES = ("leaf_getrf", "leaf_apply", "k_getrf", "k_apply", "level", "gemm", "solve_leaf", "solve_k", "solve_level")
F64, F32 = 0, 1

_STATUS = {
    ERR_ARG: "invalid argument",
    ERR_SHAPE: "shape mismatch",
    ERR_SINGULAR: "singular block",
    ERR_CUDA: "CUDA error",
    ERR_NCCL: "NCCL error",
}


class HodlrNativeError(RuntimeError):
    """The native CUDA library is unavailable or returned an error status."""


class Desc(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int32), ("r", C.c_int32), ("L", C.c_int32), ("dtype", C.c_int32),
                ("ranks", C.c_void_p)]


def make_desc(n: int, m: int, r: int, L: int, dtype: int, ranks=None) -> Desc:
    """hodlr_desc; ``ranks`` (per-level ranks, level l' at ranks[l'-1]) is kept
    alive on the returned structure."""
    d = Desc(n, m, r, L, dtype, None)
    if ranks is not None:
        arr = (C.c_int32 * len(ranks))(*[int(x) for x in ranks])
        d.ranks = C.cast(arr, C.c_void_p)
        d._ranks_keep = arr
    return d


class Factors(C.Structure):
    _fields_ = [
        ("D", C.c_void_p), ("Dinv", C.c_void_p), ("Y", C.c_void_p), ("V", C.c_void_p),
        ("K", C.c_void_p), ("Kinv", C.c_void_p),
        ("dswaps", C.c_void_p), ("dperm", C.c_void_p), ("dinfo", C.c_void_p),
        ("kswaps", C.c_void_p), ("kperm", C.c_void_p), ("kinfo", C.c_void_p),
    ]


# exported symbols and their ctypes signatures (must match include/hodlr_b200.h)
_i, _i64, _p, _d, _sz = C.c_int, C.c_int64, C.c_void_p, C.c_double, C.c_size_t
SIGNATURES = {
    "hodlr_version": (C.c_char_p, []),
    "hodlr_last_error": (C.c_char_p, []),
    "hodlr_inv_elems": (_sz, [_i]),
    "hodlr_getrf_batched": (_i, [_i, _i, _i, _p, _i64, _i64, _p, _p, _p, _p, _i64, _i64, _p]),
    "hodlr_getrs_batched": (_i, [_i, _i, _i, _i, _p, _i64, _i64, _p, _p, _i64, _i64, _p]),
    "hodlr_gemm_batched": (
        _i,
        [_i, _i, _i, _i, _i, _d, _p, _i64, _i64, _i64, _p, _i64, _i64, _i64, _d, _p, _i64, _i64, _i64, _i, _i, _p, _sz, _p],
    ),
    "hodlr_launch_count": (C.c_longlong, []),
    "hodlr_profile_enable": (None, [_i]),
    "hodlr_profile_read": (_i, [C.POINTER(C.c_double), _i]),
    "hodlr_factorize_workspace": (_sz, [C.POINTER(Desc)]),
    "hodlr_solve_workspace": (_sz, [C.POINTER(Desc), _i]),
    "hodlr_factorize": (_i, [C.POINTER(Desc), C.POINTER(Factors), _p, _sz, _p]),
    "hodlr_factorize_from_host": (_i, [C.POINTER(Desc), C.POINTER(Factors), _p, _p, _p, _p, _sz, _p, _p]),
    "hodlr_factorize_local_workspace": (_sz, [C.POINTER(Desc), _i64]),
    "hodlr_factorize_local": (_i, [C.POINTER(Desc), C.POINTER(Factors), _i64, _i64, _i, _p, _p, _sz, _p]),
    "hodlr_factorize_top": (_i, [C.POINTER(Desc), C.POINTER(Factors), _i64, _i64, _i, _p, _p, _p, _sz, _p]),
    "hodlr_solve_local": (_i, [C.POINTER(Desc), C.POINTER(Factors), _i64, _i64, _i, _p, _i64, _i, _p, _p, _sz, _p]),
    "hodlr_solve_top": (_i, [C.POINTER(Desc), C.POINTER(Factors), _i64, _i64, _i, _p, _p, _p, _i64, _i, _p, _sz, _p]),
    "hodlr_solve": (_i, [C.POINTER(Desc), C.POINTER(Factors), _p, _i64, _i, _p, _sz, _p]),
    "hodlr_matvec_workspace": (_sz, [C.POINTER(Desc), _i]),
    "hodlr_matvec": (_i, [C.POINTER(Desc), _p, _p, _p, _p, _i64, _p, _i64, _i, _p, _sz, _p]),
    "hodlr_build_workspace": (_sz, [C.POINTER(Desc)]),
    "hodlr_xorshift_uniform": (_i, [C.c_uint64, _i64, _p, _p]),
    "hodlr_build_laplace_dl": (_i, [C.POINTER(Desc), _p, _p, _p, _p, _p, _sz, _p]),
    "hodlr_build_dense": (_i, [C.POINTER(Desc), _p, _i64, _p, _p, _p, _p, _sz, _p]),
    "hodlr_build_gaussian": (_i, [C.POINTER(Desc), _p, _i, _d, _d, _p, _p, _p, _p, _sz, _p]),
    "hodlr_build_schur_plane": (_i, [C.POINTER(Desc), _p, _d, _p, _p, _p, _p, _sz, _p]),
    "hodlr_transpose_f64": (_i, [_p, _i64, _i64, _i64, _p, _i64, _p]),
}

_lib = None


def load(path: os.PathLike | None = None) -> C.CDLL:
    """Load (once) and type the native library; raise loudly if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise HodlrNativeError(
            f"native library {p} not built; run `make` (or __graft_entry__.build()) -- there is no CPU fallback"
        )
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != OK:
        lib = load()
        detail = lib.hodlr_last_error().decode() if status == ERR_CUDA else ""
        raise HodlrNativeError(f"{what}: {_STATUS.get(status, status)} {detail}".strip())


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise HodlrNativeError("no CUDA device: the HODLR B200 engine has no CPU path")
    load()
    return torch
