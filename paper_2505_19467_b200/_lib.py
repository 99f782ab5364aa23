"""ctypes binding of the kbe200 C ABI (include/kbe200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  Loading fails loudly: there is no CPU fallback for any operator.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KBE_LIB") or os.environ.get("KBE200_LIB", os.path.join(_HERE, "libkbe200.so"))

KBE_OK, KBE_ERR_ARG, KBE_ERR_CUDA, KBE_ERR_UNSUPPORTED = 0, 1, 2, 3
MAX_ITER = 16
MAX_NK = 128       # KBE_MAX_NK: largest n_k of the Sigma kernel
MAX_RANKS = 8
TILE_B = 32
TILE_S = 32
COL_CHUNK = 8
REPORT_W = 32
TAIL_CPLX = 16     # per-rank control tail of the all-gather chunk (KBE_TAIL_CPLX)
ABI_VERSION = 11

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64


class KbeProblem(ctypes.Structure):
    """Mirror of ``struct kbe_problem`` (include/kbe200.h)."""

    _fields_ = [
        ("n_k", _i32), ("k_lo", _i32), ("k_hi", _i32), ("n_steps", _i32),
        ("quad", _i32), ("limit_mode", _i32), ("hf", _i32), ("max_iter", _i32),
        ("interacting", _i32), ("nbb", _i32), ("nsb", _i32), ("pad0", _i32),
        ("dt", ctypes.c_double), ("eps", ctypes.c_double),
        ("dipole_re", ctypes.c_double), ("dipole_im", ctypes.c_double),
        ("tri", _i64),
        ("g_hist", _p), ("s_hist", _p),
        ("eps_v", _p), ("eps_c", _p), ("u_table", _p), ("u_mid", _p), ("amp", _p),
        ("row_part", _p), ("col_part", _p), ("gc_part", _p),
        ("lr_old", _p), ("col_old", _p),
        ("front_send", _p), ("front_all", _p),
        ("ctl", _p), ("reports", _p), ("phi", _p),
        ("row_part_g", _p), ("col_part_g", _p), ("lc_part", _p), ("gc_part_c", _p), ("lc_part_c", _p),
        ("g_sh", _p), ("s_sh", _p), ("v_prev", _p), ("fcol_part", _p),
        ("row_delta", _p), ("col_delta", _p), ("gc_delta", _p), ("i_red", _p), ("g_red", _p),
        ("p2p_world", _i32), ("p2p_rank", _i32), ("p2p_local", _p), ("p2p_peers", _p * 8),
    ]


# name -> (restype, argtypes); every symbol include/kbe200.h declares
SIGNATURES = {
    "kbe_abi_version": (ctypes.c_int, []),
    "kbe_plane_len": (_i64, [_i32]),
    "kbe_slice_offset": (_i64, [_i32]),
    "kbe_tri_size": (_i64, [_i32]),
    "kbe_ctl_bytes": (_i64, []),
    "kbe_sizeof_problem": (_i64, []),
    "kbe_last_error": (ctypes.c_char_p, []),
    "kbe_init_history": (ctypes.c_int, [_p, _p]),
    "kbe_sigma_frontier": (ctypes.c_int, [_p, _i32, _i32, _p]),
    "kbe_sigma_slice": (ctypes.c_int, [_i32, _i32, _p, _p, _p, _p, _i32, _i32, _p, _p, _p, _p, _p, _p]),
    "kbe_collision_frontier": (ctypes.c_int, [_p, _i32, _i32, _p]),
    "kbe_collision_slice": (ctypes.c_int, [_p, _i32, _p, _p, _p, _p, _p]),
    "kbe_collision_row": (ctypes.c_int, [_i32, _i32, _i32, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p]),
    "kbe_update": (ctypes.c_int, [_p, _i32, _i32, _i32, _p]),
    "kbe_hf_mean": (ctypes.c_int, [_p, _i32, _i32, _i32, _p]),
    "kbe_build_phi": (ctypes.c_int, [_p, _i32, _i32, _p]),
    "kbe_finish_step": (ctypes.c_int, [_p, _i32, _p]),
    "kbe_step": (ctypes.c_int, [_p, _i32, _p]),
    "kbe_run": (ctypes.c_int, [_p, _i32, _i32, _i32, _p]),
    "kbe_release": (ctypes.c_int, [_p]),
    "kbe_run_iters": (ctypes.c_int, [_p, _i32, _i32, _i32, _p]),
    "kbe_resume_step": (ctypes.c_int, [_p, _i32, _i32, _p]),
    "kbe_ctl_needs_more_offset": (_i64, []),
    "kbe_ctl_hf_sum_offset": (_i64, []),
    "kbe_max_n_k": (_i32, []),
    "kbe_set_sigma_variant": (ctypes.c_int, [_i32]),
    "kbe_launches_per_eval": (ctypes.c_int, [_p]),
    "kbe_p2p_bytes": (_i64, [_p, _i32]),
    "kbe_p2p_alloc": (ctypes.c_int, [_i64, ctypes.POINTER(_p), _p]),
    "kbe_p2p_open": (ctypes.c_int, [_p, ctypes.POINTER(_p)]),
    "kbe_p2p_close": (ctypes.c_int, [_p]),
    "kbe_p2p_free": (ctypes.c_int, [_p]),
    "kbe_p2p_publish": (ctypes.c_int, [_p, _p]),
    "kbe_p2p_read_u64": (ctypes.c_int, [_p, _p]),
    "kbe_unpack": (ctypes.c_int, [_p, _i64, _i32, _i32, _i32, _i32, _p, _p]),
    "kbe_pack": (ctypes.c_int, [_p, _p, _i32, _i32, _i32, _i64, _p, _p]),
    "kbe_unpack_retarded": (ctypes.c_int, [_p, _i64, _i32, _i32, _i32, ctypes.c_double, _p, _p]),
}

_lib = None


def lib():
    """Load libkbe200.so once; raise if it is missing or ABI-incompatible."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"kbe200 CUDA extension not built: {LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`); there is no CPU fallback"
        )
    handle = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.kbe_abi_version() != ABI_VERSION:
        raise RuntimeError(f"kbe200 ABI mismatch: library {handle.kbe_abi_version()} vs binding {ABI_VERSION}")
    if handle.kbe_sizeof_problem() != ctypes.sizeof(KbeProblem):
        raise RuntimeError("kbe200 struct layout mismatch (kbe_problem)")
    _lib = handle
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map a C status onto the reference's exception types."""
    if rc == KBE_OK:
        return
    msg = lib().kbe_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == KBE_ERR_ARG:
        raise ValueError(msg)
    if rc == KBE_ERR_UNSUPPORTED:
        raise ConfigError(msg)
    raise RuntimeError(f"CUDA error in kbe200: {msg}")


def tri_size(n_steps: int) -> int:
    return int(lib().kbe_tri_size(n_steps))


def plane_len(s: int) -> int:
    """Padded points per plane of slice s (whole 32-point blocks)."""
    return (s // 32 + 1) * 32


def slice_offset(s: int) -> int:
    q, r = divmod(s, 32)
    return 256 * (q + 1) * (16 * q + r)


def slice_index(c: int, b: int) -> int:
    """Element of (plane c, point b) inside a slice: blocks of 8 planes x 32 points."""
    return (b // 32) * 256 + c * 32 + b % 32
