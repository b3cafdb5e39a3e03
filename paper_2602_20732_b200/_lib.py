"""ctypes binding of libchess_b200.so (the C-ABI in include/chess_b200.h).

This is the same binding a maintainer would add to the reference package
(INTEGRATION.md): plain structs of device pointers and sizes, int status
codes mapped 1:1 onto the pagesel exception classes.  There is no fallback:
if the shared library is missing or fails to load, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import (
    ConfigurationError,
    EmptyContextError,
    OutOfPagesError,
    PageSelError,
)

LIB_PATH = Path(__file__).resolve().parent / "libchess_b200.so"
ABI_VERSION = 5

# enum ChessStatus
OK, ERR_CONFIG, ERR_OUT_OF_PAGES, ERR_EMPTY_CONTEXT, ERR_SHAPE, ERR_INDEX, ERR_ORDER, ERR_VALUE, ERR_CUDA, ERR_UNSUPPORTED = range(10)
# enum ChessDtype
F32, F64, BF16 = 0, 1, 2
# enum ChessPolicy
POLICY_NEVER, POLICY_ALWAYS, POLICY_FIXED, POLICY_DYNAMIC, POLICY_EVERY_STEP = range(5)
# enum ChessProvenance
PROV_NONE, PROV_SEMANTIC, PROV_WINDOW, PROV_SINK = range(4)
PROV_NAMES = {PROV_SEMANTIC: "semantic", PROV_WINDOW: "window", PROV_SINK: "sink"}


class ChessDims(C.Structure):
    _fields_ = [
        ("batch", C.c_int32),
        ("layers", C.c_int32),
        ("kv_heads", C.c_int32),
        ("q_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("page_size", C.c_int32),
        ("pages_per_chunk", C.c_int32),
        ("chunks_per_grid", C.c_int32),
        ("max_pages", C.c_int32),
        ("window_pages", C.c_int32),
        ("max_ws", C.c_int32),
        ("summary_dtype", C.c_int32),
        ("dim", C.c_int64),
        ("ld", C.c_int64),
        ("n_phys", C.c_int64),
    ]


STATE_POINTERS = [
    "k_pool", "v_pool", "page_table", "num_pages", "tail_fill", "token_count",
    "sink_count", "sealed", "num_sealed", "page_vec64", "chunk_sum64", "grid_sum64",
    "chunk_vec64", "grid_vec64", "page_vec32", "chunk_vec32", "grid_vec32", "key_sum",
    "anchor", "semantic", "n_semantic", "sel_stats", "ws_logical", "block_table",
    "ws_prov", "ws_len", "ent_ring", "ent_count", "gen_pages", "page_stats", "fire", "trigger_count",
    "pool_free", "pool_top", "pool_base", "pool_end", "pool_oom",
    "workspace",
]


class ChessState(C.Structure):
    _fields_ = [("d", ChessDims)] + [(n, C.c_void_p) for n in STATE_POINTERS] + [
        ("workspace_bytes", C.c_size_t)
    ]


class ChessSelectCfg(C.Structure):
    _fields_ = [
        ("rho_grid", C.c_double),
        ("rho_chunk", C.c_double),
        ("rho_page", C.c_double),
        ("full_scan", C.c_int32),
        ("force_all", C.c_int32),
        ("defer_ws", C.c_int32),
        ("pad_", C.c_int32),
    ]


class ChessPeerExchange(C.Structure):
    _fields_ = [
        ("world", C.c_int32),
        ("rank", C.c_int32),
        ("ld", C.c_int64),
        ("recv", C.c_void_p),
        ("flags", C.c_void_p),
        ("my_recv", C.c_void_p),
        ("my_flags", C.c_void_p),
        ("gen", C.c_void_p),
        ("err", C.c_void_p),
    ]


class ChessPeerOutputs(C.Structure):
    _fields_ = [
        ("world", C.c_int32),
        ("rank", C.c_int32),
        ("regions", C.POINTER(C.c_void_p)),
        ("flags", C.c_void_p),
        ("my_flags", C.c_void_p),
        ("gen", C.c_void_p),
        ("err", C.c_void_p),
    ]


class ChessTriggerCfg(C.Structure):
    _fields_ = [
        ("policy", C.c_int32),
        ("interval", C.c_int32),
        ("mode", C.c_int32),
        ("pad_", C.c_int32),
        ("tau_entropy", C.c_double),
        ("tau_varentropy", C.c_double),
    ]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_F = C.c_float
_U32 = C.c_uint32

# launch-ordering flag of chess_sparse_decode_ex (include/chess_b200.h)
ATTN_AFTER_DECODE = 1

# name -> (restype, argtypes).  Exactly the symbols declared in include/chess_b200.h.
SIGNATURES = {
    "chess_abi_version": (C.c_int, []),
    "chess_dims_sizeof": (C.c_size_t, []),
    "chess_state_sizeof": (C.c_size_t, []),
    "chess_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "chess_validate_dims": (C.c_int, [C.POINTER(ChessDims)]),
    "chess_workspace_bytes": (C.c_size_t, [C.POINTER(ChessDims)]),
    "chess_reset_slots": (C.c_int, [C.POINTER(ChessState), _P, _P]),
    "chess_append_kv": (C.c_int, [C.POINTER(ChessState), _P, _P, _I64, _P, _P]),
    "chess_summary_seal": (C.c_int, [C.POINTER(ChessState), _P]),
    "chess_summary_build": (C.c_int, [C.POINTER(ChessState), _P, _P]),
    "chess_summary_from_vectors": (C.c_int, [C.POINTER(ChessState), _I32, _P, _I32, _I64, _P]),
    "chess_summary_fold": (C.c_int, [C.POINTER(ChessState), _I32, _P, _I32, _I32, _I64, _P]),
    "chess_select": (C.c_int, [C.POINTER(ChessState), C.POINTER(ChessSelectCfg), _P]),
    "chess_pool_init": (C.c_int, [C.POINTER(ChessState), _P, _I32, _P]),
    "chess_pool_reserve": (C.c_int, [C.POINTER(ChessState), _P, _P]),
    "chess_pool_release": (C.c_int, [C.POINTER(ChessState), _P, _P]),
    "chess_select_partial": (C.c_int, [C.POINTER(ChessState), C.POINTER(ChessSelectCfg), _I32, _P, _I64, _P]),
    "chess_select_combine": (C.c_int, [C.POINTER(ChessState), C.POINTER(ChessSelectCfg), _I32, _P, _I32, _I64, _P]),
    "chess_append_kv_layers": (C.c_int, [C.POINTER(ChessState), _I32, _I32, _P, _P, _I64, _P, _P]),
    "chess_select_push": (C.c_int, [C.POINTER(ChessState), C.POINTER(ChessSelectCfg), _I32,
                                    C.POINTER(ChessPeerExchange), _P]),
    "chess_select_pull": (C.c_int, [C.POINTER(ChessState), C.POINTER(ChessSelectCfg), _I32,
                                    C.POINTER(ChessPeerExchange), _P]),
    "chess_sparse_decode_gather": (C.c_int, [C.POINTER(ChessState), _I32, _P, _I64, _P, _I64, _P, _F,
                                             _U32, C.POINTER(ChessPeerOutputs), _P]),
    "chess_gather_finish": (C.c_int, [C.POINTER(ChessState), C.POINTER(ChessPeerOutputs), _P, _P]),
    "chess_p2p_alloc": (C.c_int, [_I64, C.POINTER(C.c_void_p)]),
    "chess_p2p_free": (C.c_int, [_P]),
    "chess_p2p_export": (C.c_int, [_P, C.c_char_p]),
    "chess_p2p_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "chess_p2p_close": (C.c_int, [_P]),
    "chess_build_working_set": (C.c_int, [C.POINTER(ChessState), _P]),
    "chess_flush_working_sets": (C.c_int, [C.POINTER(ChessState), _P]),
    "chess_sparse_decode": (C.c_int, [C.POINTER(ChessState), _I32, _P, _I64, _P, _I64, _P, _F, _P]),
    "chess_sparse_decode_ex": (C.c_int, [C.POINTER(ChessState), _I32, _P, _I64, _P, _I64, _P, _F, _U32, _P]),
    "chess_entropy_trigger": (C.c_int, [C.POINTER(ChessState), _P, _I64, _I64, C.POINTER(ChessTriggerCfg), _P, _P]),
    "chess_record_entropy": (C.c_int, [C.POINTER(ChessState), _P, _P, C.POINTER(ChessTriggerCfg), _P]),
    "chess_score_rows": (C.c_int, [_P, _I32, _I64, _I64, _I64, _P, _P, _P]),
    "chess_mean_rows": (C.c_int, [_P, _I32, _I64, _I64, _I64, _P, _P]),
    "chess_prune": (C.c_int, [_P, _I32, _P, _I32, _P, _I32, _P, _P, _D, _D, _D, _P, _P, _P, _P]),
    "chess_prune_workspace_bytes": (C.c_size_t, [_I32, _I32, _I32]),
    "chess_topk": (C.c_int, [_P, _I32, _I32, _P, _P, _P, _I32, _P, _P]),
    "chess_working_set": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P]),
    "chess_gather_pages": (C.c_int, [_P, _I32, _P, _I32, _P, _P, _P]),
    "chess_entropy_probs": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P]),
    "chess_entropy_workspace_bytes": (C.c_size_t, [_I64]),
    "chess_entropy_logits": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P]),
    "chess_page_uncertainty": (C.c_int, [_P, _I32, _P, _P]),
    "chess_calibrate_workspace_bytes": (C.c_size_t, [_I32]),
    "chess_calibrate": (C.c_int, [_P, _P, _I32, _I64, _D, _P, _P, _P]),
}

_lib = None
_lock = threading.Lock()


class NativeLibraryError(PageSelError):
    """libchess_b200.so is missing or incompatible (no CPU fallback exists)."""


def load():
    """Load (once) and return the ctypes handle; raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = Path(os.environ.get("CHESS_B200_LIB", LIB_PATH))
        if not path.exists():
            raise NativeLibraryError(
                f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.chess_abi_version() != ABI_VERSION:
            raise NativeLibraryError("ABI version mismatch")
        if lib.chess_dims_sizeof() != C.sizeof(ChessDims) or lib.chess_state_sizeof() != C.sizeof(ChessState):
            raise NativeLibraryError("ChessDims/ChessState layout mismatch between C and ctypes")
        _lib = lib
        return lib


def last_error() -> str:
    lib = load()
    buf = C.create_string_buffer(512)
    lib.chess_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status code onto the pagesel exception hierarchy."""
    if rc == OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == ERR_OUT_OF_PAGES:
        raise OutOfPagesError(msg)
    if rc == ERR_EMPTY_CONTEXT:
        raise EmptyContextError(msg)
    if rc in (ERR_SHAPE, ERR_ORDER, ERR_VALUE):
        raise ValueError(msg)
    if rc == ERR_INDEX:
        raise IndexError(msg)
    raise NativeLibraryError(f"status {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
