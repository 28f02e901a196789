"""ctypes binding of libmarket_eq_b200.so (include/market_eq_b200.h).

There is no CPU fallback: importing the solver on a machine without the
built library or without a CUDA device raises NativeUnavailable the moment a
device operation is requested.
"""

import ctypes
import os
import threading

from .errors import MarketError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MQ_LIB") or os.path.join(_PKG, "libmarket_eq_b200.so")
TILE_ENTRIES = 2560   # MQ_TILE_ENTRIES
LONG_ROW = int(os.environ.get("MQ_LONG_ROW", "1024"))  # MQ_LONG_ROW (tuning override)
REG_ROW = 128         # MQ_REG_ROW
TILE_ROWS = 256       # MQ_TILE_ROWS
PAD = 16              # padding elements after nnz arrays read by TMA bulk copies
ABI_VERSION = 12
WS_SLOTS = 10          # MQ_WS_SLOTS
WS_MAX_ROW = 256       # MQ_WS_MAX_ROW
LONG_CAP = 1536        # MQ_LONG_CAP (long-row working-set pool per row)
MED_CAP = 128          # MQ_MED_CAP (medium-row working-set pool per row)

_lock = threading.Lock()
_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
F64 = ctypes.c_double
CINT = ctypes.c_int


class NativeUnavailable(MarketError, RuntimeError):
    """The sm_100a library or a CUDA device is missing (no CPU fallback)."""


class NativeError(MarketError, RuntimeError):
    """A CUDA call inside the native library failed."""


class MqMarket(ctypes.Structure):
    _fields_ = [("n", I64), ("m", I64), ("nnz", I64),
                ("row_ptr", P), ("col", P), ("u", P), ("u_orig", P), ("w", P),
                ("tiles", P), ("ntiles", I64), ("long_rows", P), ("nlong", I64),
                ("med_rows", P), ("nmed", I64), ("nmed_long", I64),
                ("bperm", P), ("bptr", P), ("nblk", I64), ("tiles_per_block", I64),
                ("prim_grid", ctypes.c_int32), ("row_begin", I64),
                ("cs_scale", ctypes.c_double), ("cs_xmax", ctypes.c_double)]


class MqState(ctypes.Structure):
    _fields_ = [("x", P), ("xbar", P), ("p", P), ("pbar", P), ("cs", P), ("cs_prev", P),
                ("csbar", P), ("blk_done", P), ("steps", P), ("navg", P),
                ("pass_out", P), ("faults", P), ("bucket", P), ("srow", P),
                ("xflag", P), ("xsum", P), ("ws_hdr", P), ("ws_kmax", P), ("ws_u", P),
                ("ws_x", P), ("ws_col", P), ("ws_pos", P), ("ws_list", P), ("drift", P),
                ("pl_hdr", P), ("pl_u", P), ("pl_x", P), ("pl_col", P), ("pl_pos", P),
                ("pm_hdr", P), ("pm_u", P), ("pm_x", P), ("pm_col", P), ("pm_pos", P),
                ("ws_rebuild", ctypes.c_int32), ("xbar_lazy", ctypes.c_int32),
                ("ws_lvl", P), ("pl_list", P)]


PM = ctypes.POINTER(MqMarket)
PS = ctypes.POINTER(MqState)


class MqLState(ctypes.Structure):
    _fields_ = [(k, P) for k in ("x", "xbar", "t", "t_prev", "tbar", "y", "ybar", "ru",
                                 "ru_prev", "p", "pbar", "cs", "cs_prev", "csbar", "fix",
                                 "steps", "navg", "faults")]


PL = ctypes.POINTER(MqLState)

# name -> (restype, argtypes)
_SIGS = {
    "mq_pdhcg_chunk": (CINT, [I64, I64, P, P, P, P, P, P, P, P, P, P, P, I64, F64, F64, CINT,
                              F64, CINT, P, P, P, P]),
    "mq_dual_step": (CINT, [PM, PS, CINT, P]),
    "mq_primal_step": (CINT, [PM, PS, CINT, P, P]),
    "mq_colsum_step": (CINT, [PM, PS, CINT, CINT, P]),
    "mq_colsum_finalize": (CINT, [PM, PS, CINT, P]),
    "mq_chunk_end": (CINT, [PS, CINT, P]),
    "mq_fast_chunk": (CINT, [PM, PS, CINT, P]),
    "mq_colsum": (CINT, [PM, P, P, P]),
    "mq_resid_rows": (CINT, [PM, P, P, CINT, P, P, P, P, P, P, P]),
    "mq_resid_cols": (CINT, [I64, P, P, P, P, P, P]),
    "mq_resid_rows_pair": (CINT, [PM, PS, P, P, P, P, P, P, P, P]),
    "mq_restart_moves": (CINT, [PM, P, P, P, P, P, P, P, P, P]),
    "mq_spmv": (CINT, [I64, P, P, P, P, P, P]),
    "mq_normalize_rows": (CINT, [I64, P, P, P, P, P]),
    "mq_gen_degrees": (CINT, [I64, I64, I64, CINT, F64, F64, F64, ctypes.c_ulonglong, P, P]),
    "mq_gen_fill": (CINT, [I64, I64, I64, CINT, F64, F64, F64, ctypes.c_ulonglong, P, P, P, P,
                           P]),
    "mq_scratch_doubles": (I64, []),
    "mq_tile_entries": (CINT, []),
    "mq_reg_row": (CINT, []),
    "mq_colsum_mode": (CINT, []),
    "mq_last_error": (ctypes.c_char_p, []),
    "mq_abi_version": (CINT, []),
    "mq_fixed_colsum": (CINT, []),
    "mq_x_sparse": (CINT, []),
    "mq_ws_slots": (CINT, []),
    "mq_long_cap": (CINT, []),
    "mq_med_cap": (CINT, []),
    "mq_market_bytes": (CINT, []),
    "mq_state_bytes": (CINT, []),
    "mq_avg_materialize": (CINT, [PM, PS, P]),
    "mq_ws_flush": (CINT, [PM, PS, P]),
    "mq_avg_xbar": (CINT, [PM, PS, P]),
    "mq_pdhg_step": (CINT, [PM, PL, CINT, P]),
    "mq_pdhg_colsum_only": (CINT, [PM, PL, CINT, P]),
    "mq_pdhg_finish_colsum": (CINT, [PM, PL, CINT, P]),
    "mq_pdhg_chunk_end": (CINT, [PL, CINT, P]),
    "mq_row_dot": (CINT, [PM, P, CINT, P, P]),
    "mq_pdhg_resid_rows": (CINT, [PM, P, P, P, P, P, CINT, P, P, P, P]),
    "mq_pdhg_moves": (CINT, [PM, P, P, P, P, P, P, P, P, P]),
    "mq_pdhg_opnorm_step": (CINT, [PM, P, P, P, P, P, P, P, P]),
    "mq_scaled_kkt_rows": (CINT, [PM, P, P, P, P, F64, P, P, P]),
    "mq_smoothed_gap_rows": (CINT, [PM, P, P, F64, P, P, P, P, P]),
}

EXPORTED = tuple(_SIGS)


def load_library(path=LIB_PATH):
    """Load the shared library (no device needed) and bind every symbol."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -m paper_2506_06258_b200._build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.mq_abi_version() != ABI_VERSION:
            raise NativeUnavailable("libmarket_eq_b200.so ABI version mismatch")
        _lib = lib
        return lib


def lib():
    """The library, after checking that a CUDA device is present."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 solver has no CPU fallback")
    return load_library()


def check(rc, what):
    if rc < 0:
        msg = load_library().mq_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")
    return rc


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())
