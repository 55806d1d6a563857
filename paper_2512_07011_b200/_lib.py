"""ctypes binding of the C ABI in ``include/bsfa_b200.h``.

The shared library ``_lib/libbsfa_b200.so`` is built in-tree (see
``__graft_entry__.build`` / ``Makefile``).  There is no fallback: if the
library is missing every entry point raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import BsfaError

LIB_PATH = os.environ.get("BSFA_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libbsfa_b200.so")

ABI_VERSION = 6
MAX_O_PEERS = 7

BSFA_OK = 0
BSFA_ERR_INVALID = -1
BSFA_ERR_CUDA = -2
BSFA_ERR_UNSUPPORTED = -3

GATE_THRESHOLD = 0
GATE_DENSE = 1
GATE_FRONTIER = 2
GATE_WINDOW = 3
GATE_RUNMAX = 4

CNT_REACHABLE = 0
CNT_KEPT = 1
CNT_VLOADS = 2

# Every symbol include/bsfa_b200.h declares (checked by the CPU test-suite).
EXPORTED_SYMBOLS = (
    "bsfa_abi_version",
    "bsfa_last_error",
    "bsfa_device_supported",
    "bsfa_fwd",
    "bsfa_debug_trace",
    "bsfa_calib_blockmax",
    "bsfa_calib_finalize",
    "bsfa_calib_select",
)


class NativeLibraryError(BsfaError, RuntimeError):
    """The CUDA library is missing, failed to load, or a call failed."""


class FwdArgs(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_void_p),
        ("k", ctypes.c_void_p),
        ("v", ctypes.c_void_p),
        ("q_stride_b", ctypes.c_int64), ("q_stride_h", ctypes.c_int64), ("q_stride_n", ctypes.c_int64),
        ("k_stride_b", ctypes.c_int64), ("k_stride_h", ctypes.c_int64), ("k_stride_n", ctypes.c_int64),
        ("v_stride_b", ctypes.c_int64), ("v_stride_h", ctypes.c_int64), ("v_stride_n", ctypes.c_int64),
        ("o", ctypes.c_void_p),
        ("o_stride_b", ctypes.c_int64), ("o_stride_h", ctypes.c_int64), ("o_stride_n", ctypes.c_int64),
        ("lse", ctypes.c_void_p),
        ("decisions", ctypes.c_void_p),
        ("counters", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("thresholds", ctypes.c_void_p),
        ("thr_positions", ctypes.c_int),
        ("gate_mode", ctypes.c_int),
        ("batch", ctypes.c_int), ("heads_q", ctypes.c_int), ("heads_kv", ctypes.c_int),
        ("seq_len", ctypes.c_int), ("valid_len", ctypes.c_int), ("head_dim", ctypes.c_int),
        ("b_m", ctypes.c_int), ("b_n", ctypes.c_int),
        ("causal", ctypes.c_int),
        ("scale", ctypes.c_float),
        ("inject_fault", ctypes.c_int),
        ("gate_window", ctypes.c_int),
        ("gate_lambda", ctypes.c_float),
        ("num_o_peers", ctypes.c_int),
        ("o_peers", ctypes.c_void_p * 7),
    ]


class CalibArgs(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_void_p),
        ("k", ctypes.c_void_p),
        ("q_stride_h", ctypes.c_int64), ("q_stride_n", ctypes.c_int64),
        ("k_stride_h", ctypes.c_int64), ("k_stride_n", ctypes.c_int64),
        ("heads_q", ctypes.c_int), ("heads_kv", ctypes.c_int), ("seq_len", ctypes.c_int),
        ("head_dim", ctypes.c_int),
        ("b_m", ctypes.c_int), ("b_n", ctypes.c_int),
        ("scale", ctypes.c_float),
        ("layer", ctypes.c_int), ("num_layers", ctypes.c_int), ("num_positions", ctypes.c_int),
        ("num_levels", ctypes.c_int),
        ("k_levels", ctypes.c_int * 16),
        ("finite_sum", ctypes.c_void_p),
        ("finite_cnt", ctypes.c_void_p),
        ("neg_cnt", ctypes.c_void_p),
        ("pos_cnt", ctypes.c_void_p),
        ("tie_counts", ctypes.c_void_p),
        ("block_maxima", ctypes.c_void_p),
        ("valid_len", ctypes.c_int),
    ]


_lock = threading.Lock()
_lib = None


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and type the native library; raise loudly if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeLibraryError(
                f"BSFA CUDA library not found at {p}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` or `make`")
        try:
            lib = ctypes.CDLL(p)
        except OSError as e:
            raise NativeLibraryError(f"failed to load {p}: {e}") from e
        lib.bsfa_abi_version.restype = ctypes.c_int
        lib.bsfa_abi_version.argtypes = []
        lib.bsfa_last_error.restype = ctypes.c_char_p
        lib.bsfa_last_error.argtypes = []
        lib.bsfa_device_supported.restype = ctypes.c_int
        lib.bsfa_device_supported.argtypes = []
        lib.bsfa_fwd.restype = ctypes.c_int
        lib.bsfa_fwd.argtypes = [ctypes.POINTER(FwdArgs), ctypes.c_void_p]
        lib.bsfa_debug_trace.restype = ctypes.c_int
        lib.bsfa_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.bsfa_calib_blockmax.restype = ctypes.c_int
        lib.bsfa_calib_blockmax.argtypes = [ctypes.POINTER(CalibArgs), ctypes.c_void_p]
        lib.bsfa_calib_finalize.restype = ctypes.c_int
        lib.bsfa_calib_finalize.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_void_p]
        lib.bsfa_calib_select.restype = ctypes.c_int
        lib.bsfa_calib_select.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]
        if lib.bsfa_abi_version() != ABI_VERSION:
            raise NativeLibraryError(
                f"ABI mismatch: library {lib.bsfa_abi_version()} vs binding {ABI_VERSION}")
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != BSFA_OK:
        msg = load_library().bsfa_last_error().decode(errors="replace")
        raise NativeLibraryError(f"{what} failed (code {rc}): {msg}")
