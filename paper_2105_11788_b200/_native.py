"""ctypes binding of libbisim.so (include/bisim.h).

The shared library is built in-tree (``make -C paper_2105_11788_b200/csrc``
or ``__graft_entry__.build()``).  There is deliberately no fallback: if the
library is missing or no CUDA device is visible, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BISIM_LIB (developer override: an experimental build of the same library)
# is honoured only together with BISIM_DEV=1
LIB_PATH = ((os.environ.get("BISIM_DEV") and os.environ.get("BISIM_LIB"))
            or os.path.join(_HERE, "libbisim.so"))

BISIM_OK, BISIM_BAD_INPUT, BISIM_GUARD, BISIM_CUDA, BISIM_ABORTED = 0, 1, 2, 3, 4
SHARD_VERIFY = 1
DEFAULT_GUARD = -(2 ** 63)
MODE_AUTO, MODE_PERSISTENT, MODE_STEPPED, MODE_DENSE = 0, 1, 2, 3
# schedule variants (bisim.h BISIM_FLAG_*): none changes a result
FLAG_NO_SKIP, FLAG_NO_SOLO, FLAG_CTA_MAJOR, FLAG_LITERAL_LABEL_ROUNDS = 1, 2, 4, 8
FLAG_WIDE_LAYOUT, FLAG_TWO_PASS, FLAG_BATCH_WALK = 16, 32, 64

i32p = ctypes.POINTER(ctypes.c_int32)
OBSERVER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int64, i32p, ctypes.c_int32, ctypes.c_void_p)


class Stats(ctypes.Structure):
    _fields_ = [("supersteps", ctypes.c_int64),
                ("label_rounds", ctypes.c_int64),
                ("guard_count", ctypes.c_int64),
                ("initial_blocks", ctypes.c_int32),
                ("final_blocks", ctypes.c_int32),
                ("mark_length", ctypes.c_int64),
                ("t_h2d_ms", ctypes.c_double),
                ("t_pre_ms", ctypes.c_double),
                ("t_label_ms", ctypes.c_double),
                ("t_alg_ms", ctypes.c_double),
                ("t_d2h_ms", ctypes.c_double),
                ("bytes_alg", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int32),
                ("mode", ctypes.c_int32),
                ("rounds_retired", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32),
                ("mode", ctypes.c_int32),
                ("observer", OBSERVER),
                ("observer_user", ctypes.c_void_p),
                ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_int32)]


class AutInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32),
                ("initial_state", ctypes.c_int32),
                ("m", ctypes.c_int64),
                ("num_actions", ctypes.c_int32),
                ("pad", ctypes.c_int32),
                ("error_line", ctypes.c_int64)]


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(message)


_lib = None
_lock = threading.Lock()

EXPORTS = ("bisim_bcrp", "bisim_rcpp", "bisim_bcrp_ex", "bisim_rcpp_ex", "bisim_bcrp_device",
           "bisim_rcpp_device", "bisim_preprocess", "bisim_label_partition", "bisim_last_error",
           "bisim_device_count", "bisim_stream", "bisim_version", "bisim_quotient",
           "bisim_is_stable", "bisim_canonical", "bisim_aut_parse", "bisim_aut_read_file",
           "bisim_aut_columns", "bisim_aut_label", "bisim_aut_free", "bisim_bcrp_sharded",
           "bisim_rcpp_sharded", "bisim_is_stable_under", "bisim_preprocess_sorted",
           "bisim_label_rounds_common")


def lib():
    """Load libbisim.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: build it with "
                                  "`make -C paper_2105_11788_b200/csrc` (no CPU fallback exists)")
            L = ctypes.CDLL(LIB_PATH)
            P = ctypes.POINTER
            i64 = ctypes.c_int64
            i32 = ctypes.c_int32
            L.bisim_bcrp.argtypes = [i32, i64, i32, i32p, i32p, i32p, i64, i32p, i32p, i64,
                                     P(Stats), ctypes.c_int]
            L.bisim_rcpp.argtypes = [i32, i64, i32p, i32p, i32p, i64, i32p, i32p, i64,
                                     P(Stats), ctypes.c_int]
            L.bisim_bcrp_ex.argtypes = [i32, i64, i32, i32p, i32p, i32p, i64, i32p, i32p, i64,
                                        P(Stats), P(Options)]
            L.bisim_rcpp_ex.argtypes = [i32, i64, i32p, i32p, i32p, i64, i32p, i32p, i64,
                                        P(Stats), P(Options)]
            L.bisim_bcrp_device.argtypes = [i32, i64, i32, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p, i64, ctypes.c_void_p, i32p, i64,
                                            P(Stats), P(Options)]
            L.bisim_rcpp_device.argtypes = [i32, i64, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p, i64, ctypes.c_void_p, i32p, i64,
                                            P(Stats), P(Options)]
            L.bisim_preprocess.argtypes = [i32, i64, i32, i32p, i32p, i32p, i32p, i32p, P(i64),
                                           ctypes.c_int]
            L.bisim_preprocess_sorted.argtypes = [i32, i64, i32, i32p, i32p, i32p, i32p, i32p, i32p,
                                                  i32p, i32p, i32p, i32p, i32p, P(i64),
                                                  ctypes.c_int]
            L.bisim_label_rounds_common.argtypes = [i32, i64, i32, i32p, i32p, i32p, i32p, i32p, i32p,
                                                    ctypes.c_int]
            L.bisim_label_partition.argtypes = [i32, i64, i32, i32p, i32p, i32p, ctypes.c_int]
            L.bisim_quotient.argtypes = [i32, i64, i32, i32p, i32p, i32p, i32p, i32, P(i32),
                                         P(i64), i32p, i32p, i32p, P(i32), ctypes.c_int]
            L.bisim_is_stable.argtypes = [i32, i64, i32, i32p, i32p, i32p, i32p, P(i32),
                                          ctypes.c_int]
            L.bisim_canonical.argtypes = [i32, P(i64), i32p, ctypes.c_int]
            L.bisim_is_stable_under.argtypes = [i32, i64, i32, i32p, i32p, i32p, i32p, i32p, i64,
                                                P(i32), ctypes.c_int]
            L.bisim_bcrp_sharded.argtypes = [i32, i64, i32, i32p, i32p, i32p, i64, i32p, i32p, i64,
                                             P(Stats), i32p, i32, i32]
            L.bisim_rcpp_sharded.argtypes = [i32, i64, i32p, i32p, i32p, i64, i32p, i32p, i64,
                                             P(Stats), i32p, i32, i32]
            vp = ctypes.c_void_p
            L.bisim_aut_parse.argtypes = [ctypes.c_char_p, i64, i32, P(vp), P(AutInfo)]
            L.bisim_aut_read_file.argtypes = [ctypes.c_char_p, i32, P(vp), P(AutInfo)]
            L.bisim_aut_columns.argtypes = [vp, i32p, i32p, i32p]
            L.bisim_aut_label.argtypes = [vp, i32, P(i64)]
            L.bisim_aut_free.argtypes = [vp]
            for name in ("bisim_bcrp", "bisim_rcpp", "bisim_bcrp_ex", "bisim_rcpp_ex",
                         "bisim_bcrp_device", "bisim_rcpp_device", "bisim_preprocess",
                         "bisim_label_partition", "bisim_device_count", "bisim_quotient",
                         "bisim_is_stable", "bisim_canonical", "bisim_aut_parse",
                         "bisim_aut_read_file", "bisim_aut_columns", "bisim_bcrp_sharded",
                         "bisim_rcpp_sharded", "bisim_is_stable_under", "bisim_preprocess_sorted",
           "bisim_label_rounds_common"):
                getattr(L, name).restype = ctypes.c_int
            # pointer / void results: never through the int loop above (a
            # c_int restype truncates a heap pointer to 32 bits)
            L.bisim_aut_label.restype = vp
            L.bisim_aut_free.restype = None
            L.bisim_last_error.restype = ctypes.c_char_p
            L.bisim_last_error.argtypes = []
            L.bisim_stream.restype = ctypes.c_void_p
            L.bisim_stream.argtypes = [ctypes.c_int]
            L.bisim_version.restype = ctypes.c_char_p
            L.bisim_version.argtypes = []
            _lib = L
    return _lib


def last_error() -> str:
    return lib().bisim_last_error().decode("utf-8", "replace")


def ptr(a: np.ndarray):
    return a.ctypes.data_as(i32p)


def as_i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def check(rc: int):
    if rc != BISIM_OK:
        raise NativeError(rc, last_error())
