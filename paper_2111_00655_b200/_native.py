"""ctypes binding of libcollage_b200.so (the C ABI declared in
include/collage_b200.h).

The library is the product: the placement search has no Python or CPU
implementation to fall back to.  Importing this module does not need a GPU
(graph analysis is host code), but every search entry point raises
`DeviceUnavailableError` when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int8, c_int32, c_int64, \
    c_uint8, c_uint64, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libcollage_b200.so")

CB_OK = 0
CB_ERR_CUDA = 1
CB_ERR_ARG = 2
CB_ERR_PROFILE = 3
CB_ERR_INEXACT = 4
CB_ERR_CYCLE = 5
CB_ERR_LIMIT = 6
CB_ERR_STATE = 7


class NativeError(RuntimeError):
    """A call into libcollage_b200 failed."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[cb error {code}] {message}")
        self.code = code
        self.message = message


class DeviceUnavailableError(NativeError):
    """The CUDA library or device needed by the search is missing."""


class DPResultStruct(ctypes.Structure):
    _fields_ = [
        ("cost_ms", c_double),
        ("feasible", c_int32),
        ("n_kernels", c_int32),
        ("n_levels", c_int32),
        ("n_launches", c_int32),
        ("candidates", c_int64),
        ("ties", c_int64),
        ("walk_steps", c_int64),
        ("window_safe", c_int32),
        ("first_zero_candidate", c_int32),
        ("device_ms", c_double),
    ]


class ESPlanInfo(ctypes.Structure):
    _fields_ = [
        ("genome_bits", c_int32),
        ("words", c_int32),
        ("units", c_int32),
        ("fixed_units", c_int32),
        ("edges", c_int32),
        ("infeasible_bits", c_int32),
        ("smem_path", c_int32),
        ("frontier_slots", c_int32),
        ("seed_cost", c_double),
        ("window_shift", c_int32),
        ("packed_labels", c_int32),
        ("fsm_transitions", c_int32),
        ("fsm_entry_bytes", c_int32),
    ]


_P_I32 = POINTER(c_int32)
_P_I8 = POINTER(c_int8)
_P_U8 = POINTER(c_uint8)
_P_I64 = POINTER(c_int64)
_P_F64 = POINTER(c_double)
_P_U64 = POINTER(c_uint64)

# name -> (restype, argtypes)
_SIGNATURES = {
    "cb_last_error": (c_char_p, []),
    "cb_abi_version": (c_int, []),
    "cb_device_available": (c_int, []),
    "cb_fx_sum": (c_int, [_P_F64, c_int64, _P_F64, _P_I32]),
    "cb_graph_create": (c_int, [c_int32, _P_I32, _P_I32, _P_I32, _P_U8, _P_F64, _P_I32,
                                _P_I32, _P_I8, _P_I64, _P_F64, POINTER(c_void_p)]),
    "cb_graph_destroy": (None, [c_void_p]),
    "cb_graph_analysis": (c_int, [c_void_p, _P_I32, _P_I32, _P_I32, _P_I32, _P_I32, _P_I32]),
    "cb_patterns_create": (c_int, [c_int32, c_int32, _P_I32, _P_I32, _P_I32, _P_I32, _P_I32,
                                   _P_I32, _P_I32, _P_I32, _P_I8, _P_I32, _P_I8, _P_I64,
                                   _P_F64, _P_I64, _P_I64, _P_I32, _P_I32, _P_I32,
                                   POINTER(c_void_p)]),
    "cb_patterns_destroy": (None, [c_void_p]),
    "cb_match_all": (c_int, [c_void_p, c_void_p, POINTER(c_void_p)]),
    "cb_match_pairs": (c_int, [c_void_p, c_void_p, c_int32, _P_I32, _P_I32, POINTER(c_void_p)]),
    "cb_matches_counts": (c_int, [c_void_p, _P_I64, _P_I64, _P_I64, _P_I64]),
    "cb_matches_download": (c_int, [c_void_p, _P_I32, _P_I32, _P_I32, _P_I32, _P_I32, _P_I32,
                                    _P_I32]),
    "cb_matches_destroy": (None, [c_void_p]),
    "cb_matches_price": (c_int, [c_void_p, c_void_p, c_int32, c_int32, _P_F64, _P_F64, _P_U8,
                                 _P_U8, c_int32, _P_F64, _P_F64, _P_I8]),
    "cb_matches_set_costs": (c_int, [c_void_p, _P_F64]),
    "cb_dp_solve": (c_int, [c_void_p, c_void_p, c_double, _P_I32, POINTER(DPResultStruct)]),
    "cb_dp_solve_stream": (c_int, [c_void_p, c_void_p, c_double, _P_I32, POINTER(DPResultStruct),
                                   c_void_p]),
    "cb_placement_cost_graphlevel": (c_int, [c_void_p, c_int32, _P_I32, _P_I32, _P_I32, _P_F64,
                                             c_int32, _P_U8, _P_F64, _P_F64, c_double, _P_F64]),
    "cb_es_plan_create": (c_int, [c_void_p, c_void_p, c_int32, _P_I32, c_int32, _P_U8, _P_F64,
                                  _P_F64, c_int32, c_double, POINTER(c_void_p)]),
    "cb_es_plan_query": (c_int, [c_void_p, POINTER(ESPlanInfo)]),
    "cb_es_plan_slots": (c_int, [c_void_p, _P_I32, _P_I8, _P_I32, _P_I32]),
    "cb_es_plan_set_path": (c_int, [c_void_p, c_int32]),
    "cb_es_plan_set_pool": (c_int, [c_void_p, c_int32]),
    "cb_es_plan_kernel": (c_char_p, [c_void_p]),
    "cb_es_plan_units": (c_int, [c_void_p, _P_I32, _P_I32, _P_I32, _P_I32]),
    "cb_es_plan_destroy": (None, [c_void_p]),
    "cb_fitness_device": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "cb_fitness_host": (c_int, [c_void_p, _P_U64, c_int64, _P_F64]),
    "cb_es_breed": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                            c_int64, c_uint64, c_uint64, c_uint64, c_int32, c_double,
                            c_void_p]),
    "cb_es_generation": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                                 c_void_p, c_int64, c_uint64, c_uint64, c_uint64, c_int32,
                                 c_double, c_void_p]),
    "cb_es_generation_fused": (c_int, [c_void_p]),
    "cb_elite_record": (c_int, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p, c_void_p,
                                 c_void_p]),
    "cb_elite_pick": (c_int, [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "cb_argmin_elite": (c_int, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p]),
    "cb_argmin": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded library; raises DeviceUnavailableError if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailableError(
                CB_ERR_CUDA,
                f"{LIB_PATH} is missing: build it with `python -c 'import "
                f"__graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().cb_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(code: int) -> None:
    if code != CB_OK:
        msg = last_error()
        if code == CB_ERR_CUDA:
            raise DeviceUnavailableError(code, msg)
        raise NativeError(code, msg)


def device_available() -> bool:
    try:
        return bool(lib().cb_device_available())
    except DeviceUnavailableError:
        return False


def require_device() -> None:
    if not lib().cb_device_available():
        raise DeviceUnavailableError(
            CB_ERR_CUDA, "no CUDA device: the B200 placement search has no CPU path")


# -- array helpers -------------------------------------------------------------

def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


def i8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int8)


def u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def ptr(a: np.ndarray, ctype):
    """Typed pointer to a contiguous numpy array (keeps no reference)."""
    return a.ctypes.data_as(POINTER(ctype))


class Handle:
    """Owning wrapper of an opaque native object."""

    def __init__(self, raw: int, destroy: str):
        self.raw = c_void_p(raw)
        self._destroy = destroy

    def close(self) -> None:
        if self.raw and self.raw.value and _lib is not None:
            getattr(_lib, self._destroy)(self.raw)
        self.raw = c_void_p(None)

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass
