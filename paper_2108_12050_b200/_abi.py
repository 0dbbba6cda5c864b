"""ctypes declarations of include/mhfd.h (argument marshalling only).

Every entry point keeps its C name; ``load()`` returns the loaded library.  There
is no fallback: if ``libmhfd.so`` cannot be built or loaded, this raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import _build

MHFD_OK = 0
STATUS = {0: "MHFD_OK", 1: "MHFD_ERR_INVALID_ARGUMENT", 2: "MHFD_ERR_SHAPE", 3: "MHFD_ERR_CAPACITY",
          4: "MHFD_ERR_WORKSPACE", 5: "MHFD_ERR_CUDA", 6: "MHFD_ERR_DEVICE"}
MHFD_U8, MHFD_U16, MHFD_F32 = 1, 2, 3
MHFD_DARK, MHFD_BRIGHT = 0, 1
MHFD_RESPONSE_DOG, MHFD_RESPONSE_LOG = 0, 1
MHFD_BOUNDARY_PERIODIC, MHFD_BOUNDARY_REFLECT = 0, 1
MHFD_NMS_PAPER, MHFD_NMS_26 = 0, 1
MHFD_SCHEDULE = {None: 0, "auto": 0, "tc": 1, "band": 2, "generic": 3}

# every symbol include/mhfd.h declares (checked by tests/test_abi.py)
EXPORTS = ["mhfd_params_default", "mhfd_create", "mhfd_workspace_bytes", "mhfd_detect_batch",
           "mhfd_focus_score", "mhfd_debug_dump", "mhfd_get_params", "mhfd_last_launch_count",
           "mhfd_destroy", "mhfd_status_string", "mhfd_last_error", "mhfd_abi_version",
           "mhfd_focus_score_host", "mhfd_timing_enable", "mhfd_timing_read", "mhfd_schedule_name",
           "mhfd_schedule_flops_per_pixel", "mhfd_detect_band", "mhfd_prune_candidates",
           "mhfd_prune_band", "mhfd_interaction_radius", "mhfd_downsample"]


class mhfd_params(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("min_sigma", ctypes.c_float), ("max_sigma", ctypes.c_float), ("num_scales", ctypes.c_int32),
                ("threshold", ctypes.c_float), ("overlap", ctypes.c_float), ("sat_low", ctypes.c_float),
                ("sat_high", ctypes.c_float), ("nms", ctypes.c_int32), ("strict", ctypes.c_int32),
                ("device", ctypes.c_int32), ("max_candidates", ctypes.c_int32), ("polarity", ctypes.c_int32),
                ("response", ctypes.c_int32), ("boundary", ctypes.c_int32),
                ("schedule", ctypes.c_int32)]


class mhfd_blob(ctypes.Structure):
    _fields_ = [("x", ctypes.c_int32), ("y", ctypes.c_int32), ("scale", ctypes.c_int32),
                ("response", ctypes.c_float)]


_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # MHFD_LIB: load an explicitly built variant (performance experiments only)
        path = os.environ.get("MHFD_LIB") or _build.build()
        lib = ctypes.CDLL(path)
        P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        sig = {
            "mhfd_params_default": (None, [ctypes.POINTER(mhfd_params)]),
            "mhfd_create": (i32, [ctypes.POINTER(mhfd_params), ctypes.POINTER(P)]),
            "mhfd_workspace_bytes": (i32, [P, i32, ctypes.POINTER(sz)]),
            "mhfd_detect_batch": (i32, [P, P, i32, i32, i64, P, sz, P, i32, P, P, P]),
            "mhfd_focus_score": (i32, [P, P, i32, i32, i64, P, sz, P, P, P]),
            "mhfd_debug_dump": (i32, [P, P, i32, i32, i64, P, sz, P, P, P, P, P, P, P]),
            "mhfd_get_params": (i32, [P, ctypes.POINTER(mhfd_params)]),
            "mhfd_last_launch_count": (i32, []),
            "mhfd_destroy": (None, [P]),
            "mhfd_status_string": (ctypes.c_char_p, [i32]),
            "mhfd_last_error": (ctypes.c_char_p, []),
            "mhfd_abi_version": (i32, []),
            "mhfd_focus_score_host": (i32, [P, P, i32, i32, i64, P, sz, P, sz, P, P, P]),
            "mhfd_timing_enable": (i32, [P, i32]),
            "mhfd_timing_read": (i32, [P, P, ctypes.POINTER(i32)]),
            "mhfd_schedule_name": (ctypes.c_char_p, [P, i32]),
            "mhfd_schedule_flops_per_pixel": (ctypes.c_double, [P, i32]),
            "mhfd_detect_band": (i32, [P, P, i32, i64, i32, i32, P, sz, P, i32, P, P]),
            "mhfd_prune_candidates": (i32, [P, P, i32, P, sz, P, i32, P, P, P, P]),
            "mhfd_prune_band": (i32, [P, P, i32, i32, i32, i32, i32, P, sz, P, P, P, P]),
            "mhfd_interaction_radius": (i32, [P]),
            "mhfd_downsample": (i32, [P, i32, i32, i32, i64, i32, P, i64, i32, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class MHFDError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status


def check(status: int) -> None:
    if status != MHFD_OK:
        raise MHFDError(status, load().mhfd_last_error().decode())
