"""ctypes binding of include/pirk_c.h (libpirk_b200.so).

The shared library is the only compute path: if it is missing, importing the
package still works (so CPU-only tooling can inspect it) but every entry point
raises ``RuntimeError`` -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libpirk_b200.so")
# development A/B builds only (tools/ab_build.py): load another build of the same ABI
LIB_PATH = os.environ.get("PIRK_LIB", LIB_PATH)
HEADER = os.path.join(HERE, "..", "include", "pirk_c.h")

# pirk_status
OK, EINVAL, EINTEGRATION, EORDER, ENEGRADIUS, ENOMEM, ECUDA, EUNSUPPORTED = range(8)
MODE_EXACT, MODE_FAST = 0, 1
METHOD_MM, METHOD_GB, METHOD_MC = 0, 1, 2


class PirkModel(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("decomp", C.c_int32),
        ("dim", C.c_uint64),
        ("input_dim", C.c_uint64),
        ("grid", C.c_uint64),
        ("params", C.c_double * 8),
        ("program", C.c_void_p),
    ]


_DP = C.POINTER(C.c_double)
_U64P = C.POINTER(C.c_uint64)


class PirkProblem(C.Structure):
    _fields_ = [
        ("init_lower", _DP),
        ("init_upper", _DP),
        ("input_lower", _DP),
        ("input_upper", _DP),
        ("t0", C.c_double),
        ("t1", C.c_double),
        ("h", C.c_double),
        ("tube_stride", C.c_uint64),
    ]


class PirkMcSpec(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double),
        ("delta", C.c_double),
        ("seed", C.c_uint64),
        ("samples_override", C.c_uint64),
    ]


class PirkTube(C.Structure):
    _fields_ = [
        ("times", _DP),
        ("lower", _DP),
        ("upper", _DP),
        ("max_slots", C.c_uint64),
        ("n_slots", C.c_uint64),
    ]


class PirkReport(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("m", C.c_uint64),
        ("steps", C.c_uint64),
        ("peak_state_bytes", C.c_uint64),
        ("device_state_bytes", C.c_uint64),
        ("workers", C.c_int32),
        ("exact", C.c_int32),
        ("setup_s", C.c_double),
        ("integration_s", C.c_double),
        ("reduction_s", C.c_double),
        ("kernel_launches", C.c_uint64),
    ]


class PirkWindow(C.Structure):
    _fields_ = [
        ("in0", C.c_void_p),
        ("in1", C.c_void_p),
        ("out0", C.c_void_p),
        ("out1", C.c_void_p),
        ("win_begin", C.c_uint64),
        ("win_len", C.c_uint64),
        ("out_begin", C.c_uint64),
        ("out_end", C.c_uint64),
    ]


class PirkMirror(C.Structure):
    """pirk_mirror (include/pirk_c.h): units < lo_end also to lo0/lo1, units
    >= hi_begin also to hi0/hi1 (indexed from out_begin)."""
    _fields_ = [
        ("lo0", C.c_void_p),
        ("lo1", C.c_void_p),
        ("lo_end", C.c_uint64),
        ("hi0", C.c_void_p),
        ("hi1", C.c_void_p),
        ("hi_begin", C.c_uint64),
    ]


# Every symbol include/pirk_c.h declares, with its ctypes signature.
_MP = C.POINTER(PirkModel)
_PP = C.POINTER(PirkProblem)
_TP = C.POINTER(PirkTube)
_RP = C.POINTER(PirkReport)
SIGNATURES = {
    "pirk_abi_version": (C.c_int32, []),
    "pirk_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "pirk_create_multi": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]),
    "pirk_lane_count": (C.c_int32, [C.c_void_p]),
    "pirk_device_count": (C.c_int32, []),
    "pirk_lane_device": (C.c_int32, [C.c_void_p, C.c_int32]),
    "pirk_release_cache": (C.c_int, [C.c_void_p]),
    "pirk_set_record_callback": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "pirk_destroy": (None, [C.c_void_p]),
    "pirk_last_error": (C.c_char_p, [C.c_void_p]),
    "pirk_set_mode": (C.c_int, [C.c_void_p, C.c_int32]),
    "pirk_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pirk_get_stream": (C.c_void_p, [C.c_void_p]),
    "pirk_launch_count": (C.c_uint64, [C.c_void_p]),
    "pirk_plan_steps": (C.c_int, [C.c_double, C.c_double, C.c_double, _U64P, C.POINTER(C.c_int32)]),
    "pirk_record_schedule": (C.c_uint64, [C.c_double, C.c_double, C.c_double, C.c_uint64, _U64P, _DP]),
    "pirk_sample_count": (C.c_int, [C.c_uint64, C.c_double, C.c_double, _U64P]),
    "pirk_supports": (C.c_int32, [_MP, C.c_int32]),
    "pirk_mixed_monotonicity": (C.c_int, [C.c_void_p, _MP, _PP, _TP, _RP]),
    "pirk_growth_bound": (C.c_int, [C.c_void_p, _MP, _PP, _TP, _RP]),
    "pirk_monte_carlo": (C.c_int, [C.c_void_p, _MP, _PP, C.POINTER(PirkMcSpec), _TP, _RP]),
    "pirk_monte_carlo_range": (C.c_int, [C.c_void_p, _MP, _PP, C.c_uint64, C.c_uint64,
                                         C.c_uint64, _TP, _RP]),
    "pirk_coverage_estimate": (C.c_int, [C.c_void_p, _MP, _PP, _DP, _DP, C.c_uint64,
                                         C.c_uint64, _DP]),
    "pirk_engine_create": (C.c_int, [C.c_void_p, _MP, C.c_int32, _PP, C.POINTER(C.c_void_p)]),
    "pirk_engine_advance": (C.c_int, [C.c_void_p, C.c_uint64]),
    "pirk_engine_status": (C.c_int, [C.c_void_p, _U64P]),
    "pirk_engine_read": (C.c_int, [C.c_void_p, _DP, _DP]),
    "pirk_engine_destroy": (None, [C.c_void_p]),
    "pirk_program_create": (C.c_int, [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                      C.POINTER(C.c_void_p)]),
    "pirk_program_compile": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_size_t, _U64P]),
    "pirk_program_cubin": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64]),
    "pirk_program_set_stencil": (C.c_int, [C.c_void_p, C.c_uint64]),
    "pirk_program_destroy": (None, [C.c_void_p]),
    "pirk_step_window": (C.c_int, [C.c_void_p, _MP, C.c_int32, C.POINTER(PirkWindow), _DP, _DP,
                                   C.c_double, C.c_double, C.c_uint64, C.c_void_p]),
    "pirk_step_window_mirror": (C.c_int, [C.c_void_p, _MP, C.c_int32, C.POINTER(PirkWindow),
                                          C.POINTER(PirkMirror), _DP, _DP, C.c_double, C.c_double,
                                          C.c_uint64, C.c_void_p]),
    "pirk_ipc_export": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_uint64)]),
    "pirk_ipc_open": (C.c_int, [C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]),
    "pirk_ipc_close": (C.c_int, [C.c_void_p]),
    "pirk_wait_flag": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
    "pirk_signal_flag": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
}

# pirk_record_fn (include/pirk_c.h)
RECORD_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint64, C.c_double, C.POINTER(C.c_double),
                        C.POINTER(C.c_double), C.c_uint64)

_lib = None
_lock = threading.Lock()


def lib():
    """Load libpirk_b200.so (raises RuntimeError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"PIRK device library not built: {LIB_PATH} is missing "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                    "there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            if L.pirk_abi_version() != 1:
                raise RuntimeError("libpirk_b200.so ABI version mismatch")
            _lib = L
    return _lib


def dptr(a):
    """numpy float64 array -> double* (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_DP)
