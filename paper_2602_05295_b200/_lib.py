"""ctypes binding of ``libhlbm.so`` (the C-ABI in ``include/hlbm.h``).

There is no fallback: if the shared library is missing the import fails loudly,
and every compute entry point runs on the GPU through this library.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HLBM_OK, HLBM_EINVAL, HLBM_EDIVERGED, HLBM_ECUDA = 0, 1, 2, 3
BC_CODES = {"periodic": 0, "inflow": 1, "outflow": 2, "wall": 3}
PRECISIONS = {"fp32": 0, "q16": 1}

LIB_PATH = Path(__file__).resolve().parent / "libhlbm.so"


class HlbmConfig(C.Structure):
    _fields_ = [
        ("struct_size", C.c_int32),
        ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
        ("gnx", C.c_int32), ("gny", C.c_int32), ("gnz", C.c_int32),
        ("x0", C.c_int32), ("x_lo_remote", C.c_int32), ("x_hi_remote", C.c_int32),
        ("tau", C.c_double), ("force", C.c_double * 3),
        ("bc", C.c_int32 * 6), ("u_in", C.c_double * 3),
        ("precision", C.c_int32),
        ("qmin", C.c_double * 10), ("qmax", C.c_double * 10), ("bits", C.c_int32 * 10),
        ("dither", C.c_int32), ("seed", C.c_uint32), ("device", C.c_int32), ("xseg", C.c_int32),
        ("q", C.c_int32),
    ]


class HlbmStats(C.Structure):
    _fields_ = [
        ("step", C.c_int64),
        ("t_fluid_ms", C.c_double), ("t_copy_ms", C.c_double), ("t_solid_ms", C.c_double),
        ("mass", C.c_double), ("momentum", C.c_double * 3), ("max_u", C.c_double),
        ("saturation", C.c_int64 * 10), ("n_fluid", C.c_int64), ("finite", C.c_int32),
        ("force", C.c_double * 3), ("torque", C.c_double * 3),
    ]


# name -> (restype, argtypes); must list every entry point of include/hlbm.h
_P = C.c_void_p
_DP = C.POINTER(C.c_double)
SIGNATURES = {
    "hlbm_version": (C.c_char_p, []),
    "hlbm_device_count": (C.c_int, []),
    "hlbm_config_init": (None, [C.POINTER(HlbmConfig)]),
    "hlbm_create": (C.c_int, [C.POINTER(HlbmConfig), C.POINTER(_P)]),
    "hlbm_destroy": (None, [_P]),
    "hlbm_last_error": (C.c_char_p, [_P]),
    "hlbm_set_mask": (C.c_int, [_P, _P, _P, _P]),
    "hlbm_set_mesh": (C.c_int, [_P, _DP, C.c_int64, C.POINTER(C.c_int32), C.c_int64, _DP]),
    "hlbm_set_solid_motion": (C.c_int, [_P, _DP]),
    "hlbm_get_cut_links": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_uint32), _DP,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "hlbm_set_moments": (C.c_int, [_P, _DP, _DP, _DP]),
    "hlbm_get_moments": (C.c_int, [_P, _DP, _DP, _DP]),
    "hlbm_get_moments_box": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_int32, _DP, _DP, _DP]),
    "hlbm_init_modes": (C.c_int, [_P, C.c_double, _DP, C.c_int32]),
    "hlbm_step": (C.c_int, [_P, C.c_int32, C.POINTER(HlbmStats)]),
    "hlbm_step_async": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "hlbm_fluid_update": (C.c_int, [_P, C.c_int32]),
    "hlbm_solid_correction": (C.c_int, [_P, C.POINTER(HlbmStats)]),
    "hlbm_stream": (C.c_int, [_P]),
    "hlbm_read_stats": (C.c_int, [_P, C.POINTER(HlbmStats)]),
    "hlbm_step_reference": (C.c_int, [_P, C.c_int32]),
    "hlbm_step_fused": (C.c_int, [_P, C.c_int32, C.POINTER(HlbmStats)]),
    "hlbm_step_percell": (C.c_int, [_P, C.c_int32, C.POINTER(HlbmStats)]),
    "hlbm_get_boundary": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_int64)]),
    "hlbm_get_codes": (C.c_int, [_P, C.POINTER(C.c_uint32)]),
    "hlbm_set_codes": (C.c_int, [_P, C.POINTER(C.c_uint32)]),
    "hlbm_get_state": (C.c_int, [_P, _P]),
    "hlbm_set_state": (C.c_int, [_P, _P]),
    "hlbm_set_step_count": (C.c_int, [_P, C.c_int64]),
    "hlbm_set_stream": (C.c_int, [_P, _P]),
    "hlbm_halo_planes": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                                   C.POINTER(C.c_int64)]),
    "hlbm_next_halo_planes": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                                        C.POINTER(C.c_int64)]),
    "hlbm_ipc_export": (C.c_int, [_P, _P, C.POINTER(C.c_int32)]),
    "hlbm_ipc_open": (C.c_int, [_P, C.c_int32, _P, C.c_int32, C.c_int32]),
    "hlbm_ipc_sync": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "hlbm_halo_push": (C.c_int, [_P, C.c_int32, C.c_void_p]),
    "hlbm_ipc_close": (C.c_int, [_P]),
    "hlbm_step_begin": (C.c_int, [_P, C.c_int32]),
    "hlbm_step_range": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "hlbm_step_range_on": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_void_p]),
    "hlbm_step_end": (C.c_int, [_P]),
    "hlbm_state_buffer": (C.c_int, [_P, C.POINTER(_P), C.POINTER(C.c_int64)]),
    "hlbm_step_count": (C.c_int64, [_P]),
    "hlbm_launch_count": (C.c_int64, [_P]),
}

_lib = None


def load() -> C.CDLL:
    """Load libhlbm.so (built by ``__graft_entry__.build()`` / ``make -C csrc``)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("HLBM_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise ImportError(
            f"libhlbm.so not found at {path}: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(code: int, ctx=None) -> None:
    if code == HLBM_OK:
        return
    msg = "unknown error"
    if ctx is not None:
        raw = load().hlbm_last_error(ctx)
        msg = raw.decode() if raw else msg
    if code == HLBM_EINVAL:
        raise ValueError(msg)
    if code == HLBM_EDIVERGED:
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_DP)


def u32ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint32))
