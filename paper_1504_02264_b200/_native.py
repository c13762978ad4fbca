"""ctypes binding of liblesb200.so (the C ABI in include/les_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every device entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# LESB_LIB: an alternative build of the same library (kernel experiments)
LIB_PATH = os.environ.get("LESB_LIB") or os.path.join(PKG, "liblesb200.so")

LESB_U, LESB_V, LESB_W, LESB_P, LESB_MASK, LESB_FGH, LESB_FGH_OLD, LESB_RHS = range(8)
LESB_REDBLACK, LESB_TWINNED = 0, 1
LESB_HALO_STORED, LESB_HALO_PRESS = 0, 1
LESB_OK, LESB_NONFINITE = 0, 1
STAGE_NAMES = ("velnw", "bondv1", "velfg", "feedbf", "les", "adam", "press")

FP = C.POINTER(C.c_float)
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)


class lesb_desc(C.Structure):
    _fields_ = [
        ("im", C.c_int), ("jm", C.c_int), ("km", C.c_int),
        ("i_offset", C.c_int), ("west_boundary", C.c_int), ("east_boundary", C.c_int),
        ("dx1", FP), ("dy1", FP), ("dzn", FP),
        ("dt", C.c_float), ("vn", C.c_float), ("cs", C.c_float),
        ("csd2", FP), ("csd2_scalar", C.c_float),
        ("device", C.c_int),
    ]


class lesb_coeffs(C.Structure):
    _fields_ = [
        ("cn1", FP), ("cn1_scalar", C.c_float),
        ("cn2l", FP), ("cn2s", FP), ("cn3l", FP), ("cn3s", FP), ("cn4l", FP), ("cn4s", FP),
    ]


_SIGS = {
    "lesb_last_error": (C.c_char_p, []),
    "lesb_abi_version": (C.c_int, []),
    "lesb_create": (C.c_int, [C.POINTER(lesb_desc), C.POINTER(C.c_void_p)]),
    "lesb_destroy": (C.c_int, [C.c_void_p]),
    "lesb_set_coeffs": (C.c_int, [C.c_void_p, C.POINTER(lesb_coeffs)]),
    "lesb_set_physics": (C.c_int, [C.c_void_p, C.c_float, C.c_float, C.c_float, FP, C.c_float]),
    "lesb_upload": (C.c_int, [C.c_void_p, C.c_int, FP]),
    "lesb_download": (C.c_int, [C.c_void_p, C.c_int, FP]),
    "lesb_stage_upload": (C.c_int, [C.c_void_p, C.c_int, FP]),
    "lesb_stage_commit": (C.c_int, [C.c_void_p]),
    "lesb_download_async": (C.c_int, [C.c_void_p, C.c_int, FP]),
    "lesb_copies_wait": (C.c_int, [C.c_void_p]),
    "lesb_device_ptr": (C.c_void_p, [C.c_void_p, C.c_int]),
    "lesb_stream": (C.c_void_p, [C.c_void_p]),
    "lesb_synchronize": (C.c_int, [C.c_void_p]),
    "lesb_check_finite": (C.c_int, [C.c_void_p, IP]),
    "lesb_velnw": (C.c_int, [C.c_void_p]),
    "lesb_bondv1": (C.c_int, [C.c_void_p, FP, FP, FP]),
    "lesb_velfg": (C.c_int, [C.c_void_p]),
    "lesb_feedbf": (C.c_int, [C.c_void_p]),
    "lesb_les_viscosity": (C.c_int, [C.c_void_p]),
    "lesb_adam": (C.c_int, [C.c_void_p]),
    "lesb_divergence": (C.c_int, [C.c_void_p, FP]),
    "lesb_strain_magnitude": (C.c_int, [C.c_void_p, FP]),
    "lesb_press": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_float, DP]),
    "lesb_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_int]),
    "lesb_link_nccl": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "lesb_link_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "lesb_group_step": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, FP, FP, FP, C.c_int, C.c_int, C.c_float, DP, IP]),
    "lesb_group_sor_solve": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, DP]),
    "lesb_sor_solve": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_int, DP]),
    "lesb_step": (C.c_int, [C.c_void_p, FP, FP, FP, C.c_int, C.c_int, C.c_float, DP, IP]),
    "lesb_run_steps": (C.c_int, [C.c_void_p, C.c_int, FP, C.c_int, C.c_int, C.c_int, C.c_float, IP, IP]),
    "lesb_set_inflow": (C.c_int, [C.c_void_p, FP, FP, FP]),
    "lesb_step_async": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_float]),
    "lesb_poll_failure": (C.c_int, [C.c_void_p, IP, IP, IP]),
    "lesb_kernels_per_step": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "lesb_copy_state": (C.c_int, [C.c_void_p, C.c_void_p]),
    "lesb_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "lesb_set_sor_path": (C.c_int, [C.c_void_p, C.c_int]),
    "lesb_sor_path_in_use": (C.c_int, [C.c_void_p, C.c_int]),
    "lesb_set_default_sor_path": (C.c_int, [C.c_int]),
    "lesb_last_step_times": (C.c_int, [C.c_void_p, FP]),
    "lesb_solve_pressure": (C.c_int, [C.c_int, C.c_int, C.c_int, FP, FP, C.POINTER(lesb_coeffs),
                                      C.c_float, C.c_int, C.c_int, C.c_int, FP, DP, C.c_int]),
    "lesb_redblack_iteration": (C.c_int, [C.c_int, C.c_int, C.c_int, FP, FP, C.POINTER(lesb_coeffs),
                                          C.c_float, C.c_int, DP, C.c_int]),
    "lesb_twinned_sweep": (C.c_int, [C.c_int, C.c_int, C.c_int, FP, FP, FP, C.POINTER(lesb_coeffs),
                                     C.c_float, DP, C.c_int]),
    "lesb_boundary_decode": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_longlong, C.c_longlong, IP, IP, IP]),
    "lesb_boundary_audit": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_longlong)]),
    "lesb_boundp_faces": (C.c_int, [C.c_void_p]),
}

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    """A CUDA / argument error reported by liblesb200."""


def load():
    """Load liblesb200.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1504_02264_b200.build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().lesb_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> int:
    if rc < 0:
        raise NativeError(f"{what} failed ({rc}): {last_error()}")
    return rc


def fptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(FP)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(DP)


def f32c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def make_coeffs(c, keep: list) -> lesb_coeffs:
    """lesb_coeffs view of a SorCoeffs (arrays kept alive in ``keep``).  A
    constant cn1 field is passed as a scalar (4 B/cell/iteration less)."""
    cn1 = f32c(c.cn1)
    vecs = [f32c(getattr(c, n)) for n in ("cn2l", "cn2s", "cn3l", "cn3s", "cn4l", "cn4s")]
    keep.extend(vecs)
    uniform = cn1.size > 0 and bool(np.all(cn1 == cn1.flat[0]))
    if uniform:
        cn1_ptr, cn1s = None, float(cn1.flat[0])
    else:
        keep.append(cn1)
        cn1_ptr, cn1s = fptr(cn1), 0.0
    return lesb_coeffs(cn1_ptr, cn1s, *[fptr(v) for v in vecs])
