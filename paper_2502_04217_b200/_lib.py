"""ctypes binding of libfftlasso_b200.so (the C ABI in include/fftlasso_b200.h).

The library is built in-tree (``paper_2502_04217_b200/libfftlasso_b200.so``,
see ``csrc/Makefile`` / ``__graft_entry__.build``).  There is no CPU fallback:
if the library or a CUDA device is missing, the first call raises
``BackendUnavailableError``.  Status codes map onto the reference's exception
types (errors.py:4-25).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    BackendUnavailableError,
    InteriorViolationError,
    NumericalBreakdownError,
    StalledError,
    UnsupportedShapeError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfftlasso_b200.so")

FL_OK, FL_E_SHAPE, FL_E_VALUE, FL_E_INTERIOR, FL_E_BREAKDOWN, FL_E_STALLED, FL_E_CUDA, FL_E_NOMEM = range(8)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_I = ctypes.c_int


class FlState(ctypes.Structure):
    _fields_ = [(f, _P) for f in ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2")]


class FlAssess(ctypes.Structure):
    _fields_ = [(f, _D) for f in ("stationarity", "dual_equality", "multiplier_gap", "primal",
                                   "complementarity", "min_product", "dot_nu_s1", "dot_nu_s2",
                                   "barrier_residual")]


class FlPcgResult(ctypes.Structure):
    _fields_ = [("iterations", _I64), ("converged", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("residual_norm", _D), ("norm0", _D)]


# name -> (restype, argtypes); every symbol declared in include/fftlasso_b200.h
SIGNATURES = {
    "fl_version": (_I, []),
    "fl_last_error": (ctypes.c_char_p, []),
    "fl_plan_create": (_I, [_I, ctypes.POINTER(_I64), _I, ctypes.POINTER(_P)]),
    "fl_plan_create_ex": (_I, [_I, ctypes.POINTER(_I64), _I, _I, ctypes.POINTER(_P)]),
    "fl_plan_destroy": (_I, [_P]),
    "fl_plan_n": (_I64, [_P]),
    "fl_synthesize": (_I, [_P, _P, _P, _P]),
    "fl_analyze": (_I, [_P, _P, _P, _P]),
    "fl_axis_pass": (_I, [_P, _I, _I, _P, _P, _P]),
    "fl_fused_mask_pass": (_I, [_P, _P, _P, _P, _P, ctypes.POINTER(_D), _P]),
    "fl_slab_pack_x": (_I, [_I64, _I64, _I64, _I, _P, _P, _P]),
    "fl_slab_unpack_x": (_I, [_I64, _I64, _I64, _I, _P, _P, _P]),
    "fl_slab_pack_y": (_I, [_I64, _I64, _I64, _I, _P, _P, _P]),
    "fl_slab_unpack_y": (_I, [_I64, _I64, _I64, _I, _P, _P, _P]),
    "fl_mask_build": (_I, [_I64, _P, _P, _P, ctypes.POINTER(_I64), _P]),
    "fl_noisy_embed": (_I, [ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.c_uint64,
                            _D, _P, _P, _P]),
    "fl_embed": (_I, [_I64, _P, _P, _P, _P, _P]),
    "fl_gather_observed": (_I, [_I64, _P, _P, _P, _P, _P]),
    "fl_gram": (_I, [_P, _P, _P, _P, _P]),
    "fl_residual_adjoint": (_I, [_P, _P, _P, _P, _P, _P]),
    "fl_barrier_diagonals": (_I, [_I64] + [_P] * 10 + [_P]),
    "fl_kkt_apply": (_I, [_P] * 8 + [ctypes.POINTER(_D), _P]),
    "fl_kkt_epilogue": (_I, [_I64] + [_P] * 6 + [ctypes.POINTER(_D), _P]),
    "fl_kkt_order": (_I, [_P]),
    "fl_kkt_apply_profiled": (_I, [_P] * 8 + [ctypes.POINTER(_D), ctypes.POINTER(_I), _P]),
    "fl_precond_apply": (_I, [_I64] + [_P] * 6 + [_P]),
    "fl_newton_rhs": (_I, [_I64, ctypes.POINTER(FlState), _P, _P, _P, _D, _D] + [_P] * 8 + [_P]),
    "fl_recover_eliminated": (_I, [_I64] + [_P] * 12 + [_P]),
    "fl_set_pcg_loop": (_I, [_I]),
    "fl_pcg_work_doubles": (_I64, [_I64]),
    "fl_pcg_kkt": (_I, [_P] * 7 + [_D, _D, _I64, ctypes.POINTER(FlPcgResult), _P, _I64, _P]),
    "fl_ipm_newton_pcg": (_I, [_P, _P, ctypes.POINTER(FlState), _P, _D, _D, _P, _P, _P, _P, _D, _D, _I64,
                               ctypes.POINTER(FlPcgResult), _P]),
    "fl_ipm_newton_step": (_I, [_P, _P, ctypes.POINTER(FlState), _P, _D, _D, _D, _P, _P, _P, _P, _D, _D, _I64,
                                _P, _P]),
    "fl_pcg_step_update_dev": (_I, [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "fl_pcg_step_pupdate_dev": (_I, [_I64, _P, _P, _P, _D, _P, _P, _P]),
    "fl_pcg_step_alpha": (_I, [_P, _P, _P, _P]),
    "fl_fused_mask_pass_dev": (_I, [_P, _P, _P, _P, _P, _P]),
    "fl_pcg_step_init": (_I, [_I64] + [_P] * 6 + [ctypes.POINTER(_D), _P]),
    "fl_pcg_step_update": (_I, [_I64, _P, _P, _D, _P, _P, _P, _P, ctypes.POINTER(_D), _P]),
    "fl_pcg_step_pupdate": (_I, [_I64, _P, _P, _P, _D, _P, ctypes.POINTER(_D), _P]),
    "fl_objective_terms": (_I, [_I64, _P, _P, _P, _I64, _P, ctypes.POINTER(_D), _P]),
    "fl_ipm_init": (_I, [_I64, ctypes.POINTER(FlState), _D, _P]),
    "fl_ipm_assess": (_I, [_I64, ctypes.POINTER(FlState), _P, _D, _D, ctypes.POINTER(FlAssess), _P]),
    "fl_ipm_ratios": (_I, [_I64, ctypes.POINTER(FlState), _P, _P, _D, _P, _P,
                           ctypes.POINTER(_D), _P]),
    "fl_ipm_direction": (_I, [_I64, ctypes.POINTER(FlState), _P, _P, _D] + [_P] * 8 + [_P]),
    "fl_ipm_update": (_I, [_I64, ctypes.POINTER(FlState), _P, _P, _D, _P, _P, _D, _D, _P]),
    "fl_ipm_update_explicit": (_I, [_I64, ctypes.POINTER(FlState), ctypes.POINTER(FlState),
                                    _D, _D, _P]),
    "fl_lasso_objective": (_I, [_P, _P, _P, _P, _D, _P, ctypes.POINTER(_D), _P]),
    "fl_dot": (_I, [_I64, _P, _P, ctypes.POINTER(_D), _P]),
    "fl_max_abs": (_I, [_I64, _P, ctypes.POINTER(_D), _P]),
    "fl_min": (_I, [_I64, _P, ctypes.POINTER(_D), _P]),
    "fl_ftb_ratio": (_I, [_I64, _P, _P, ctypes.POINTER(_D), _P]),
    "fl_axpy": (_I, [_I64, _D, _P, _P, _P]),
    "fl_xpby": (_I, [_I64, _P, _D, _P, _P]),
    "fl_mask_bragg": (_I, [_I, ctypes.POINTER(_I64), _I64, _D, _P, _P, ctypes.POINTER(_I64), _P]),
    "fl_soft_threshold": (_I, [_I64, _P, _D, _P, _P]),
    "fl_slab_x_to_y_peers": (_I, [_I64, _I64, _I64, _I, _I, _P, ctypes.POINTER(_P), _P]),
    "fl_slab_y_to_x_peers": (_I, [_I64, _I64, _I64, _I, _I, _P, ctypes.POINTER(_P), _P]),
    "fl_slab_x_to_y_peers_planes": (_I, [_I64, _I64, _I64, _I, _I, _I64, _I64, _P, ctypes.POINTER(_P), _P]),
    "fl_ipc_alloc": (_I, [_I64, ctypes.POINTER(_P), ctypes.c_char_p]),
    "fl_ipc_open": (_I, [ctypes.c_char_p, ctypes.POINTER(_P)]),
    "fl_ipc_close": (_I, [_P]),
    "fl_dev_free": (_I, [_P]),
    "fl_ista_step": (_I, [_I64, _P, _P, _P, _D, _P, ctypes.POINTER(_D), _P]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the shared library (no CUDA context is created)."""
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise BackendUnavailableError(
                        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                        " or `make -C paper_2502_04217_b200/csrc`")
                _lib = load_library()
    return _lib


def check(status: int) -> None:
    """Raise the reference exception type for a non-OK status."""
    if status == FL_OK:
        return
    msg = (lib().fl_last_error() or b"").decode(errors="replace")
    if status == FL_E_SHAPE:
        raise UnsupportedShapeError(msg)
    if status == FL_E_VALUE:
        raise ValueError(msg)
    if status == FL_E_INTERIOR:
        raise InteriorViolationError(msg)
    if status == FL_E_BREAKDOWN:
        raise NumericalBreakdownError(msg)
    if status == FL_E_STALLED:
        raise StalledError(msg)
    if status == FL_E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libfftlasso_b200 CUDA error: {msg}")


def call(name: str, *args):
    check(getattr(lib(), name)(*args))
