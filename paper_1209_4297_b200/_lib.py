"""ctypes binding of the native library (include/ridc_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a)
into ``paper_1209_4297_b200/libridc_b200.so``.  There is no fallback: if the
shared object is missing or cannot load, every entry point raises.
"""

import ctypes
import os
import threading

from .errors import raise_for_status
from .problems import CProblem

# RIDC_CHECKED=1 loads the checked build (RIDC_CHECK assertions compiled in,
# __graft_entry__.build(checked=True)): diagnostics only, slower
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        "libridc_b200_checked.so" if os.environ.get("RIDC_CHECKED") == "1" else "libridc_b200.so")

_lock = threading.Lock()
_lib = None


class RidcInfo(ctypes.Structure):
    _fields_ = [
        ("levels", ctypes.c_int32), ("restarts", ctypes.c_int32), ("steps", ctypes.c_int64),
        ("ticks_per_interval", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
        ("tile", ctypes.c_int32), ("halo", ctypes.c_int32), ("items_per_level", ctypes.c_int32),
        ("threads", ctypes.c_int32), ("ring_vectors", ctypes.c_int64),
        ("lam", ctypes.c_double), ("r", ctypes.c_double),
        ("path", ctypes.c_int32), ("fell_back", ctypes.c_int32),
    ]


(PATH_TICK, PATH_RESIDENT_FEBE, PATH_RESIDENT_LEVELS, PATH_CARRY_FEBE, PATH_SWEEP_FEBE, PATH_SWEEP2D_FEBE,
 PATH_SWEEP2D_LEVELS, PATH_SWEEP_LEVELS, PATH_SWEEP_WARP_FEBE, PATH_CARRY_LEVELS,
 PATH_RESIDENT_CARRY_LEVELS, PATH_WARP_CARRY_FEBE) = range(12)
PATH_NAMES = {PATH_TICK: "tick", PATH_RESIDENT_FEBE: "resident_febe", PATH_RESIDENT_LEVELS: "resident_levels",
              PATH_CARRY_FEBE: "carry_febe", PATH_SWEEP_FEBE: "sweep_febe", PATH_SWEEP2D_FEBE: "sweep2d_febe",
              PATH_SWEEP2D_LEVELS: "sweep2d_levels", PATH_SWEEP_LEVELS: "sweep_levels",
              PATH_SWEEP_WARP_FEBE: "sweep_warp_febe", PATH_CARRY_LEVELS: "carry_levels",
              PATH_RESIDENT_CARRY_LEVELS: "resident_carry_levels", PATH_WARP_CARRY_FEBE: "warp_carry_febe"}


# name -> (restype, argtypes); every symbol include/ridc_b200.h declares
_P = ctypes.POINTER
_d = ctypes.c_double
_dp = _P(ctypes.c_double)
_vp = ctypes.c_void_p
SIGNATURES = {
    "ridc_create": (ctypes.c_int, [_P(CProblem), _d, _d, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                   _vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, _P(_vp)]),
    "ridc_run": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _dp]),
    "ridc_run_device": (ctypes.c_int, [_vp, _vp, _vp, _dp]),
    "ridc_info_get": (ctypes.c_int, [_vp, _P(RidcInfo)]),
    "ridc_set_watchdog": (ctypes.c_int, [_vp, _d]),
    "ridc_destroy": (ctypes.c_int, [_vp]),
    "ridc_last_error": (ctypes.c_char_p, [_vp]),
    "ridc_op_apply": (ctypes.c_int, [_P(CProblem), ctypes.c_int32, _vp, _vp, ctypes.c_int32]),
    "ridc_op_solve": (ctypes.c_int, [_P(CProblem), _d, _vp, _vp, ctypes.c_int32]),
    "ridc_op_step": (ctypes.c_int, [_P(CProblem), _d, _vp, ctypes.c_int32, _P(_vp), _dp, _dp, _vp,
                                    ctypes.c_int32]),
    "ridc_op_step_rows": (ctypes.c_int, [_P(CProblem), _d, _vp, ctypes.c_int32, _P(_vp), _dp, _vp,
                                         ctypes.c_int32]),
    "ridc_debug_phase_trace": (ctypes.c_int, [_vp, _P(ctypes.c_longlong), ctypes.c_int32]),
    "ridc_pipe_handle_bytes": (ctypes.c_int64, []),
    "ridc_pipe_create": (ctypes.c_int, [_P(CProblem), _d, _d, ctypes.c_int32, ctypes.c_int64,
                                        ctypes.c_int32, _vp, ctypes.c_int64, ctypes.c_int32,
                                        ctypes.c_int32, ctypes.c_int32, _d, _P(_vp)]),
    "ridc_pipe_create_shard": (ctypes.c_int, [_P(CProblem), _d, _d, ctypes.c_int32, ctypes.c_int64,
                                              ctypes.c_int32, _vp, ctypes.c_int64, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                              _d, _P(_vp)]),
    "ridc_pipe_connect_shard": (ctypes.c_int, [_vp, _P(_vp)]),
    "ridc_pipe_export": (ctypes.c_int, [_vp, _vp]),
    "ridc_pipe_connect": (ctypes.c_int, [_vp, _vp, _vp]),
    "ridc_pipe_run_interval": (ctypes.c_int, [_vp, ctypes.c_int32, _vp, _vp, _dp]),
    "ridc_pipe_info": (ctypes.c_int, [_vp, _P(RidcInfo)]),
    "ridc_pipe_reset": (ctypes.c_int, [_vp]),
    "ridc_pipe_set_resident": (ctypes.c_int, [_vp, ctypes.c_int32]),
    "ridc_pipe_resident": (ctypes.c_int, [_vp]),
    "ridc_pipe_destroy": (ctypes.c_int, [_vp]),
    "ridc_pipe_last_error": (ctypes.c_char_p, [_vp]),
    "ridc_ark_create": (ctypes.c_int, [_P(CProblem), _d, _d, ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp, _vp,
                                       ctypes.c_int32, _P(_vp)]),
    "ridc_ark_run": (ctypes.c_int, [_vp, _vp, _vp, _dp]),
    "ridc_ark_run_device": (ctypes.c_int, [_vp, _vp, _vp, _dp]),
    "ridc_ark_info": (ctypes.c_int, [_vp, _P(ctypes.c_int64), _P(ctypes.c_int32)]),
    "ridc_ark_path": (ctypes.c_int, [_vp]),
    "ridc_ark_destroy": (ctypes.c_int, [_vp]),
    "ridc_ark_last_error": (ctypes.c_char_p, [_vp]),
    "ridc_shards_create": (ctypes.c_int, [_P(CProblem), _d, _d, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                          _vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _P(_vp)]),
    "ridc_shards_create_multi": (ctypes.c_int, [_P(CProblem), _d, _d, ctypes.c_int32, ctypes.c_int64,
                                                ctypes.c_int32, _vp, ctypes.c_int64, ctypes.c_int32, _vp, _d,
                                                _P(_vp)]),
    "ridc_shards_run": (ctypes.c_int, [_vp, _vp, _vp, _dp]),
    "ridc_shards_info": (ctypes.c_int, [_vp, _P(ctypes.c_int64)]),
    "ridc_shards_destroy": (ctypes.c_int, [_vp]),
    "ridc_shards_last_error": (ctypes.c_char_p, [_vp]),
}


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"native library {LIB_PATH} not built; run __graft_entry__.build() "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(code: int, ctx=None) -> None:
    if code:
        msg = lib().ridc_last_error(ctx)
        raise_for_status(code, msg.decode() if msg else "")


def check_pipe(code: int, pipe=None) -> None:
    if code:
        msg = lib().ridc_pipe_last_error(pipe)
        raise_for_status(code, msg.decode() if msg else "")


def check_ark(code: int, ark=None) -> None:
    if code:
        msg = lib().ridc_ark_last_error(ark)
        raise_for_status(code, msg.decode() if msg else "")


def check_shards(code: int, g=None) -> None:
    if code:
        msg = lib().ridc_shards_last_error(g)
        raise_for_status(code, msg.decode() if msg else "")
