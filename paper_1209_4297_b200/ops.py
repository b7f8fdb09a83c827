"""Single device operators behind the reference's per-step API.

* ``stiff_value``      ~ ImplicitSolver.stiff_value   (steppers.py:66-70)
* ``nonstiff_value``   ~ SplitIVP.eval_nonstiff       (problems.py:133, :164)
* ``solve_shifted``    ~ ImplicitSolver.solve_shifted (steppers.py:72-78 -> linalg.py:59-63)
* ``level_step``       ~ predict_step / correct_step  (engine.py:193-231), fused

Each is one native kernel launch (``ridc_op_*``); inputs may be numpy
arrays (copied to the device) or CUDA tensors.
"""

import ctypes

import numpy as np

from . import _lib, device as D
from .errors import DimensionMismatch
from .problems import ProblemDescriptor

OP_STIFF, OP_NONSTIFF = 0, 1


def _check_len(n, *xs):
    """Every input holds n points (before any device transfer)."""
    for x in xs:
        size = x.numel() if hasattr(x, "numel") else np.asarray(x).size
        if size != n:
            raise DimensionMismatch(f"state has length {size}, expected {n}")


def _dev(x, dev, n):
    """x as a contiguous float64 vector of n points on CUDA device `dev`.

    The C-ABI takes no lengths (it writes nx*ny doubles), so the dimension is
    checked here, as the reference's steppers._check_step_args does
    (steppers.py:107-111): an undersized buffer raises DimensionMismatch
    instead of becoming an out-of-bounds device write."""
    t = D.torch()
    if isinstance(x, t.Tensor):
        if x.dtype != t.float64 or not x.is_cuda:
            raise TypeError("device inputs must be float64 CUDA tensors")
        if x.device.index != dev:
            raise ValueError(f"tensor on cuda:{x.device.index}, the operation runs on cuda:{dev}")
        if x.numel() != n:
            raise DimensionMismatch(f"state has length {x.numel()}, expected {n}")
        return x.contiguous().view(-1)
    a = np.asarray(x)
    if a.size != n:
        raise DimensionMismatch(f"state has length {a.size}, expected {n}")
    return D.to_device(a.reshape(-1), dev)


def _out(x, like_tensor):
    t = D.torch()
    return like_tensor if isinstance(x, t.Tensor) else D.to_host(like_tensor)


def _apply(pd: ProblemDescriptor, op: int, y, dev: int = 0):
    yd = _dev(y, dev, pd.dimension)
    out = D.torch().empty_like(yd)
    cp = pd.to_c()
    _lib.check(_lib.lib().ridc_op_apply(ctypes.byref(cp), op, yd.data_ptr(), out.data_ptr(), dev))
    return _out(y, out)


def stiff_value(pd: ProblemDescriptor, y, dev: int = 0):
    return _apply(pd, OP_STIFF, y, dev)


def nonstiff_value(pd: ProblemDescriptor, y, dev: int = 0):
    return _apply(pd, OP_NONSTIFF, y, dev)


def solve_shifted(pd: ProblemDescriptor, coeff: float, rhs, dev: int = 0):
    """x with (I - coeff * L_S) x = rhs."""
    rd = _dev(rhs, dev, pd.dimension)
    x = D.torch().empty_like(rd)
    cp = pd.to_c()
    _lib.check(_lib.lib().ridc_op_solve(ctypes.byref(cp), float(coeff), rd.data_ptr(),
                                        x.data_ptr(), dev))
    return _out(rhs, x)


def level_step(pd: ProblemDescriptor, dt: float, eta, window=(), cs=(), cn=(), dev: int = 0):
    """Fused level step: rhs = eta + dt f^N(eta) + sum_k cs_k f^S(w_k) + cn_k f^N(w_k);
    returns (I - dt L_S)^{-1} rhs."""
    _check_len(pd.dimension, eta, *window)
    ed = _dev(eta, dev, pd.dimension)
    wins = [_dev(w, dev, pd.dimension) for w in window]
    k = len(wins)
    out = D.torch().empty_like(ed)
    ptrs = (ctypes.c_void_p * max(k, 1))(*[w.data_ptr() for w in wins])
    csa = np.ascontiguousarray(cs, dtype=np.float64) if k else np.zeros(1)
    cna = np.ascontiguousarray(cn, dtype=np.float64) if k else np.zeros(1)
    cp = pd.to_c()
    dp = ctypes.POINTER(ctypes.c_double)
    _lib.check(_lib.lib().ridc_op_step(
        ctypes.byref(cp), float(dt), ed.data_ptr(), k, ptrs,
        csa.ctypes.data_as(dp), cna.ctypes.data_as(dp), out.data_ptr(), dev))
    return _out(eta, out)


def level_step_rows(pd: ProblemDescriptor, dt: float, eta, fs_rows, fn_rows, w, i_new, i_old,
                    dev: int = 0):
    """Reference-form corrector (LevelWindow with f^S/f^N rows, engine.py:177-187):
    rhs = eta + dt f^N(eta) - dt fs[i_new] - dt fn[i_old] + sum_a w_a (fs_a + fn_a)."""
    _check_len(pd.dimension, eta)
    k = len(w)
    if len(fs_rows) != k or len(fn_rows) != k:
        raise DimensionMismatch(f"window holds {len(fs_rows)}/{len(fn_rows)} rows, weights need {k}")
    _check_len(pd.dimension, *fs_rows, *fn_rows)
    ed = _dev(eta, dev, pd.dimension)
    rows = [_dev(r, dev, pd.dimension) for r in list(fs_rows) + list(fn_rows)]
    ca = [w[a] - (dt if a == i_new else 0.0) for a in range(k)] + \
         [w[a] - (dt if a == i_old else 0.0) for a in range(k)]
    out = D.torch().empty_like(ed)
    ptrs = (ctypes.c_void_p * len(rows))(*[r.data_ptr() for r in rows])
    caa = np.ascontiguousarray(ca, dtype=np.float64)
    cp = pd.to_c()
    _lib.check(_lib.lib().ridc_op_step_rows(
        ctypes.byref(cp), float(dt), ed.data_ptr(), len(rows), ptrs,
        caa.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.data_ptr(), dev))
    return _out(eta, out)
