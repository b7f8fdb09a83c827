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
from .problems import ProblemDescriptor

OP_STIFF, OP_NONSTIFF = 0, 1


def _dev(x, dev):
    t = D.torch()
    if isinstance(x, t.Tensor):
        if x.dtype != t.float64 or not x.is_cuda:
            raise TypeError("device inputs must be float64 CUDA tensors")
        return x.contiguous()
    return D.to_device(x, dev)


def _out(x, like_tensor):
    t = D.torch()
    return like_tensor if isinstance(x, t.Tensor) else D.to_host(like_tensor)


def _apply(pd: ProblemDescriptor, op: int, y, dev: int = 0):
    yd = _dev(y, dev)
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
    rd = _dev(rhs, dev)
    x = D.torch().empty_like(rd)
    cp = pd.to_c()
    _lib.check(_lib.lib().ridc_op_solve(ctypes.byref(cp), float(coeff), rd.data_ptr(),
                                        x.data_ptr(), dev))
    return _out(rhs, x)


def level_step(pd: ProblemDescriptor, dt: float, eta, window=(), cs=(), cn=(), dev: int = 0):
    """Fused level step: rhs = eta + dt f^N(eta) + sum_k cs_k f^S(w_k) + cn_k f^N(w_k);
    returns (I - dt L_S)^{-1} rhs."""
    ed = _dev(eta, dev)
    wins = [_dev(w, dev) for w in window]
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
    ed = _dev(eta, dev)
    k = len(w)
    rows = [_dev(r, dev) for r in list(fs_rows) + list(fn_rows)]
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
