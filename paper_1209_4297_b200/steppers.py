"""ARK (IMEX) steps on the device: the reference's steppers.py comparators.

``integrate_ark(ivp, tab, t0, y0, t1, steps, solver=None)`` and
``ark_step(ivp, tab, t_n, y_n, dt, solver=None)`` keep the signatures of
steppers.py:122-155 and march on the GPU through ``ridc_ark_*``
(include/ridc_b200.h): every stage is one fused launch (stage sum with
recomputed f^S / f^N, shifted solve with that stage's factors), the whole
march one CUDA graph.  ``fbe_step`` (steppers.py:114-119) is the RIDC
predictor step.  The ``solver`` argument is accepted for signature
compatibility and ignored (factors live on the device).  There is no CPU
fallback: a bare-callable SplitIVP raises ConfigError.
"""

import ctypes

import numpy as np

from . import _lib
from . import device as D
from .errors import DimensionMismatch
from .problems import as_descriptor
from .tableaus import ButcherPair

__all__ = ["ArkEngine", "ark_step", "integrate_ark", "fbe_step"]


def _check_step_args(n: int, y_n: np.ndarray, dt: float) -> None:
    """steppers.py:105-109."""
    if dt <= 0:
        raise ValueError(f"dt must be positive, got {dt}")
    if y_n.shape[0] != n:
        raise DimensionMismatch(f"state has length {y_n.shape[0]}, expected {n}")


class ArkEngine:
    """A prepared device ARK march (``ridc_ark_create``): tiling, per-stage
    factors, the CUDA graph of all steps."""

    def __init__(self, ivp, tab: ButcherPair, t0: float, t1: float, steps: int, device: int = 0):
        if steps < 1:
            raise ValueError("steps must be positive")
        self.desc = as_descriptor(ivp)
        self.problem = self.desc.problem
        self.tab = tab
        self.steps = int(steps)
        D.require_cuda(device)
        s = tab.stages
        arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in
                (tab.a_implicit, tab.a_explicit, tab.b_implicit, tab.b_explicit)]
        self._keep = arrs
        cp = self.problem.to_c()
        h = ctypes.c_void_p()
        _lib.check_ark(_lib.lib().ridc_ark_create(
            ctypes.byref(cp), float(t0), float(t1), self.steps, s, *[a.ctypes.data for a in arrs],
            device, ctypes.byref(h)))
        self._h = h

    @property
    def info(self) -> dict:
        nl, ni = ctypes.c_int64(0), ctypes.c_int32(0)
        _lib.check_ark(_lib.lib().ridc_ark_info(self._h, ctypes.byref(nl), ctypes.byref(ni)), self._h)
        path = _lib.lib().ridc_ark_path(self._h)
        return {"kernel_launches": nl.value, "items_per_step": ni.value, "path": path,
                "path_name": _lib.PATH_NAMES.get(path, "?")}

    def run(self, y0) -> tuple:
        """March from a host state -> (final ndarray, device seconds)."""
        n = self.problem.dimension
        y0 = np.ascontiguousarray(y0, dtype=np.float64)
        if y0.shape != (n,):
            raise DimensionMismatch(f"state has length {y0.shape[0]}, expected {n}")
        out = np.empty(n)
        wall = ctypes.c_double(0.0)
        _lib.check_ark(_lib.lib().ridc_ark_run(self._h, y0.ctypes.data, out.ctypes.data, ctypes.byref(wall)),
                       self._h)
        return out, wall.value

    def run_device(self, y0_dev, out_dev) -> float:
        wall = ctypes.c_double(0.0)
        _lib.check_ark(_lib.lib().ridc_ark_run_device(self._h, y0_dev.data_ptr(), out_dev.data_ptr(),
                                                      ctypes.byref(wall)), self._h)
        return wall.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().ridc_ark_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def integrate_ark(ivp, tab: ButcherPair, t0: float, y0, t1: float, steps: int, solver=None) -> np.ndarray:
    """March ``steps`` uniform ARK steps from (t0, y0) to t1 (steppers.py:145-155)."""
    if steps < 1:
        raise ValueError("steps must be positive")
    with ArkEngine(ivp, tab, t0, t1, steps) as eng:
        final, _ = eng.run(np.asarray(y0, dtype=np.float64))
    return final


def ark_step(ivp, tab: ButcherPair, t_n: float, y_n, dt: float, solver=None) -> np.ndarray:
    """One coupled DIRK/explicit step (steppers.py:122-142)."""
    y_n = np.asarray(y_n, dtype=np.float64)
    _check_step_args(as_descriptor(ivp).problem.dimension, y_n, dt)
    # the problems are autonomous: march (0, dt) so the step uses the caller's dt
    # bit for bit ((t_n + dt) - t_n can differ from dt in the last bits)
    with ArkEngine(ivp, tab, 0.0, dt, 1) as eng:
        final, _ = eng.run(y_n)
    return final


def fbe_step(ivp, t_n: float, y_n, dt: float, solver=None) -> np.ndarray:
    """Forward-backward Euler (steppers.py:114-119): the RIDC predictor step."""
    from .engine import predict_step
    y_n = np.asarray(y_n, dtype=np.float64)
    _check_step_args(as_descriptor(ivp).problem.dimension, y_n, dt)
    eta, _, _ = predict_step(ivp, t_n, y_n, dt)
    return eta

