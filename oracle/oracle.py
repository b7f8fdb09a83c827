"""ctypes front-end of the CPU oracle (oracle/ridc_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  Never imported by the
product package.  See ridc_oracle.c for what it restates (file:line of the
reference for every function).
"""

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libridc_oracle.so")
_lock = threading.Lock()
_lib = None

OK, CONFIG, DIM, NONFINITE, PROTOCOL = 0, 1, 2, 3, 4


class _Problem(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("c_x", ctypes.c_double), ("c_y", ctypes.c_double),
        ("d_x", ctypes.c_double), ("d_y", ctypes.c_double),
        ("rho", ctypes.c_double), ("h_x", ctypes.c_double), ("h_y", ctypes.c_double),
    ]


def build() -> str:
    """Compile the oracle with its Makefile (gcc) if the .so is missing or stale."""
    src = os.path.join(_HERE, "ridc_oracle.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            dp = ctypes.POINTER(ctypes.c_double)
            pp = ctypes.POINTER(_Problem)
            L.orc_fs.argtypes = [pp, dp, dp]
            L.orc_fn.argtypes = [pp, dp, dp]
            L.orc_solve.argtypes = [pp, ctypes.c_double, dp, dp]
            L.orc_solve.restype = ctypes.c_int
            L.orc_run.argtypes = [pp, ctypes.c_int, ctypes.c_long, ctypes.c_int, ctypes.c_double,
                                  dp, dp, dp, dp, dp, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_long, dp]
            L.orc_run.restype = ctypes.c_int
            L.orc_predict_step.argtypes = [pp, ctypes.c_double, dp, dp, dp, dp]
            L.orc_predict_step.restype = ctypes.c_int
            L.orc_correct_step.argtypes = [pp, ctypes.c_double, dp, dp, dp, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, dp, dp, dp, dp]
            L.orc_correct_step.restype = ctypes.c_int
            L.orc_last_error.restype = ctypes.c_char_p
            _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _prob(pd) -> _Problem:
    return _Problem(pd.kind, pd.nx, pd.ny, 0, pd.c_x, pd.c_y, pd.d_x, pd.d_y, pd.rho, pd.h_x, pd.h_y)


def _vec(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if n is not None and a.shape[0] != n:
        raise ValueError(f"length {a.shape[0]} != {n}")
    return a


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        super().__init__(f"oracle status {code}: {msg}")


def _check(rc):
    if rc != OK:
        raise OracleError(rc, lib().orc_last_error().decode())


def stiff(pd, u):
    u = _vec(u, pd.nx * pd.ny)
    out = np.empty_like(u)
    p = _prob(pd)
    lib().orc_fs(ctypes.byref(p), _ptr(u), _ptr(out))
    return out


def nonstiff(pd, u):
    u = _vec(u, pd.nx * pd.ny)
    out = np.empty_like(u)
    p = _prob(pd)
    lib().orc_fn(ctypes.byref(p), _ptr(u), _ptr(out))
    return out


def solve(pd, coeff, rhs):
    """x with (I - coeff * L_S) x = rhs (replaces linalg.qr_solve)."""
    rhs = _vec(rhs, pd.nx * pd.ny)
    x = np.empty_like(rhs)
    p = _prob(pd)
    _check(lib().orc_solve(ctypes.byref(p), coeff, _ptr(rhs), _ptr(x)))
    return x


def predict_step(pd, dt, eta):
    eta = _vec(eta, pd.nx * pd.ny)
    out = [np.empty_like(eta) for _ in range(3)]
    p = _prob(pd)
    _check(lib().orc_predict_step(ctypes.byref(p), dt, _ptr(eta), *[_ptr(o) for o in out]))
    return tuple(out)


def correct_step(pd, dt, eta, fs_win, fn_win, i_new, i_old, weights):
    n = pd.nx * pd.ny
    eta = _vec(eta, n)
    fs_win = np.ascontiguousarray(fs_win, dtype=np.float64)
    fn_win = np.ascontiguousarray(fn_win, dtype=np.float64)
    w = _vec(weights)
    k = w.shape[0]
    out = [np.empty_like(eta) for _ in range(3)]
    p = _prob(pd)
    _check(lib().orc_correct_step(ctypes.byref(p), dt, _ptr(eta), _ptr(fs_win), _ptr(fn_win), k,
                                  i_new, i_old, _ptr(w), *[_ptr(o) for o in out]))
    return tuple(out)


def run(pd, y0, levels, steps, restarts, dt, weights, workers=1, record_trajectory=False,
        level_finals=False, watchdog_seconds=30.0, max_steps=0):
    """Full RIDC-FBE run (run_serial / run_pipelined semantics).

    Returns dict(final_state, level_finals, trajectory, wall_seconds).
    ``max_steps`` > 0 bounds the run to that many steps of one interval
    (CPU-baseline sampling).
    """
    n = pd.nx * pd.ny
    y0 = _vec(y0, n)
    w = _vec(weights)
    final = np.empty(n)
    lf = np.empty((levels, n)) if level_finals else None
    traj = np.empty((steps + 1, n)) if record_trajectory else None
    wall = ctypes.c_double(0.0)
    p = _prob(pd)
    _check(lib().orc_run(ctypes.byref(p), levels, steps, restarts, dt, _ptr(w), _ptr(y0),
                         _ptr(final), _ptr(lf), _ptr(traj), workers, watchdog_seconds,
                         max_steps, ctypes.byref(wall)))
    return {"final_state": final, "level_finals": lf, "trajectory": traj,
            "wall_seconds": wall.value}


def ark(pd, a_implicit, a_explicit, b_implicit, b_explicit, y0, t0, t1, steps):
    """integrate_ark / ark_step (steppers.py:122-155) with stage_accumulate's
    summation order (kernels.py:149-158: out = y, then += dt*aI*ks + dt*aE*kn per
    stage j); the shifted solves are orc_solve (Thomas / Sherman-Morrison) in
    place of the dense QR.  Raises RuntimeError with the reference's message on
    a non-finite step (steppers.py:153-154)."""
    a_implicit, a_explicit = np.asarray(a_implicit), np.asarray(a_explicit)
    b_implicit, b_explicit = np.asarray(b_implicit), np.asarray(b_explicit)
    dt = (t1 - t0) / steps
    s = b_implicit.shape[0]
    y = np.array(y0, dtype=np.float64)
    n = y.shape[0]
    for k in range(steps):
        ks = np.empty((s, n))
        kn = np.empty((s, n))
        for i in range(s):
            rhs = y.copy()
            for j in range(i):
                rhs += (dt * a_implicit[i, j]) * ks[j] + (dt * a_explicit[i, j]) * kn[j]
            aii = a_implicit[i, i]
            ys = rhs if aii == 0.0 else solve(pd, aii * dt, rhs)
            ks[i] = stiff(pd, ys)
            kn[i] = nonstiff(pd, ys)
        out = y.copy()
        for j in range(s):
            out += (dt * b_implicit[j]) * ks[j] + (dt * b_explicit[j]) * kn[j]
        y = out
        if not np.isfinite(y).all():
            raise RuntimeError(f"ARK march produced non-finite entries at step {k + 1}")
    return y
