"""RIDC-FBE marching on B200: the reference's engine API over the native path.

Public surface mirrors ``ridc.engine`` (pkg/src/ridc/engine.py):
``RidcConfig`` (:57-91), ``RidcSolution`` (:94-100), ``startup_delay``
(:50-54), ``restart_partition`` (:103-118), ``LevelWindow`` (:200-210),
``predict_step`` / ``correct_step`` (:193-231), ``run_serial`` (:476-494),
``run_pipelined`` (:497-522).

Both executors run the same device engine (``ridc_create`` + ``ridc_run``):
all levels of the lagged pipeline march on one GPU, one fused kernel per
tick, the whole run replayed from a CUDA graph.  Every level's arithmetic
depends only on published states, never on timing, so results are bitwise
identical between executors and across ``workers`` -- the reference's
determinism gate (engine.py:497-503) holds by construction and is tested.
The one-level-per-GPU pipeline across processes lives in
:mod:`paper_1209_4297_b200.distributed`.

Differences a reference user may notice:
* the problem must be structured (our ``build_*`` systems, or a reference
  system object carrying ``.spec``); opaque callables raise ConfigError;
* ``wall_seconds`` is device time of the marching (CUDA events), setup excluded
  as in the reference (engine.py:482);
* ``trace`` is the deterministic tick schedule (tick-major, level ascending).
"""

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib, device as D, ops
from .errors import ConfigError, DimensionMismatch, PipelineProtocolError
from .problems import StructuredIVP, as_descriptor
from .quadrature import MAX_LEVEL, pack_weight_tables

__all__ = ["RidcConfig", "RidcSolution", "LevelWindow", "Engine", "startup_delay",
           "restart_partition", "predict_step", "correct_step", "run_serial", "run_pipelined",
           "pipeline_devices", "schedule", "MAX_LEVELS"]

MAX_LEVELS = MAX_LEVEL + 1
RECORD_TRAJECTORY = 1
TICK_ONLY = 2   # include/ridc_b200.h RIDC_TICK_ONLY (testing: disable the resident march)
RESIDENT_SEGMENTS = 4   # RIDC_RESIDENT_SEGMENTS (experimental: resident march on segmented lines)


def startup_delay(j: int) -> int:
    """Steps level j waits before entering the pipeline: j(j+1)/2 (engine.py:50-54)."""
    if j < 0:
        raise ValueError("level must be non-negative")
    return j * (j + 1) // 2


@dataclass
class RidcConfig:
    """One run; total order = levels.  Validation as engine.py:71-87.

    ``workers`` keeps the reference meaning (1..levels) and is validated; on
    one device all levels share the GPU regardless (results do not depend on
    it).  ``device`` selects the CUDA ordinal.
    """

    levels: int
    steps: int
    restarts: int = 1
    workers: int = 1
    newton_tol: float = 1e-12
    newton_max_iter: int = 25
    record_trajectory: bool = False
    trace: bool = False
    watchdog_seconds: float = 30.0
    device: int = 0

    def __post_init__(self):
        if not 1 <= self.levels <= MAX_LEVELS:
            raise ConfigError(f"levels must be in 1..{MAX_LEVELS}, got {self.levels}")
        if self.steps < 1 or self.restarts < 1:
            raise ConfigError("steps and restarts must be positive")
        if self.steps % self.restarts:
            raise ConfigError(
                f"steps ({self.steps}) must be divisible by restarts ({self.restarts})")
        fill = startup_delay(self.levels) + 1
        per = self.steps // self.restarts
        if per < fill:
            raise ConfigError(
                f"each restart interval has {per} steps; {self.levels} levels need >= {fill}")
        if not 1 <= self.workers <= self.levels:
            raise ConfigError(f"workers must be in 1..levels, got {self.workers}")

    @property
    def steps_per_interval(self) -> int:
        return self.steps // self.restarts


@dataclass
class RidcSolution:
    final_state: np.ndarray
    level_finals: list
    wall_seconds: float
    trajectory: Optional[np.ndarray] = None
    trace: Optional[list] = None


def restart_partition(t_start: float, t_end: float, restarts: int, total_steps: int):
    """Uniform sub-intervals sharing one global dt (engine.py:103-118)."""
    if restarts < 1 or total_steps < 1:
        raise ConfigError("restarts and total_steps must be positive")
    if total_steps % restarts:
        raise ConfigError(
            f"total_steps ({total_steps}) must be divisible by restarts ({restarts})")
    per = total_steps // restarts
    dt = (t_end - t_start) / total_steps
    parts = []
    for r in range(restarts):
        ta = t_start + r * per * dt
        tb = t_end if r == restarts - 1 else t_start + (r + 1) * per * dt
        parts.append((ta, tb, per))
    return parts


def schedule(levels: int, steps_per_interval: int):
    """The device tick schedule: tick k runs level j on step k - startup_delay(j).

    Returns [(tick, [(level, target), ...]), ...] for one interval.  The top
    level finishes at tick steps + levels(levels-1)/2.
    """
    out = []
    ticks = steps_per_interval + startup_delay(levels - 1)
    for k in range(1, ticks + 1):
        act = [(j, k - startup_delay(j)) for j in range(levels)
               if 1 <= k - startup_delay(j) <= steps_per_interval]
        if act:
            out.append((k, act))
    return out


def _trace(cfg: RidcConfig):
    tr = []
    for _r in range(cfg.restarts):
        for _k, act in schedule(cfg.levels, cfg.steps_per_interval):
            for j, t in act:
                tr.append((len(tr), j, t))
    return tr


class Engine:
    """A prepared run context (``ridc_create``): rings, factors, CUDA graph.

    Setup is done once here (the analogue of ``_prepare``, engine.py:465-473);
    ``run`` / ``run_device`` then only march.
    """

    def __init__(self, ivp, config: RidcConfig, tick_only: bool = False, resident_segments: bool = False):
        self.ivp = as_descriptor(ivp)
        self.config = config
        self.problem = self.ivp.problem
        self.dt = (self.ivp.t_end - self.ivp.t_start) / config.steps
        self.weights = pack_weight_tables(config.levels, self.dt)
        D.require_cuda(config.device)
        flags = RECORD_TRAJECTORY if config.record_trajectory else 0
        if tick_only:
            flags |= TICK_ONLY
        if resident_segments:
            flags |= RESIDENT_SEGMENTS
        cp = self.problem.to_c()
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().ridc_create(
            ctypes.byref(cp), float(self.ivp.t_start), float(self.ivp.t_end), config.levels,
            config.steps, config.restarts, self.weights.ctypes.data, self.weights.shape[0],
            config.device, flags, ctypes.byref(h)))
        self._h = h
        _lib.check(_lib.lib().ridc_set_watchdog(self._h, float(config.watchdog_seconds)), self._h)

    @property
    def info(self) -> dict:
        inf = _lib.RidcInfo()
        _lib.check(_lib.lib().ridc_info_get(self._h, ctypes.byref(inf)), self._h)
        d = {f: getattr(inf, f) for f, _ in inf._fields_}
        d["path_name"] = _lib.PATH_NAMES.get(d["path"], "?")
        return d

    def run(self, y0=None) -> RidcSolution:
        """One full run from host memory (H2D, marching, D2H)."""
        n = self.problem.dimension
        y0 = self.ivp.initial_state if y0 is None else np.ascontiguousarray(y0, dtype=np.float64)
        if y0.shape != (n,):
            raise ConfigError(f"y0 must have shape ({n},)")
        final = np.empty(n)
        lf = np.empty((self.config.levels, n))
        traj = np.empty((self.config.steps + 1, n)) if self.config.record_trajectory else None
        wall = ctypes.c_double(0.0)
        _lib.check(_lib.lib().ridc_run(
            self._h, y0.ctypes.data, final.ctypes.data, lf.ctypes.data,
            None if traj is None else traj.ctypes.data, ctypes.byref(wall)), self._h)
        return RidcSolution(final_state=final, level_finals=[lf[j] for j in range(lf.shape[0])],
                            wall_seconds=wall.value, trajectory=traj,
                            trace=_trace(self.config) if self.config.trace else None)

    def run_device(self, y0_dev, out_dev) -> float:
        """March from a device-resident state into a device buffer; returns device seconds.

        Both tensors must be float64, contiguous, of the problem's dimension and
        on the engine's device (the C-ABI takes no lengths).  The library runs on
        its own stream, so the caller's current stream is synchronised first
        (y0 may still be in production there)."""
        t = D.torch()
        n = self.problem.dimension
        for name, x in (("y0", y0_dev), ("out", out_dev)):
            if not isinstance(x, t.Tensor) or x.dtype != t.float64 or not x.is_cuda:
                raise TypeError(f"{name} must be a float64 CUDA tensor")
            if x.device.index != self.config.device:
                raise ValueError(f"{name} is on cuda:{x.device.index}, the engine on cuda:{self.config.device}")
            if x.numel() != n or not x.is_contiguous():
                raise DimensionMismatch(f"{name} has length {x.numel()}, expected {n} (contiguous)")
        t.cuda.current_stream(y0_dev.device).synchronize()
        wall = ctypes.c_double(0.0)
        _lib.check(_lib.lib().ridc_run_device(self._h, y0_dev.data_ptr(), out_dev.data_ptr(),
                                              ctypes.byref(wall)), self._h)
        return wall.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().ridc_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_serial(ivp, config: RidcConfig, solver=None) -> RidcSolution:
    """Reference executor semantics (engine.py:476-494) on the device engine."""
    with Engine(ivp, config) as eng:
        return eng.run()


def pipeline_devices(config: RidcConfig):
    """GPUs the concurrent executor spreads the levels over: ``workers`` is the
    GPU count, capped by the visible devices; level j runs on
    GPU (device + j % g).  A single entry means one device."""
    t = D.torch()
    visible = t.cuda.device_count() if t.cuda.is_available() else 0
    g = max(1, min(config.workers, visible - config.device))
    return [config.device + (j % g) for j in range(config.levels)] if g > 1 else [config.device]


def run_pipelined(ivp, config: RidcConfig, solver=None) -> RidcSolution:
    """Concurrent executor semantics (engine.py:497-522); bitwise equal to run_serial.

    The reference's worker threads own levels round-robin (engine.py:447-456);
    here ``workers`` > 1 with that many GPUs visible places level j on GPU
    j % workers (distributed.ConcurrentPipeline: one host thread and stream
    per level, device-side flags, peer stores over NVLink; with one level per
    GPU each rank is one resident launch).  With one visible GPU, or when a
    trajectory is recorded, every level marches on ``config.device``.  Either
    way the states are bitwise those of run_serial (the tiling depends only on
    the problem and dt)."""
    devs = pipeline_devices(config)
    if len(set(devs)) > 1 and not config.record_trajectory:
        from .distributed import ConcurrentPipeline
        pipe = ConcurrentPipeline(ivp, config, devices=devs)
        try:
            final, finals = pipe.run()
            wall = pipe.device_seconds
        finally:
            pipe.close()
        return RidcSolution(final_state=final, level_finals=finals, wall_seconds=wall,
                            trace=_trace(config) if config.trace else None)
    with Engine(ivp, config) as eng:
        return eng.run()


# ---------------------------------------------------------------- single steps

@dataclass(frozen=True)
class LevelWindow:
    """Previous-level data at the stencil nodes, in weight order (engine.py:200-210).

    The reference's constructor ``LevelWindow(fs, fn, new_index, old_index)``
    (f^S / f^N rows of the previous level) works unchanged.  The device-path
    form :meth:`from_states` carries eta^{[j-1]} at the nodes instead; f^S and
    f^N are then recomputed from the states by the device stencils.
    """

    fs: Optional[np.ndarray]
    fn: Optional[np.ndarray]
    new_index: int
    old_index: int
    states: Optional[np.ndarray] = None

    @classmethod
    def from_states(cls, states, new_index: int, old_index: int) -> "LevelWindow":
        return cls(None, None, new_index, old_index, states)


def _resolve(ivp):
    return as_descriptor(ivp)


def _step_device(x) -> int:
    """The device a single step runs on: the input tensor's, else the current one."""
    t = D.torch()
    if isinstance(x, t.Tensor) and x.is_cuda:
        return x.device.index
    D.require_cuda()
    return t.cuda.current_device()


def predict_step(ivp, t_n: float, eta_n, dt: float, solver=None):
    """One predictor step -> (eta_new, f_stiff, f_nonstiff) at the new node (engine.py:193-197)."""
    pd = _resolve(ivp).problem
    if dt <= 0:
        raise ValueError(f"dt must be positive, got {dt}")
    dev = _step_device(eta_n)
    eta_new = ops.level_step(pd, dt, eta_n, dev=dev)
    return eta_new, ops.stiff_value(pd, eta_new, dev), ops.nonstiff_value(pd, eta_new, dev)


def correct_step(level: int, ivp, t_n: float, eta_n, prev_level_window, weights, dt: float,
                 solver=None):
    """One corrector step for level >= 1 (engine.py:213-231)."""
    if level < 1:
        raise ValueError("correct_step needs level >= 1")
    pd = _resolve(ivp).problem
    if dt <= 0:
        raise ValueError(f"dt must be positive, got {dt}")
    w = np.asarray(getattr(weights, "weights", weights), dtype=np.float64)
    win = prev_level_window
    i_new, i_old = win.new_index, win.old_index
    k = w.shape[0]
    if not (0 <= i_new < k and 0 <= i_old < k):
        raise PipelineProtocolError("window indices out of range")
    dev = _step_device(eta_n)
    if getattr(win, "states", None) is not None:
        states = np.asarray(win.states)
        if states.shape[0] != k:
            raise PipelineProtocolError(f"window holds {states.shape[0]} nodes, weights need {k}")
        cs = [w[a] - (dt if a == i_new else 0.0) for a in range(k)]
        cn = [w[a] - (dt if a == i_old else 0.0) for a in range(k)]
        eta_new = ops.level_step(pd, dt, eta_n, list(states), cs, cn, dev=dev)
    else:
        fs, fn = np.asarray(win.fs), np.asarray(win.fn)
        if fs.shape[0] != k or fn.shape[0] != k:
            raise PipelineProtocolError(f"window holds {fs.shape[0]} nodes, weights need {k}")
        eta_new = ops.level_step_rows(pd, dt, eta_n, fs, fn, w, i_new, i_old, dev=dev)
    return eta_new, ops.stiff_value(pd, eta_new, dev), ops.nonstiff_value(pd, eta_new, dev)
