"""Method-of-lines problems as structured descriptors for the device path.

Mirrors the reference's ``ridc.problems`` (pkg/src/ridc/problems.py):
``AdvectionDiffusionSpec`` / ``BurgersSpec`` / ``build_advection_diffusion``
/ ``build_burgers`` / presets / ``error_norms``, and adds the problem kinds the
north-star configurations name (1-D and 2-D reaction-diffusion, 2-D
advection-diffusion, SURVEY.md §7 hard part 5).

The reference's ``SplitIVP`` carries opaque Python callables and a dense
(n, n) stiff operator (ivp.py:31-66), which cannot run on a device and is
infeasible beyond n ~ 4096.  Here every system carries a ``ProblemDescriptor``
(kind enum + stencil coefficients + grid) that crosses the C-ABI
(include/ridc_b200.h, ``ridc_problem``); the operators are the stencils the
reference's dense matrices encode:

* adv-diff 1-D periodic (problems.py:109-138): f^N = c/dx (u_{i+1} - u_i),
  f^S = d/dx^2 (u_{i-1} - 2u_i + u_{i+1}); u0 = 2 + sin(2 pi x), x_i = i dx.
* Burgers 1-D Dirichlet (problems.py:141-168, kernels.py:160-168):
  f^N = -(u_{i+1}^2 - u_{i-1}^2)/(4dx) with zero ghosts, f^S = eps D.
* reaction-diffusion 1-D periodic (new): f^N = rho u (1-u), f^S = d D.
* adv-diff 2-D periodic (new): f^S = I (x) D_xx (x-line diffusion, implicit);
  f^N = upwind advection in x and y + y-diffusion (explicit).
* reaction-diffusion 2-D periodic (new): f^S = x-line diffusion;
  f^N = rho u (1-u) + y-diffusion.

2-D states are flattened row-major: index = row * nx + col (x fastest), so
every implicit x-line is contiguous in HBM.
"""

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .errors import ConfigError, DimensionMismatch

__all__ = [
    "KIND_ADV_DIFF_1D", "KIND_BURGERS_1D", "KIND_REACTION_DIFFUSION_1D",
    "KIND_ADV_DIFF_2D", "KIND_REACTION_DIFFUSION_2D",
    "ProblemDescriptor", "StructuredIVP",
    "AdvectionDiffusionSpec", "BurgersSpec", "ReactionDiffusionSpec",
    "AdvectionDiffusion2DSpec", "ReactionDiffusion2DSpec",
    "AdvectionDiffusionSystem", "BurgersSystem", "ReactionDiffusionSystem",
    "AdvectionDiffusion2DSystem", "ReactionDiffusion2DSystem",
    "build_advection_diffusion", "build_burgers", "build_reaction_diffusion",
    "build_advection_diffusion_2d", "build_reaction_diffusion_2d",
    "build_system", "error_norms", "exact_advection_diffusion",
    "adv_diff_desk", "adv_diff_paper", "burgers_desk", "burgers_paper",
    "reaction_diffusion_c2", "adv_diff_2d_c3", "reaction_diffusion_2d_c4",
    "as_descriptor",
]

KIND_ADV_DIFF_1D = 1
KIND_BURGERS_1D = 2
KIND_REACTION_DIFFUSION_1D = 3
KIND_ADV_DIFF_2D = 4
KIND_REACTION_DIFFUSION_2D = 5

_KIND_NAMES = {
    KIND_ADV_DIFF_1D: "adv-diff",
    KIND_BURGERS_1D: "burgers",
    KIND_REACTION_DIFFUSION_1D: "reaction-diffusion",
    KIND_ADV_DIFF_2D: "adv-diff-2d",
    KIND_REACTION_DIFFUSION_2D: "reaction-diffusion-2d",
}


class CProblem(ctypes.Structure):
    """ABI mirror of ``ridc_problem`` (include/ridc_b200.h)."""

    _fields_ = [
        ("kind", ctypes.c_int32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("c_x", ctypes.c_double), ("c_y", ctypes.c_double),
        ("d_x", ctypes.c_double), ("d_y", ctypes.c_double),
        ("rho", ctypes.c_double), ("h_x", ctypes.c_double), ("h_y", ctypes.c_double),
    ]


@dataclass(frozen=True)
class ProblemDescriptor:
    """Kind enum + stencil coefficients + grid: everything the device needs."""

    kind: int
    nx: int
    ny: int = 1
    c_x: float = 0.0
    c_y: float = 0.0
    d_x: float = 0.0
    d_y: float = 0.0
    rho: float = 0.0
    h_x: float = 1.0
    h_y: float = 1.0

    def __post_init__(self):
        if self.kind not in _KIND_NAMES:
            raise ConfigError(f"unknown problem kind {self.kind}")
        if self.nx < 3 or self.ny < 1:
            raise ConfigError(f"grid {self.ny}x{self.nx} too small (need nx >= 3)")
        if self.kind in (KIND_ADV_DIFF_2D, KIND_REACTION_DIFFUSION_2D) and self.ny < 3:
            raise ConfigError("2-D problems need ny >= 3")
        if self.kind not in (KIND_ADV_DIFF_2D, KIND_REACTION_DIFFUSION_2D) and self.ny != 1:
            raise ConfigError("1-D problems have ny == 1")
        if not self.d_x > 0:
            raise ConfigError("the stiff x-diffusivity must be positive")

    @property
    def dimension(self) -> int:
        return self.nx * self.ny

    @property
    def name(self) -> str:
        return _KIND_NAMES[self.kind]

    @property
    def is_2d(self) -> bool:
        return self.ny > 1 or self.kind in (KIND_ADV_DIFF_2D, KIND_REACTION_DIFFUSION_2D)

    def stiffness(self, dt: float) -> float:
        """r = dt * d_x / h_x^2, the off-diagonal magnitude of (I - dt D)."""
        return dt * self.d_x / (self.h_x * self.h_x)

    def to_c(self) -> CProblem:
        return CProblem(self.kind, self.nx, self.ny, 0, self.c_x, self.c_y, self.d_x,
                        self.d_y, self.rho, self.h_x, self.h_y)


@dataclass(frozen=True)
class StructuredIVP:
    """The device-path analogue of ``SplitIVP`` (ivp.py:31-66).

    ``eval_nonstiff`` / ``eval_stiff`` run the device stencils through the
    C-ABI (``ridc_op_apply``); there is no host implementation.
    ``stiff_linear_operator`` is None: the operator is structured, never dense.
    """

    problem: ProblemDescriptor
    t_start: float
    t_end: float
    initial_state: np.ndarray
    stiff_linear_operator: None = None

    def __post_init__(self):
        if not self.t_start < self.t_end:
            raise ValueError(f"need t_start < t_end, got [{self.t_start}, {self.t_end}]")
        y0 = np.ascontiguousarray(self.initial_state, dtype=np.float64).reshape(-1)
        if y0.shape[0] != self.problem.dimension:
            raise DimensionMismatch(
                f"state has length {y0.shape[0]}, expected {self.problem.dimension}")
        if not np.isfinite(y0).all():
            raise ValueError("state contains NaN or Inf entries")
        y0.setflags(write=False)
        object.__setattr__(self, "initial_state", y0)

    @property
    def dimension(self) -> int:
        return self.problem.dimension

    def eval_nonstiff(self, t: float, y) -> np.ndarray:
        from . import ops
        return ops.nonstiff_value(self.problem, y)

    def eval_stiff(self, t: float, y) -> np.ndarray:
        from . import ops
        return ops.stiff_value(self.problem, y)


def _grid_count(dx: float) -> int:
    """problems.py:46-50: dx must evenly divide the unit interval."""
    m = round(1.0 / dx)
    if m < 3 or abs(m * dx - 1.0) > 1e-12:
        raise ConfigError(f"dx={dx} must evenly divide the unit interval")
    return m


# ----------------------------------------------------------------- 1-D specs

@dataclass(frozen=True)
class AdvectionDiffusionSpec:
    """problems.py:53-63 (same fields and defaults)."""

    c: float = 0.1
    d: float = 1e-3
    dx: float = 1e-3
    t_end: float = 40.0

    def __post_init__(self):
        if self.c <= 0 or self.d <= 0:
            raise ConfigError("advection speed and diffusivity must be positive")
        _grid_count(self.dx)


@dataclass(frozen=True)
class BurgersSpec:
    """problems.py:66-75."""

    eps: float = 1e-3
    dx: float = 1e-3
    t_end: float = 1.0

    def __post_init__(self):
        if self.eps <= 0:
            raise ConfigError("viscosity must be positive")
        _grid_count(self.dx)


@dataclass(frozen=True)
class ReactionDiffusionSpec:
    """1-D periodic logistic reaction-diffusion on [0, 1): u_t = d u_xx + rho u(1-u).

    u0 = 0.5 + amplitude sin(2 pi x) + U(-noise, noise) from
    ``np.random.default_rng(seed)``.
    """

    d: float = 1e-6
    rho: float = 1.0
    n: int = 1 << 20
    t_end: float = 1.0
    amplitude: float = 0.25
    noise: float = 1e-3
    seed: int = 0

    def __post_init__(self):
        if self.d <= 0:
            raise ConfigError("diffusivity must be positive")
        if self.n < 3:
            raise ConfigError("need at least 3 grid points")


@dataclass(frozen=True)
class AdvectionDiffusion2DSpec:
    """2-D periodic advection-diffusion on [0,1)^2, x-line implicit diffusion.

    u_t = cx u_x + cy u_y + dxx u_xx + dyy u_yy, upwind forward differences
    for the advection as in the 1-D reference; u0 = 2 + sin(2 pi x) sin(2 pi y).
    Explicit y-diffusion: stable for dyy dt ny^2 <= 1/2.
    """

    cx: float = 0.1
    cy: float = 0.1
    dxx: float = 1e-2
    dyy: float = 1e-3
    nx: int = 4096
    ny: int = 4096
    t_end: float = 0.02

    def __post_init__(self):
        if self.dxx <= 0 or self.dyy < 0 or self.cx < 0 or self.cy < 0:
            raise ConfigError("need dxx > 0 and non-negative cx, cy, dyy")


@dataclass(frozen=True)
class ReactionDiffusion2DSpec:
    """2-D periodic logistic reaction-diffusion, x-line implicit diffusion."""

    dxx: float = 1e-3
    dyy: float = 1e-4
    rho: float = 1.0
    nx: int = 8192
    ny: int = 8192
    t_end: float = 0.05
    amplitude: float = 0.25
    noise: float = 1e-3
    seed: int = 0

    def __post_init__(self):
        if self.dxx <= 0 or self.dyy < 0:
            raise ConfigError("need dxx > 0 and dyy >= 0")


# ----------------------------------------------------------------- systems

@dataclass(frozen=True)
class _System:
    spec: object
    ivp: StructuredIVP

    @property
    def problem(self) -> ProblemDescriptor:
        return self.ivp.problem

    @property
    def name(self) -> str:
        return self.problem.name

    @property
    def dx(self) -> float:
        return self.problem.h_x


class AdvectionDiffusionSystem(_System):
    pass


class BurgersSystem(_System):
    pass


class ReactionDiffusionSystem(_System):
    pass


class AdvectionDiffusion2DSystem(_System):
    pass


class ReactionDiffusion2DSystem(_System):
    pass


def build_advection_diffusion(spec: AdvectionDiffusionSpec) -> AdvectionDiffusionSystem:
    """problems.py:109-138: periodic grid of M = 1/dx unknowns at x_i = i dx."""
    m = _grid_count(spec.dx)
    x = np.arange(m) * spec.dx
    u0 = 2.0 + np.sin(2.0 * np.pi * x)
    pd = ProblemDescriptor(KIND_ADV_DIFF_1D, nx=m, c_x=spec.c, d_x=spec.d, h_x=spec.dx)
    return AdvectionDiffusionSystem(spec, StructuredIVP(pd, 0.0, spec.t_end, u0))


def build_burgers(spec: BurgersSpec) -> BurgersSystem:
    """problems.py:141-168: interior unknowns u_1..u_{M-1}, zero Dirichlet ghosts."""
    m = _grid_count(spec.dx)
    n = m - 1
    x = (np.arange(n) + 1) * spec.dx
    u0 = np.sin(2.0 * np.pi * x) + 0.5 * np.sin(np.pi * x)
    pd = ProblemDescriptor(KIND_BURGERS_1D, nx=n, d_x=spec.eps, h_x=spec.dx)
    return BurgersSystem(spec, StructuredIVP(pd, 0.0, spec.t_end, u0))


def _rd_initial(n: int, amplitude: float, noise: float, seed: int, shape=None):
    rng = np.random.default_rng(seed)
    if shape is None:
        x = np.arange(n) / n
        base = 0.5 + amplitude * np.sin(2.0 * np.pi * x)
        return base + rng.uniform(-noise, noise, n)
    ny, nx = shape
    x = np.arange(nx) / nx
    y = np.arange(ny) / ny
    base = 0.5 + amplitude * np.outer(np.sin(2.0 * np.pi * y), np.sin(2.0 * np.pi * x))
    return (base + rng.uniform(-noise, noise, (ny, nx))).reshape(-1)


def build_reaction_diffusion(spec: ReactionDiffusionSpec) -> ReactionDiffusionSystem:
    h = 1.0 / spec.n
    u0 = _rd_initial(spec.n, spec.amplitude, spec.noise, spec.seed)
    pd = ProblemDescriptor(KIND_REACTION_DIFFUSION_1D, nx=spec.n, d_x=spec.d, rho=spec.rho, h_x=h)
    return ReactionDiffusionSystem(spec, StructuredIVP(pd, 0.0, spec.t_end, u0))


def build_advection_diffusion_2d(spec: AdvectionDiffusion2DSpec) -> AdvectionDiffusion2DSystem:
    hx, hy = 1.0 / spec.nx, 1.0 / spec.ny
    x = np.arange(spec.nx) * hx
    y = np.arange(spec.ny) * hy
    u0 = (2.0 + np.outer(np.sin(2.0 * np.pi * y), np.sin(2.0 * np.pi * x))).reshape(-1)
    pd = ProblemDescriptor(KIND_ADV_DIFF_2D, nx=spec.nx, ny=spec.ny, c_x=spec.cx, c_y=spec.cy,
                           d_x=spec.dxx, d_y=spec.dyy, h_x=hx, h_y=hy)
    return AdvectionDiffusion2DSystem(spec, StructuredIVP(pd, 0.0, spec.t_end, u0))


def build_reaction_diffusion_2d(spec: ReactionDiffusion2DSpec) -> ReactionDiffusion2DSystem:
    hx, hy = 1.0 / spec.nx, 1.0 / spec.ny
    u0 = _rd_initial(spec.nx * spec.ny, spec.amplitude, spec.noise, spec.seed,
                     shape=(spec.ny, spec.nx))
    pd = ProblemDescriptor(KIND_REACTION_DIFFUSION_2D, nx=spec.nx, ny=spec.ny, d_x=spec.dxx,
                           d_y=spec.dyy, rho=spec.rho, h_x=hx, h_y=hy)
    return ReactionDiffusion2DSystem(spec, StructuredIVP(pd, 0.0, spec.t_end, u0))


def build_system(spec):
    """Dispatch on the spec type (also accepts the reference's own spec objects)."""
    name = type(spec).__name__
    if name == "AdvectionDiffusionSpec":
        return build_advection_diffusion(AdvectionDiffusionSpec(spec.c, spec.d, spec.dx, spec.t_end))
    if name == "BurgersSpec":
        return build_burgers(BurgersSpec(spec.eps, spec.dx, spec.t_end))
    if isinstance(spec, ReactionDiffusionSpec):
        return build_reaction_diffusion(spec)
    if isinstance(spec, AdvectionDiffusion2DSpec):
        return build_advection_diffusion_2d(spec)
    if isinstance(spec, ReactionDiffusion2DSpec):
        return build_reaction_diffusion_2d(spec)
    raise ConfigError(f"unsupported problem spec {name}")


def as_descriptor(obj):
    """Resolve (descriptor, t_start, t_end, y0) from anything run_* accepts.

    Accepts a StructuredIVP, one of our systems, or a reference system object
    (``ridc.problems.AdvectionDiffusionSystem`` / ``BurgersSystem``, converted
    through its ``spec``).  A bare reference ``SplitIVP`` with opaque
    callables cannot run on the device and is rejected with ``ConfigError``
    (SURVEY.md §8b): there is no CPU fallback.
    """
    if isinstance(obj, StructuredIVP):
        return obj
    if isinstance(obj, _System):
        return obj.ivp
    spec = getattr(obj, "spec", None)
    if spec is not None:
        sys_ = build_system(spec)
        ivp = getattr(obj, "ivp", None)
        if ivp is not None and getattr(ivp, "initial_state", None) is not None:
            y0 = np.asarray(ivp.initial_state, dtype=np.float64)
            if y0.shape == sys_.ivp.initial_state.shape:
                return StructuredIVP(sys_.problem, float(ivp.t_start), float(ivp.t_end), y0)
        return sys_.ivp
    raise ConfigError(
        "the device engine needs a structured problem (our build_* systems or a reference "
        "system with a .spec); an opaque-callable SplitIVP cannot run on the GPU")


# ----------------------------------------------------------------- presets

def adv_diff_desk() -> AdvectionDiffusionSystem:
    """problems.py:199-200."""
    return build_advection_diffusion(AdvectionDiffusionSpec(dx=1.0 / 200, t_end=4.0))


def adv_diff_paper() -> AdvectionDiffusionSystem:
    """problems.py:203-204."""
    return build_advection_diffusion(AdvectionDiffusionSpec())


def burgers_desk() -> BurgersSystem:
    """problems.py:207-208."""
    return build_burgers(BurgersSpec(dx=1.0 / 500))


def burgers_paper() -> BurgersSystem:
    """problems.py:211-212."""
    return build_burgers(BurgersSpec())


def reaction_diffusion_c2(n: int = 1 << 20) -> ReactionDiffusionSystem:
    """BASELINE.json configs[1]: 1-D reaction-diffusion, N = 2^20 (T=1, Nt=1e4 -> r ~ 110)."""
    return build_reaction_diffusion(ReactionDiffusionSpec(n=n))


def adv_diff_2d_c3(n: int = 4096) -> AdvectionDiffusion2DSystem:
    """BASELINE.json configs[2]: 2-D advection-diffusion 4096^2."""
    return build_advection_diffusion_2d(AdvectionDiffusion2DSpec(nx=n, ny=n))


def reaction_diffusion_2d_c4(n: int = 8192) -> ReactionDiffusion2DSystem:
    """BASELINE.json configs[3]: 2-D reaction-diffusion 8192^2."""
    return build_reaction_diffusion_2d(ReactionDiffusion2DSpec(nx=n, ny=n))


# ----------------------------------------------------------------- norms / oracles

def error_norms(u: np.ndarray, ref: np.ndarray, dx: float) -> tuple:
    """(max norm, dx-weighted discrete 2-norm) of u - ref (problems.py:188-193)."""
    diff = np.asarray(u) - np.asarray(ref)
    return float(np.abs(diff).max()), float(np.sqrt(dx * np.dot(diff, diff)))


def exact_advection_diffusion(spec: AdvectionDiffusionSpec, t: float) -> np.ndarray:
    """Closed-form semi-discrete solution of the periodic 1-D problem.

    u(t) = 2 + Im(exp(lambda t) exp(2 pi i x)) with
    lambda = (c/dx)(e^{2 pi i dx} - 1) + (2d/dx^2)(cos(2 pi dx) - 1)
    (the circulant eigenvalue of A + D on the sin(2 pi x) mode).
    """
    m = _grid_count(spec.dx)
    x = np.arange(m) * spec.dx
    th = 2.0 * np.pi * spec.dx
    lam = (spec.c / spec.dx) * (np.exp(1j * th) - 1.0) + (2.0 * spec.d / spec.dx ** 2) * (math.cos(th) - 1.0)
    return 2.0 + np.imag(np.exp(lam * t) * np.exp(2j * np.pi * x))


def reference_solution(problem, t_end: float, refinement: int, base_steps: int, solver=None) -> np.ndarray:
    """Error baseline (problems.py:171-185): the same semi-discrete system marched
    with the fourth-order ARK pair at ``refinement`` x the finest study step count,
    on the device (steppers.integrate_ark)."""
    from .steppers import integrate_ark
    from .tableaus import imex4_tableau
    if refinement < 8:
        raise ConfigError(f"refinement must be >= 8, got {refinement}")
    if base_steps < 1:
        raise ConfigError("base_steps must be positive")
    ivp = as_descriptor(problem)
    return integrate_ark(ivp, imex4_tableau(), ivp.t_start, np.array(ivp.initial_state), t_end,
                         refinement * base_steps)

