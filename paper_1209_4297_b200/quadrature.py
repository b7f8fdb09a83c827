"""Deferred-correction quadrature weights (host precompute).

Mirrors the public surface of the reference's ``ridc.quadrature``
(pkg/src/ridc/quadrature.py:31-119): ``QuadratureWeights``,
``steady_weights``, ``startup_weights``, ``apply_quadrature``, ``MAX_LEVEL``.

The weights are exact rationals.  The reference integrates each Lagrange
basis polynomial term by term (quadrature.py:49-66); here the same rationals
are obtained by solving the moment equations  sum_k w_k x_k^m = int x^m,
m = 0..j, exactly over ``Fraction`` (the unique interpolatory rule on j+1
distinct nodes), then rounded to double and scaled by dt exactly as the
reference does (``float(frac) * dt``, quadrature.py:81, :97), so both give
bitwise-identical doubles.  The device kernels receive these doubles; they
never recompute them.
"""

from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache
from typing import Optional

import numpy as np

from .errors import DimensionMismatch

__all__ = ["MAX_LEVEL", "QuadratureWeights", "steady_weights", "startup_weights",
           "apply_quadrature", "pack_weight_tables", "weight_table_offsets"]

MAX_LEVEL = 11


@dataclass(frozen=True)
class QuadratureWeights:
    """j+1 integral weights for one correction level, each carrying dt."""

    level: int
    regime: str                 # "steady" | "startup"
    start_index: Optional[int]  # n for startup, None for steady
    dt: float
    weights: np.ndarray

    def __post_init__(self):
        if self.weights.shape != (self.level + 1,):
            raise ValueError("weight count must be level + 1")
        total = float(self.weights.sum())
        if abs(total - self.dt) > 1e-13 * abs(self.dt):
            raise ValueError(f"weights sum to {total!r}, expected dt={self.dt!r}")


def _moment_rule(nodes: tuple, lo: Fraction, hi: Fraction) -> list:
    """Exact interpolatory weights on ``nodes`` for the integral over [lo, hi]."""
    k = len(nodes)
    rows = [[Fraction(x) ** m for x in nodes] + [(hi ** (m + 1) - lo ** (m + 1)) / (m + 1)]
            for m in range(k)]
    # Gauss-Jordan over the rationals (Vandermonde is nonsingular on distinct nodes)
    for col in range(k):
        piv = next(r for r in range(col, k) if rows[r][col] != 0)
        rows[col], rows[piv] = rows[piv], rows[col]
        inv = 1 / rows[col][col]
        rows[col] = [v * inv for v in rows[col]]
        for r in range(k):
            if r != col and rows[r][col] != 0:
                f = rows[r][col]
                rows[r] = [a - f * b for a, b in zip(rows[r], rows[col])]
    return [rows[i][k] for i in range(k)]


def _check_level(j: int) -> None:
    if j < 1:
        raise ValueError("correction level must be >= 1 (the prediction level uses no quadrature)")
    if j > MAX_LEVEL:
        raise ValueError(f"correction level {j} exceeds the supported maximum {MAX_LEVEL}")


@lru_cache(maxsize=None)
def _steady_fracs(j: int) -> tuple:
    # node k sits at t_{n+1-k}; in units of dt relative to t_n: 1 - k
    return tuple(_moment_rule(tuple(Fraction(1 - k) for k in range(j + 1)), Fraction(0), Fraction(1)))


@lru_cache(maxsize=None)
def _startup_fracs(j: int, n: int) -> tuple:
    # node k sits at t_k; integrate over [t_n, t_{n+1}]
    return tuple(_moment_rule(tuple(Fraction(k) for k in range(j + 1)), Fraction(n), Fraction(n + 1)))


def _scaled(fracs, dt: float) -> np.ndarray:
    w = np.array([float(f) for f in fracs]) * dt
    w.setflags(write=False)
    return w


def steady_weights(j: int, dt: float) -> QuadratureWeights:
    """Trailing stencil; index k pairs with node t_{n+1-k} (quadrature.py:76-85)."""
    _check_level(j)
    if dt <= 0:
        raise ValueError("dt must be positive")
    return QuadratureWeights(j, "steady", None, dt, _scaled(_steady_fracs(j), dt))


def startup_weights(j: int, n: int, dt: float) -> QuadratureWeights:
    """Left-anchored stencil for step n -> n+1; index k pairs with t_k (quadrature.py:88-101)."""
    _check_level(j)
    if dt <= 0:
        raise ValueError("dt must be positive")
    if not 0 <= n < j - 1:
        raise ValueError(f"startup weights need 0 <= n < j-1, got n={n}, j={j}; use steady_weights")
    return QuadratureWeights(j, "startup", n, dt, _scaled(_startup_fracs(j, n), dt))


def apply_quadrature(w: QuadratureWeights, rhs_window) -> np.ndarray:
    """Weighted sum of a window of rhs vectors (quadrature.py:104-119)."""
    rows = np.asarray(rhs_window, dtype=np.float64)
    scalar = rows.ndim == 1
    if scalar:
        rows = rows[:, None]
    if rows.shape[0] != w.weights.shape[0]:
        raise DimensionMismatch(
            f"window has {rows.shape[0]} entries, weights need {w.weights.shape[0]}")
    out = w.weights @ rows
    return float(out[0]) if scalar else out


def weight_table_offsets(levels: int):
    """Offsets into the packed table: steady j=1..L-1, then startup (j,n), n<j-1.

    This packed layout is the one ``ridc_create`` (include/ridc_b200.h) and the
    CPU oracle both read.
    """
    steady, startup, off = {}, {}, 0
    for j in range(1, levels):
        steady[j] = off
        off += j + 1
    for j in range(2, levels):
        for n in range(j - 1):
            startup[(j, n)] = off
            off += j + 1
    return steady, startup, off


def pack_weight_tables(levels: int, dt: float) -> np.ndarray:
    """All weight tables of a run (engine.py:143-152), packed for the C-ABI."""
    steady, startup, total = weight_table_offsets(levels)
    out = np.zeros(max(total, 1), dtype=np.float64)
    for j, off in steady.items():
        out[off:off + j + 1] = steady_weights(j, dt).weights
    for (j, n), off in startup.items():
        out[off:off + j + 1] = startup_weights(j, n, dt).weights
    return out
