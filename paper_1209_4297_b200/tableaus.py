"""Coupled implicit/explicit Butcher pairs of the ARK comparators.

Same objects as the reference's tableaus.py:27-127 (``ButcherPair``,
``imex3_tableau``, ``imex4_tableau``): exact rational coefficients evaluated
once to double precision, lower-triangular DIRK table for the stiff part and
strictly lower explicit table for the non-stiff part, row sums checked
against ``c`` to 1e-14 at construction.  The device consumes them through
``ridc_ark_create`` (include/ridc_b200.h).
"""

from dataclasses import dataclass
from fractions import Fraction as F

import numpy as np

from .errors import ConfigError

__all__ = ["ButcherPair", "imex3_tableau", "imex4_tableau"]

ROW_SUM_TOL = 1e-14


@dataclass(frozen=True)
class ButcherPair:
    """DIRK table + explicit table sharing the abscissae ``c`` (tableaus.py:27-66)."""

    c: np.ndarray
    a_implicit: np.ndarray
    a_explicit: np.ndarray
    b_implicit: np.ndarray
    b_explicit: np.ndarray
    strict: bool = True

    def __post_init__(self):
        s = self.c.shape[0]
        for name in ("a_implicit", "a_explicit"):
            if getattr(self, name).shape != (s, s):
                raise ConfigError(f"{name} must be {s}x{s}")
        for name in ("b_implicit", "b_explicit"):
            if getattr(self, name).shape != (s,):
                raise ConfigError(f"{name} must have {s} entries")
        if np.any(np.triu(self.a_implicit, 1) != 0.0):
            raise ConfigError("a_implicit must be lower triangular")
        if np.any(np.triu(self.a_explicit, 0) != 0.0):
            raise ConfigError("a_explicit must be strictly lower triangular")
        if self.strict:
            for name in ("a_implicit", "a_explicit"):
                dev = np.abs(getattr(self, name).sum(axis=1) - self.c).max()
                if dev > ROW_SUM_TOL:
                    raise ConfigError(f"{name} row sums deviate from c by {dev:.2e}")
        for arr in (self.c, self.a_implicit, self.a_explicit, self.b_implicit, self.b_explicit):
            arr.setflags(write=False)

    @property
    def stages(self) -> int:
        return int(self.c.shape[0])

    def shifts(self, dt: float) -> list:
        """Distinct nonzero solve coefficients a_ii * dt (studies.py:166-168)."""
        return sorted({float(a) * dt for a in np.diag(self.a_implicit) if a != 0.0})


def _dense(rows, s):
    out = np.zeros((s, s))
    for i, row in enumerate(rows):
        for j, v in enumerate(row):
            out[i, j] = float(v)
    return out


def _pair(c, a_imp, a_exp, b_imp, b_exp) -> ButcherPair:
    s = len(c)
    return ButcherPair(np.array([float(v) for v in c]), _dense(a_imp, s), _dense(a_exp, s),
                       np.array([float(v) for v in b_imp]), np.array([float(v) for v in b_exp]))


# (c, implicit rows, explicit rows, b implicit, b explicit) per scheme
_IMEX3 = (
    [0, F(1, 2), F(1, 2), 1, 1],
    [[0], [0, F(1, 2)], [F(1, 4), F(-5, 12), F(2, 3)], [2, F(-7, 2), F(1, 2), 2],
     [F(1, 6), 0, F(2, 3), F(-5, 6), 1]],
    [[], [F(1, 2)], [F(1, 4), F(1, 4)], [0, 1, 0], [F(1, 6), 0, F(2, 3), F(1, 6)]],
    [F(1, 6), 0, F(2, 3), F(-5, 6), 1],
    [F(1, 6), 0, F(2, 3), F(1, 6), 0],
)

_IMEX4 = (
    [0, F(1, 3), F(1, 3), F(1, 2), F(1, 2), 1, 1],
    [[0], [F(-1, 6), F(1, 2)], [F(1, 6), F(-1, 3), F(1, 2)], [F(3, 8), F(-3, 8), 0, F(1, 2)],
     [F(1, 8), 0, F(3, 8), F(-1, 2), F(1, 2)], [F(-1, 2), 0, 3, -3, 1, F(1, 2)],
     [F(1, 6), 0, 0, 0, F(2, 3), F(-1, 2), F(2, 3)]],
    [[], [F(1, 3)], [F(1, 6), F(1, 6)], [F(1, 8), 0, F(3, 8)], [F(1, 8), 0, F(3, 8), 0],
     [F(1, 2), 0, F(-3, 2), 0, 2], [F(1, 6), 0, 0, 0, F(2, 3), F(1, 6)]],
    [F(1, 6), 0, 0, 0, F(2, 3), F(-1, 2), F(2, 3)],
    [F(1, 6), 0, 0, 0, F(2, 3), F(1, 6), 0],
)


def imex3_tableau() -> ButcherPair:
    """Third-order pair, 5 stages (tableaus.py:82-101)."""
    return _pair(*_IMEX3)


def imex4_tableau() -> ButcherPair:
    """Fourth-order pair, 7 stages (tableaus.py:104-127)."""
    return _pair(*_IMEX4)
