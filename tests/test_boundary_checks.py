"""Host-side argument checks of the drop-in boundary (no GPU needed: every
check fires before the first device call).  The C-ABI takes no lengths, so
the Python layer rejects mis-sized buffers the way the reference's
steppers._check_step_args does (steppers.py:107-111)."""

import numpy as np
import pytest

from paper_1209_4297_b200 import engine as E, ops, problems as P
from paper_1209_4297_b200.errors import DimensionMismatch, PipelineProtocolError


def _pd(n=64):
    return P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / n, t_end=1.0)).problem


def test_ops_reject_wrong_length():
    pd = _pd()
    with pytest.raises(DimensionMismatch):
        ops.level_step(pd, 0.01, np.ones(63))
    with pytest.raises(DimensionMismatch):
        ops.level_step(pd, 0.01, np.ones(64), [np.ones(64), np.ones(65)], [0.1, 0.1], [0.1, 0.1])
    with pytest.raises(DimensionMismatch):
        ops.solve_shifted(pd, 0.01, np.ones(10))
    with pytest.raises(DimensionMismatch):
        ops.stiff_value(pd, np.ones((2, 64)))
    with pytest.raises(DimensionMismatch):
        ops.level_step_rows(pd, 0.01, np.ones(64), [np.ones(64)] * 2, [np.ones(64)] * 3, [0.5, 0.5], 0, 1)


def test_predict_step_rejects_bad_dt():
    s = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 64, t_end=1.0))
    with pytest.raises(ValueError):
        E.predict_step(s, 0.0, s.ivp.initial_state, 0.0)


def test_level_window_reference_constructor():
    """LevelWindow(fs, fn, new_index, old_index) as engine.py:200-210."""
    fs, fn = np.zeros((3, 8)), np.ones((3, 8))
    w = E.LevelWindow(fs, fn, 0, 1)
    assert w.fs is fs and w.fn is fn and w.new_index == 0 and w.old_index == 1 and w.states is None
    w2 = E.LevelWindow.from_states(np.zeros((3, 8)), 0, 1)
    assert w2.fs is None and w2.states.shape == (3, 8)


def test_correct_step_window_index_checks():
    s = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 64, t_end=1.0))
    w = E.LevelWindow(np.zeros((3, 64)), np.zeros((3, 64)), 0, 5)
    with pytest.raises(PipelineProtocolError):
        E.correct_step(2, s, 0.0, s.ivp.initial_state, w, [0.1, 0.2, 0.3], 0.01)
