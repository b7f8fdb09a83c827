"""Edge cases of the device path against the oracle (the reference's algebra):
ragged and minimum grids (nx = 3, non-multiples of 16, one past a chunk /
whole-line / segment boundary), the maximum level count (12) at the
pipeline-fill minimum step count, restarts at their limit, 2-D with ny = 3,
the stiffness limit of the segmented solve, and the resident whole-line march
at its size limit.  Bar: normwise 1e-10."""

import numpy as np
import pytest

import _golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402
from paper_1209_4297_b200.errors import ConfigError  # noqa: E402
from paper_1209_4297_b200.quadrature import pack_weight_tables  # noqa: E402

TOL = 1e-10


def _rd(n, d, t_end, seed=0):
    s = P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=d, t_end=t_end, seed=seed))
    return s.ivp


def _ad(n, t_end):
    pd = P.ProblemDescriptor(P.KIND_ADV_DIFF_1D, nx=n, c_x=0.1, d_x=1e-3, h_x=1.0 / n)
    x = np.arange(n) / n
    return P.StructuredIVP(pd, 0.0, t_end, 2.0 + np.sin(2 * np.pi * x))


def _bu(n, t_end):
    pd = P.ProblemDescriptor(P.KIND_BURGERS_1D, nx=n, d_x=1e-3, h_x=1.0 / (n + 1))
    x = np.arange(1, n + 1) / (n + 1)
    return P.StructuredIVP(pd, 0.0, t_end, np.sin(np.pi * x) + 0.5 * np.sin(2 * np.pi * x))


def _check(ivp, levels, steps, restarts=1):
    sol = E.run_serial(ivp, E.RidcConfig(levels=levels, steps=steps, restarts=restarts))
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, levels, steps, restarts, dt, pack_weight_tables(levels, dt),
                level_finals=True)
    assert G.normwise(sol.final_state, ref["final_state"]) <= TOL
    for j in range(levels):
        assert G.normwise(sol.level_finals[j], ref["level_finals"][j]) <= TOL
    return sol


@pytest.mark.parametrize("n", [3, 5, 17, 31, 1000, 1023, 1025, 4095, 4097, 8191, 8192, 8193, 8209, 100003])
@pytest.mark.parametrize("levels", [1, 3])
def test_ragged_sizes_rd(n, levels):
    _check(_rd(n, 1e-3, 0.01), levels, 12)


@pytest.mark.parametrize("n", [3, 16, 33, 8190, 8195, 20001])
def test_ragged_sizes_adv_and_burgers(n):
    _check(_ad(n, 0.02), 2, 10)
    _check(_bu(n, 0.002), 2, 10)


def test_max_levels_at_fill_minimum():
    """12 levels need >= startup_delay(12) + 1 = 79 steps per interval (engine.py:81-87)."""
    ivp = _ad(256, 0.5)
    _check(ivp, 12, 79)
    _check(ivp, 12, 158, restarts=2)
    with pytest.raises(ConfigError):
        E.run_serial(ivp, E.RidcConfig(levels=12, steps=78))


def test_2d_minimum_rows_and_ragged_columns():
    for nx, ny in ((3, 3), (17, 3), (4097, 3), (9001, 5)):
        pd = P.ProblemDescriptor(P.KIND_ADV_DIFF_2D, nx=nx, ny=ny, c_x=0.1, c_y=0.1, d_x=1e-3, d_y=1e-4,
                                 h_x=1.0 / nx, h_y=1.0 / ny)
        y0 = 2.0 + np.random.default_rng(nx).uniform(-0.1, 0.1, nx * ny)
        _check(P.StructuredIVP(pd, 0.0, 0.01, y0), 3, 8)


def test_stiffness_limit_of_segmented_solve():
    """Very stiff long lines need a truncation halo wider than an item: ConfigError,
    never a wrong answer; the same stiffness on a whole line is exact."""
    with pytest.raises(ConfigError):
        E.run_serial(_rd(1 << 16, 1.0, 1.0), E.RidcConfig(levels=1, steps=2))
    _check(_rd(4096, 1.0, 0.5), 2, 4)          # r ~ 4e6 on a whole line


def test_resident_whole_line_limit():
    """8192 points: the largest whole line, marched by one resident CTA."""
    ivp = _rd(8192, 1e-4, 0.05)
    with E.Engine(ivp, E.RidcConfig(levels=1, steps=50)) as eng:
        assert eng.info["kernel_launches"] == 2 and eng.info["items_per_level"] == 1
    _check(ivp, 1, 50)
