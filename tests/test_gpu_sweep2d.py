"""The 2-D streaming FEBE sweep (csrc/ridc_sweep2d.cuh): every CTA sweeps a
block of rows, each row of the previous state read once, the completed
right-hand side of the row above solved as a cyclic x-line.  Against the tick
kernel (<= 1e-13: the same solve, different association), the CPU oracle
(<= 1e-10) and itself (bitwise across repeated runs)."""

import numpy as np
import pytest

import _golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402
from paper_1209_4297_b200.quadrature import pack_weight_tables  # noqa: E402


def _ad(nx, ny, steps, t_full=0.02, nt_full=1000):
    s = P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=nx, ny=ny, t_end=t_full * steps / nt_full))
    return s.ivp


def _rd(nx, ny, steps, t_full=0.05, nt_full=1000):
    s = P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=nx, ny=ny, t_end=t_full * steps / nt_full))
    return s.ivp


CASES = [
    # (id, ivp builder, steps, restarts, trajectory)
    ("ad-4096x700", lambda: _ad(4096, 700, 12), 12, 1, False),
    ("rd-8192x400", lambda: _rd(8192, 400, 10), 10, 1, False),
    ("ad-2048x1300-restarts", lambda: _ad(2048, 1300, 12), 12, 3, False),
    ("rd-4096x600-traj", lambda: _rd(4096, 600, 8), 8, 2, True),
]


@pytest.mark.parametrize("name,builder,steps,restarts,traj", CASES, ids=[c[0] for c in CASES])
def test_sweep2d_matches_tick_and_oracle(name, builder, steps, restarts, traj):
    ivp = builder()
    cfg = E.RidcConfig(levels=1, steps=steps, restarts=restarts, record_trajectory=traj)
    with E.Engine(ivp, cfg) as sw, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert sw.info["path_name"] == "sweep2d_febe", sw.info
        a, b = sw.run(), tick.run()
        a2 = sw.run()
    assert np.array_equal(a.final_state, a2.final_state)
    assert G.normwise(a.final_state, b.final_state) <= 1e-13
    if traj:
        assert G.normwise(a.trajectory, b.trajectory) <= 1e-13
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, 1, steps, restarts, dt, pack_weight_tables(1, dt))
    assert G.normwise(a.final_state, ref["final_state"]) <= 1e-10


def test_sweep2d_nonfinite_step():
    """A blow-up is reported at the step it happens (engine.py:160-164)."""
    s = P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=4096, ny=600, t_end=0.05 * 8 / 1000))
    y0 = np.array(s.ivp.initial_state)
    y0[123 * 4096 + 77] = np.inf
    ivp = P.StructuredIVP(s.ivp.problem, s.ivp.t_start, s.ivp.t_end, np.zeros_like(y0))
    with E.Engine(ivp, E.RidcConfig(levels=1, steps=8)) as eng:
        assert eng.info["path_name"] == "sweep2d_febe"
        with pytest.raises(Exception) as ei:
            eng.run(y0)
    assert "non-finite entries at step 1" in str(ei.value)


LEVEL_CASES = [
    # (id, ivp builder, levels, steps, restarts, trajectory)
    ("ad-4096x500-p2", lambda: _ad(4096, 500, 12), 2, 12, 1, False),
    ("ad-4096x400-p4-r2", lambda: _ad(4096, 400, 24), 4, 24, 2, False),
    ("rd-8192x320-p3", lambda: _rd(8192, 320, 10), 3, 10, 1, False),
    ("rd-4096x300-p4-traj", lambda: _rd(4096, 300, 12), 4, 12, 1, True),
]


@pytest.mark.parametrize("name,builder,levels,steps,restarts,traj", LEVEL_CASES, ids=[c[0] for c in LEVEL_CASES])
def test_sweep2d_levels_match_tick_and_oracle(name, builder, levels, steps, restarts, traj):
    """RIDC orders >= 2 on 2-D grids: one row sweep per active level per tick
    (csrc/ridc_sweep2d_levels.cuh), every level's final against the tick kernel
    and the oracle."""
    ivp = builder()
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, record_trajectory=traj)
    with E.Engine(ivp, cfg) as sw, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert sw.info["path_name"] == "sweep2d_levels", sw.info
        a, b = sw.run(), tick.run()
        a2 = sw.run()
    assert np.array_equal(a.final_state, a2.final_state)
    assert G.normwise(a.final_state, b.final_state) <= 1e-12
    for j in range(levels):
        assert G.normwise(a.level_finals[j], b.level_finals[j]) <= 1e-12, j
    if traj:
        assert G.normwise(a.trajectory, b.trajectory) <= 1e-12
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, levels, steps, restarts, dt, pack_weight_tables(levels, dt),
                level_finals=True)
    assert G.normwise(a.final_state, ref["final_state"]) <= 1e-10
    for j in range(levels):
        assert G.normwise(a.level_finals[j], ref["level_finals"][j]) <= 1e-10, j
