"""Parity at the north_star's own sizes (BASELINE.json configs[1..4], SURVEY.md
§8d C2-C5): the CUDA path against the CPU oracle (oracle/ridc_oracle.c, pinned
to the reference's golden vectors by tests/test_oracle_golden.py), final state
and every level's final, normwise max|gpu - oracle| / max|oracle| <= 1e-10.

Each case runs the workload's own grid and dt (the configuration's Nt sets
dt = T / Nt) for a bounded number of steps -- at least the pipeline fill plus
ten steps, so every level reaches its steady window -- except C2 FEBE, which
runs the bench's full Nt = 10^4.  The oracle runs one thread per level
(engine.py's workers), so the largest cases take tens of seconds of host time.
"""

import os

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

TOL = 1e-10


def _host_bytes_free():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 1 << 62


def _oracle_bytes(n, levels):
    # oracle rings: (j+2) x (state, fs, fn) for j < top, 6 vectors per level, + finals
    rings = sum(3 * (j + 2) for j in range(levels - 1))
    return 8 * n * (rings + 6 * levels + levels + 4)


def _shorten(system, nt_full, steps):
    """The workload's grid and dt, marched for `steps` of its Nt_full steps."""
    ivp = system.ivp
    t1 = ivp.t_start + (ivp.t_end - ivp.t_start) * steps / nt_full
    return P.StructuredIVP(ivp.problem, ivp.t_start, t1, ivp.initial_state)


def _check(ivp, levels, steps, restarts=1):
    n = ivp.problem.dimension
    need = _oracle_bytes(n, levels) + 8 * n * (levels + 4)
    if need > 0.8 * _host_bytes_free():
        pytest.skip(f"oracle needs {need / 2**30:.1f} GiB host memory")
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts)
    sol = E.run_serial(ivp, cfg)
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, levels, steps, restarts, dt, pack_weight_tables(levels, dt),
                workers=min(levels, max(1, os.cpu_count() or 1)), level_finals=True)
    errs = [G.normwise(sol.final_state, ref["final_state"])]
    errs += [G.normwise(sol.level_finals[j], ref["level_finals"][j]) for j in range(levels)]
    print(f"n={n} p={levels} steps={steps}: final {errs[0]:.3e}, levels {max(errs[1:]):.3e}")
    assert max(errs) <= TOL, errs
    return sol


def test_c2_febe_full_nt():
    """configs[1], the bench workload itself: N = 2^20, Nt = 10^4, FEBE."""
    _check(P.reaction_diffusion_c2().ivp, 1, 10000)


@pytest.mark.parametrize("levels", [2, 4])
def test_c2_orders(levels):
    """configs[1] at orders 2 and 4 (all levels on one GPU), 400 steps of dt = 1e-4."""
    _check(_shorten(P.reaction_diffusion_c2(), 10000, 400), levels, 400)


def test_c3_full_grid_p4():
    """configs[2]: 2-D adv-diff 4096 x 4096, RIDC order 4, C3's dt (T / 1000),
    fill (11 steps) + 10."""
    _check(_shorten(P.adv_diff_2d_c3(), 1000, 21), 4, 21)


def test_c3_full_grid_febe():
    _check(_shorten(P.adv_diff_2d_c3(), 1000, 21), 1, 21)


def test_c4_p8():
    """configs[3]: 2-D reaction-diffusion with 8192-point x-lines at RIDC order 8
    (1024 rows: the oracle's rings of the full 8192^2 grid exceed host memory),
    C4's spacing and dt, fill (37 steps) + 10."""
    spec = P.ReactionDiffusion2DSpec(nx=8192, ny=1024)
    full = P.ReactionDiffusion2DSpec()
    # keep C4's y-spacing h_y = 1/8192 (explicit y-diffusion) on fewer rows: the
    # same grid, a 1024-row periodic strip
    system = P.build_reaction_diffusion_2d(spec)
    pd = system.problem
    pd = P.ProblemDescriptor(pd.kind, pd.nx, pd.ny, pd.c_x, pd.c_y, pd.d_x, full.dyy, pd.rho,
                             1.0 / full.nx, 1.0 / full.ny)
    ivp = P.StructuredIVP(pd, 0.0, full.t_end * 47 / 1000, system.ivp.initial_state)
    _check(ivp, 8, 47)


def _c5(exp, steps):
    n = 1 << exp
    spec = P.ReactionDiffusionSpec(n=n, d=1e-6 * (float(1 << 20) / n) ** 2, t_end=1.0 * steps / 10000)
    return P.build_reaction_diffusion(spec).ivp


@pytest.mark.parametrize("exp", [22, 24, 26])
@pytest.mark.parametrize("levels", [1, 4])
def test_c5_sweep_sizes(exp, levels):
    """configs[4] grid sizes beyond C2 (tick kernel, segmented lines), r held at
    C2's ~110 as in tools/sweep.py; fill + 10 steps (p = 4) or 20 (FEBE)."""
    steps = 21 if levels == 4 else 20
    _check(_c5(exp, steps), levels, steps)
