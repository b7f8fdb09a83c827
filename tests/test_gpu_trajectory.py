"""Trajectory recording (RidcSolution.trajectory, engine.py:94-100, :506-521)
in both device modes: kept whole on the device, or streamed step by step to
pinned host memory through a copy stream with an 8-slot top ring (the mode
chosen when (steps+1) states do not fit comfortably, forced here with
RIDC_TRAJ_STREAM=1).  Both must agree bitwise, and with the reference's own
trajectory (golden ad_n128_p4_r2)."""

import os

import numpy as np
import pytest

import _golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402


def _run(ivp, cfg, stream):
    old = os.environ.get("RIDC_TRAJ_STREAM")
    os.environ["RIDC_TRAJ_STREAM"] = "1" if stream else "0"
    try:
        with E.Engine(ivp, cfg) as eng:
            return eng.run(), eng.info
    finally:
        if old is None:
            del os.environ["RIDC_TRAJ_STREAM"]
        else:
            os.environ["RIDC_TRAJ_STREAM"] = old


@pytest.mark.parametrize("levels,steps,restarts", [(1, 40, 1), (1, 60, 3), (3, 60, 2), (4, 120, 2)])
@pytest.mark.parametrize("n", [1000, 20000])
def test_streamed_trajectory_equals_device_trajectory(levels, steps, restarts, n):
    s = P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-4, t_end=0.01))
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, record_trajectory=True)
    a, ia = _run(s, cfg, stream=False)
    b, ib = _run(s, cfg, stream=True)
    assert ib["ring_vectors"] < ia["ring_vectors"]          # the top ring holds 8 slots, not steps + 1
    assert a.trajectory.shape == b.trajectory.shape == (steps + 1, n)
    if ia["path_name"] == ib["path_name"]:
        assert np.array_equal(a.trajectory, b.trajectory)
        assert np.array_equal(a.final_state, b.final_state)
    else:   # e.g. the carry-exchange march (device trajectory) vs the tick graph (streamed): same solve
        assert G.normwise(a.trajectory, b.trajectory) <= 1e-13
        assert G.normwise(a.final_state, b.final_state) <= 1e-13
    assert np.array_equal(b.trajectory[-1], b.final_state)
    assert np.array_equal(b.trajectory[0], s.ivp.initial_state)


def test_streamed_trajectory_matches_reference_golden():
    runs, arr = G.run_cases()
    case = next(c for c in runs if c["name"] == "ad_n128_p4_r2")
    ivp = P.StructuredIVP(G.descriptor(case["problem"]), 0.0, case["t_end"], arr[case["name"] + "/y0"])
    cfg = E.RidcConfig(levels=case["levels"], steps=case["steps"], restarts=case["restarts"],
                       record_trajectory=True)
    sol, _ = _run(ivp, cfg, stream=True)
    assert G.normwise(sol.trajectory, arr[case["name"] + "/trajectory"]) <= 1e-10
