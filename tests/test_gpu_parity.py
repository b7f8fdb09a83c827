"""GPU parity: the device engine vs the reference's own outputs (golden
vectors) and vs the CPU oracle, through the C-ABI.  Bar: normwise relative
error <= 1e-10 (north_star / SURVEY.md §8c); bitwise determinism across
executors and repeated runs (engine.py:497-503)."""

import numpy as np
import pytest

import _golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1209_4297_b200 import engine as E, ops, problems as P  # noqa: E402
from paper_1209_4297_b200.errors import NonFiniteStateError  # noqa: E402
from paper_1209_4297_b200.quadrature import pack_weight_tables, steady_weights  # noqa: E402

TOL = 1e-10
RUNS, ARR = G.run_cases()


def _ivp(case):
    pd = G.descriptor(case["problem"])
    return P.StructuredIVP(pd, 0.0, case["t_end"], ARR[case["name"] + "/y0"])


def _oracle(ivp, levels, steps, restarts=1, **kw):
    dt = (ivp.t_end - ivp.t_start) / steps
    return O.run(ivp.problem, ivp.initial_state, levels, steps, restarts, dt,
                 pack_weight_tables(levels, dt), **kw)


@pytest.mark.parametrize("case", RUNS, ids=[c["name"] for c in RUNS])
def test_engine_matches_reference_golden(case):
    ivp = _ivp(case)
    cfg = E.RidcConfig(levels=case["levels"], steps=case["steps"], restarts=case["restarts"],
                       record_trajectory=case["trajectory"])
    sol = E.run_serial(ivp, cfg)
    name = case["name"]
    tol = G.tolerance(case["levels"])
    err = G.normwise(sol.final_state, ARR[name + "/final"])
    print(f"{name}: engine vs reference {err:.3e}")
    assert err <= tol
    for j in range(case["levels"]):
        assert G.normwise(sol.level_finals[j], ARR[name + "/level_finals"][j]) <= tol
    if case["trajectory"]:
        assert sol.trajectory.shape == ARR[name + "/trajectory"].shape
        assert G.normwise(sol.trajectory, ARR[name + "/trajectory"]) <= TOL
    # and against the oracle, which tracks the reference to ~1e-12 (1.4e-10 at 12 levels)
    ref = _oracle(ivp, case["levels"], case["steps"], case["restarts"])
    assert G.normwise(sol.final_state, ref["final_state"]) <= tol


def test_bitwise_determinism_executors_and_repeats():
    ivp = P.adv_diff_paper().ivp
    cfg = E.RidcConfig(levels=4, steps=2000, restarts=2, workers=4)
    a = E.run_pipelined(ivp, cfg).final_state
    b = E.run_serial(ivp, E.RidcConfig(levels=4, steps=2000, restarts=2, workers=1)).final_state
    with E.Engine(ivp, cfg) as eng:
        c = eng.run().final_state
        d = eng.run().final_state
    assert np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(c, d)


@pytest.mark.parametrize("kind_builder", [
    lambda: P.adv_diff_paper(),
    lambda: P.burgers_paper(),
    lambda: P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=4096, d=1e-3)),
    lambda: P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=1 << 16)),
    lambda: P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=64, ny=48)),
    lambda: P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=96, ny=32)),
], ids=["adv-diff", "burgers", "rd1d", "rd1d-seg", "ad2d", "rd2d"])
def test_operators_match_oracle(kind_builder):
    s = kind_builder()
    pd = s.problem
    u = s.ivp.initial_state + 0.1 * np.random.default_rng(3).standard_normal(pd.dimension)
    for dev_fn, orc_fn in ((ops.stiff_value, O.stiff), (ops.nonstiff_value, O.nonstiff)):
        got, ref = dev_fn(pd, u), orc_fn(pd, u)
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.abs(got - ref).max() <= 1e-13 * scale


SOLVE_CASES = [
    # (descriptor, coeff): whole-line exact and segmented truncated-halo paths
    (P.ProblemDescriptor(P.KIND_ADV_DIFF_1D, nx=7, c_x=0.1, d_x=1e-3, h_x=1 / 7), 50.0),
    (P.ProblemDescriptor(P.KIND_ADV_DIFF_1D, nx=1024, c_x=0.1, d_x=1e-3, h_x=1 / 1024), 4e-3),
    (P.ProblemDescriptor(P.KIND_REACTION_DIFFUSION_1D, nx=4094, d_x=1.0, rho=1.0, h_x=1 / 4094), 1e-3),
    (P.ProblemDescriptor(P.KIND_REACTION_DIFFUSION_1D, nx=8193, d_x=1e-6, rho=1.0, h_x=1 / 8193), 1e-2),
    (P.ProblemDescriptor(P.KIND_REACTION_DIFFUSION_1D, nx=1 << 20, d_x=1e-6, rho=1.0, h_x=2.0 ** -20), 1e-4),
    (P.ProblemDescriptor(P.KIND_REACTION_DIFFUSION_1D, nx=100003, d_x=1.0, rho=1.0, h_x=1e-5), 2e-8),
    (P.ProblemDescriptor(P.KIND_BURGERS_1D, nx=999, d_x=1e-3, h_x=1e-3), 1e-3),
    (P.ProblemDescriptor(P.KIND_BURGERS_1D, nx=50001, d_x=1.0, h_x=1 / 50002), 1e-7),
    (P.ProblemDescriptor(P.KIND_ADV_DIFF_2D, nx=4096, ny=5, c_x=0.1, c_y=0.1, d_x=1e-2, d_y=1e-3,
                         h_x=1 / 4096, h_y=0.2), 2e-5),
    (P.ProblemDescriptor(P.KIND_REACTION_DIFFUSION_2D, nx=20000, ny=3, d_x=1e-3, d_y=1e-4, rho=1.0,
                         h_x=1 / 20000, h_y=1 / 3), 5e-5),
]


@pytest.mark.parametrize("pd,coeff", SOLVE_CASES, ids=[f"k{p.kind}-{p.ny}x{p.nx}" for p, _ in SOLVE_CASES])
def test_solve_matches_oracle(pd, coeff):
    rng = np.random.default_rng(11)
    rhs = 1.0 + rng.standard_normal(pd.dimension)
    x = ops.solve_shifted(pd, coeff, rhs)
    xr = O.solve(pd, coeff, rhs)
    r = coeff * pd.d_x / pd.h_x ** 2
    # two backward-stable solvers agree to ~cond * eps, cond(I - dt L) ~ 1 + 4r
    assert G.normwise(x, xr) <= 1e-14 + 4e-16 * (1 + 4 * r)
    # residual of the structured system
    res = x - coeff * O.stiff(pd, x) - rhs
    assert np.abs(res).max() <= 1e-12 * np.abs(rhs).max() * (1 + 4 * coeff * pd.d_x / pd.h_x ** 2)


def test_segmented_solve_beyond_halo_limit_raises():
    """r ~ 6.7e4 on a line longer than one CTA needs a >1919-point truncation halo:
    documented limit, reported as ConfigError, never a silent fallback."""
    from paper_1209_4297_b200.errors import ConfigError
    pd = P.ProblemDescriptor(P.KIND_REACTION_DIFFUSION_1D, nx=8192, d_x=1.0, rho=1.0, h_x=1 / 8192)
    with pytest.raises(ConfigError):
        ops.solve_shifted(pd, 1e-3, np.ones(8192))


def test_predict_correct_kats(golden):
    cases, arr = golden
    spec = P.AdvectionDiffusionSpec(dx=1 / 64, t_end=1.0)
    sysm = P.build_advection_diffusion(spec)
    eta = sysm.ivp.initial_state
    dt = 0.01
    e1, fs1, fn1 = E.predict_step(sysm, 0.0, eta, dt)
    assert G.normwise(e1, arr["kat/predict/eta_new"]) <= 1e-13
    assert np.abs(fs1 - arr["kat/predict/fs"]).max() <= 1e-9 * np.abs(arr["kat/predict/fs"]).max()
    assert np.abs(fn1 - arr["kat/predict/fn"]).max() <= 1e-9 * np.abs(arr["kat/predict/fn"]).max()
    w = steady_weights(2, dt)
    win = E.LevelWindow.from_states(arr["kat/correct/window_states"], 0, 1)
    ec, _, _ = E.correct_step(2, sysm, 0.0, eta, win, w, dt)
    assert G.normwise(ec, arr["kat/correct/eta_new"]) <= 1e-13
    # the reference's own constructor: LevelWindow(fs, fn, new_index, old_index)
    ref_win = E.LevelWindow(arr["kat/correct/fs_win"], arr["kat/correct/fn_win"], 0, 1)
    ec2, _, _ = E.correct_step(2, sysm, 0.0, eta, ref_win, w, dt)
    assert G.normwise(ec2, arr["kat/correct/eta_new"]) <= 1e-13


def test_nonfinite_is_reported_like_the_reference(golden):
    cases, _ = golden
    c = next(c for c in cases if c["name"] == "bu_n255_blowup")
    system = P.build_burgers(P.BurgersSpec(dx=1 / 256, t_end=0.5))
    with pytest.raises(NonFiniteStateError) as ei:
        E.run_serial(system, E.RidcConfig(levels=1, steps=c["steps"]))
    assert str(ei.value) == c["message"]


def test_c2_shape_against_oracle():
    """BASELINE configs[1] grid (N = 2^20, r ~ 110, segmented solve), bounded steps."""
    system = P.reaction_diffusion_c2()
    ivp = P.StructuredIVP(system.problem, 0.0, 0.02, system.ivp.initial_state)   # dt = 1e-4
    for levels in (1, 3):
        sol = E.run_serial(ivp, E.RidcConfig(levels=levels, steps=200))
        ref = _oracle(ivp, levels, 200, level_finals=True)
        assert G.normwise(sol.final_state, ref["final_state"]) <= TOL
        for j in range(levels):
            assert G.normwise(sol.level_finals[j], ref["level_finals"][j]) <= TOL


def test_2d_against_oracle():
    s = P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=512, ny=256, t_end=0.002))
    sol = E.run_serial(s, E.RidcConfig(levels=4, steps=40))
    ref = _oracle(s.ivp, 4, 40)
    assert G.normwise(sol.final_state, ref["final_state"]) <= TOL
    s2 = P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=9000, ny=8, t_end=0.001))
    sol = E.run_serial(s2, E.RidcConfig(levels=3, steps=20, restarts=2))
    ref = _oracle(s2.ivp, 3, 20, 2)
    assert G.normwise(sol.final_state, ref["final_state"]) <= TOL


def test_mean_conservation():
    """Acceptance 8: periodic adv-diff mean drift <= 1e-12 relative over 1000 RIDC4 steps."""
    s = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 200, t_end=4.0))
    sol = E.run_serial(s, E.RidcConfig(levels=4, steps=1000))
    m0 = s.ivp.initial_state.mean()
    assert abs(sol.final_state.mean() - m0) <= 1e-12 * abs(m0)


def _slopes(levels, steps_list, t_end, dx=1 / 200):
    spec = P.AdvectionDiffusionSpec(dx=dx, t_end=t_end)
    s = P.build_advection_diffusion(spec)
    exact = P.exact_advection_diffusion(spec, t_end)
    errs = []
    for n in steps_list:
        sol = E.run_serial(s, E.RidcConfig(levels=levels, steps=n))
        errs.append(np.abs(sol.final_state - exact).max())
    return [np.log(errs[i] / errs[i + 1]) / np.log(steps_list[i + 1] / steps_list[i])
            for i in range(len(errs) - 1)], errs


@pytest.mark.parametrize("levels", [1, 2, 3, 4])
def test_order_ladder(levels):
    """Acceptance 1 (order p), against the exact semi-discrete solution."""
    sl, _ = _slopes(levels, [100, 200, 400, 800], 4.0)
    if levels == 1:
        assert abs(sl[-1] - 1.0) <= 0.2
    else:
        assert sl[-1] >= levels - 0.4


def test_order_eight():
    sl, errs = _slopes(8, [200, 400], 40.0)
    assert sl[-1] >= 7.0, (sl, errs)


def test_restart_trend():
    """Restarts reduce the error at long horizons (PAPER Fig. 3; F8 at T=40)."""
    spec = P.AdvectionDiffusionSpec(dx=1 / 200, t_end=40.0)
    s = P.build_advection_diffusion(spec)
    exact = P.exact_advection_diffusion(spec, 40.0)
    e1 = np.abs(E.run_serial(s, E.RidcConfig(levels=4, steps=4000)).final_state - exact).max()
    e10 = np.abs(E.run_serial(s, E.RidcConfig(levels=4, steps=4000, restarts=10)).final_state - exact).max()
    assert e10 < e1


def test_engine_info_and_launch_count():
    s = P.reaction_diffusion_c2(n=1 << 16)
    with E.Engine(s, E.RidcConfig(levels=4, steps=100), tick_only=True) as eng:
        inf = eng.info
        assert inf["ticks_per_interval"] == 100 + 6
        assert inf["kernel_launches"] == 1 + 106   # seed + one tick launch per tick
    with E.Engine(s, E.RidcConfig(levels=4, steps=100, restarts=2)) as eng:
        assert eng.info["kernel_launches"] == 3 * 2   # resident level march: 2 seeds + 1 launch per interval
        assert inf["halo"] > 0 and inf["items_per_level"] >= 8


def test_burgers_layer_propagates_right():
    """SPEC acceptance 10 (PAPER Fig. 5): at eps = 1e-3, desk scale, the steepest
    descent of u sits strictly further right at t = 1 than at t = 0.2."""
    s = P.burgers_desk()
    steps = 1000
    sol = E.run_serial(s, E.RidcConfig(levels=4, steps=steps, record_trajectory=True))
    dx = s.problem.h_x
    def front(u):
        return int(np.argmin(np.diff(u))) * dx
    x02 = front(sol.trajectory[steps // 5])
    x1 = front(sol.trajectory[steps])
    assert x1 > x02, (x02, x1)
