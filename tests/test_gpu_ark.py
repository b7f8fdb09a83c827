"""Device ARK comparators (ridc_ark_*) vs the reference's integrate_ark
golden vectors and the oracle; convergence orders 3 and 4 against the exact
semi-discrete adv-diff solution (the paper's Fig. 4b / 6b comparators)."""

import numpy as np
import pytest

import _golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1209_4297_b200 import problems as P, steppers as S, studies  # noqa: E402
from paper_1209_4297_b200.errors import NonFiniteStateError  # noqa: E402
from paper_1209_4297_b200.tableaus import imex3_tableau, imex4_tableau  # noqa: E402

ARK, ARR = G.ark_cases()


def _tab(scheme):
    return imex3_tableau() if scheme == "imex3" else imex4_tableau()


@pytest.mark.parametrize("case", ARK, ids=[c["name"] for c in ARK])
def test_device_ark_matches_reference_golden(case):
    pd = G.descriptor(case["problem"])
    y0 = ARR[case["name"] + "/y0"]
    ivp = P.StructuredIVP(pd, 0.0, case["t_end"], y0)
    tab = _tab(case["scheme"])
    y = S.integrate_ark(ivp, tab, 0.0, y0, case["t_end"], case["steps"])
    assert G.normwise(y, ARR[case["name"] + "/final"]) <= 1e-10
    ref = O.ark(pd, tab.a_implicit, tab.a_explicit, tab.b_implicit, tab.b_explicit, y0, 0.0,
                case["t_end"], case["steps"])
    assert G.normwise(y, ref) <= 1e-10


def test_segmented_long_line_against_oracle():
    """C2-shaped grid (2^16 points, truncated-halo segments), imex4."""
    s = P.reaction_diffusion_c2(n=1 << 16)
    ivp = P.StructuredIVP(s.problem, 0.0, 0.002, s.ivp.initial_state)
    tab = imex4_tableau()
    with S.ArkEngine(ivp, tab, 0.0, 0.002, 20) as eng:
        y, wall = eng.run(ivp.initial_state)
        inf = eng.info
    # the carry-exchange path adds the run's tag-epoch bump to the seed launch
    assert inf["path_name"] == "carry_levels", inf
    assert inf["items_per_step"] == tab.stages and inf["kernel_launches"] == 2 + 20 * tab.stages
    ref = O.ark(s.problem, tab.a_implicit, tab.a_explicit, tab.b_implicit, tab.b_explicit,
                ivp.initial_state, 0.0, 0.002, 20)
    assert G.normwise(y, ref) <= 1e-10 and wall > 0


@pytest.mark.parametrize("scheme", ["imex3", "imex4"])
@pytest.mark.parametrize("exp", [16, 20])
def test_ark_carry_levels_vs_tick(scheme, exp, monkeypatch):
    """Periodic RD lines of 512-point chunks run every ARK stage on the
    carry-exchange tick (csrc/ridc_carry_levels.cuh, one chunk per warp): the
    same stage solves as the tick kernel to rounding (<= 1e-12), the oracle
    to <= 1e-10, and repeat runs bitwise (C2's grid and dt at exp = 20)."""
    s = P.reaction_diffusion_c2(n=1 << exp)
    steps = 20 if exp < 20 else 8   # the numpy oracle takes ~1.5 s per imex4 step at 2^20
    ivp = P.StructuredIVP(s.problem, 0.0, 1e-4 * steps, s.ivp.initial_state)
    tab = _tab(scheme)
    # imex3's stiffest stage (a_ii = 2) at C2's r ~ 110 has a carry reach of 618
    # points: 1024-point chunks (32 points per lane) there
    with S.ArkEngine(ivp, tab, 0.0, 1e-4 * steps, steps) as eng:
        assert eng.info["path_name"] == "carry_levels", eng.info
        a, _ = eng.run(ivp.initial_state)
        a2, _ = eng.run(ivp.initial_state)
    monkeypatch.setenv("RIDC_NO_CARRYLEV", "1")
    with S.ArkEngine(ivp, tab, 0.0, 1e-4 * steps, steps) as eng:
        assert eng.info["path_name"] == "tick", eng.info
        b, _ = eng.run(ivp.initial_state)
    assert np.array_equal(a, a2)
    assert G.normwise(a, b) <= 1e-12
    ref = O.ark(s.problem, tab.a_implicit, tab.a_explicit, tab.b_implicit, tab.b_explicit,
                ivp.initial_state, 0.0, 1e-4 * steps, steps)
    assert G.normwise(a, ref) <= 1e-10


@pytest.mark.parametrize("scheme,order", [("imex3", 3), ("imex4", 4)])
def test_ark_order(scheme, order):
    spec = P.AdvectionDiffusionSpec(dx=1 / 200, t_end=4.0)
    s = P.build_advection_diffusion(spec)
    exact = P.exact_advection_diffusion(spec, 4.0)
    errs = [np.abs(studies.integrate_scheme(s, scheme, n)[0] - exact).max() for n in (50, 100, 200)]
    slope = np.log(errs[-2] / errs[-1]) / np.log(2.0)
    assert slope >= order - 0.3, (errs, slope)


def test_ark_step_and_reference_solution():
    s = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 64, t_end=1.0))
    tab = imex3_tableau()
    y1 = S.ark_step(s, tab, 0.0, s.ivp.initial_state, 0.01)
    ref = O.ark(s.problem, tab.a_implicit, tab.a_explicit, tab.b_implicit, tab.b_explicit,
                s.ivp.initial_state, 0.0, 0.01, 1)
    assert G.normwise(y1, ref) <= 1e-12
    r = P.reference_solution(s, 1.0, 8, 10)
    assert np.isfinite(r).all() and r.shape == s.ivp.initial_state.shape


def test_ark_nonfinite_message():
    s = P.build_burgers(P.BurgersSpec(dx=1 / 256, t_end=0.5))
    with pytest.raises(NonFiniteStateError) as ei:
        S.integrate_ark(s, imex3_tableau(), 0.0, s.ivp.initial_state, 0.5, 20)
    assert str(ei.value).startswith("ARK march produced non-finite entries at step ")
