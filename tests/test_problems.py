"""Problem descriptors and the reference-system boundary."""

import numpy as np
import pytest

from paper_1209_4297_b200 import problems as P
from paper_1209_4297_b200.errors import ConfigError, DimensionMismatch


def test_presets_match_reference_shapes():
    assert P.adv_diff_desk().ivp.dimension == 200
    assert P.adv_diff_paper().ivp.dimension == 1000
    assert P.burgers_desk().ivp.dimension == 499
    assert P.burgers_paper().ivp.dimension == 999


def test_initial_states():
    s = P.adv_diff_desk()
    x = np.arange(200) / 200
    assert np.allclose(s.ivp.initial_state, 2 + np.sin(2 * np.pi * x))
    b = P.burgers_desk()
    x = (np.arange(499) + 1) / 500
    assert np.allclose(b.ivp.initial_state, np.sin(2 * np.pi * x) + 0.5 * np.sin(np.pi * x))
    rd = P.reaction_diffusion_c2(n=1024)
    assert rd.ivp.dimension == 1024 and abs(rd.ivp.initial_state.mean() - 0.5) < 1e-3


def test_descriptor_validation():
    with pytest.raises(ConfigError):
        P.ProblemDescriptor(kind=9, nx=10)
    with pytest.raises(ConfigError):
        P.ProblemDescriptor(kind=P.KIND_ADV_DIFF_1D, nx=2, d_x=1.0)
    with pytest.raises(ConfigError):
        P.ProblemDescriptor(kind=P.KIND_ADV_DIFF_2D, nx=8, ny=2, d_x=1.0)
    with pytest.raises(ConfigError):
        P.AdvectionDiffusionSpec(dx=0.3)
    with pytest.raises(DimensionMismatch):
        P.StructuredIVP(P.adv_diff_desk().problem, 0.0, 1.0, np.zeros(3))


def test_exact_solution_at_zero():
    spec = P.AdvectionDiffusionSpec(dx=1 / 200, t_end=4.0)
    assert np.allclose(P.exact_advection_diffusion(spec, 0.0), P.build_advection_diffusion(spec).ivp.initial_state)


def test_error_norms():
    inf, l2 = P.error_norms(np.array([1.0, 2.0]), np.array([1.0, 0.0]), 0.5)
    assert inf == 2.0 and l2 == pytest.approx(np.sqrt(0.5 * 4))


def test_reference_system_is_accepted(reference):
    from ridc import problems as RP
    sysr = RP.build_advection_diffusion(RP.AdvectionDiffusionSpec(dx=1 / 128, t_end=0.5))
    ivp = P.as_descriptor(sysr)
    assert ivp.problem.kind == P.KIND_ADV_DIFF_1D and ivp.problem.nx == 128
    assert np.array_equal(ivp.initial_state, sysr.ivp.initial_state)
    bu = P.as_descriptor(RP.build_burgers(RP.BurgersSpec(dx=1 / 64)))
    assert bu.problem.kind == P.KIND_BURGERS_1D and bu.problem.nx == 63
    with pytest.raises(ConfigError):
        P.as_descriptor(sysr.ivp)          # opaque callables: no device path, no fallback


def test_reference_dense_operators_match_descriptor(reference):
    """The stencil coefficients reproduce the reference's dense rows (problems.py:119-124)."""
    from ridc import problems as RP
    from oracle import oracle as O
    sysr = RP.build_advection_diffusion(RP.AdvectionDiffusionSpec(dx=1 / 64, t_end=1.0))
    pd = P.as_descriptor(sysr).problem
    u = np.random.default_rng(1).standard_normal(64)
    assert np.allclose(O.stiff(pd, u), sysr.diffusion_matrix @ u, rtol=1e-13, atol=1e-9)
    assert np.allclose(O.nonstiff(pd, u), sysr.advection_matrix @ u, rtol=1e-13, atol=1e-11)
