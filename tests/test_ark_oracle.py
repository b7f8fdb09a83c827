"""Pin the oracle's ARK restatement (oracle.ark: steppers.integrate_ark,
steppers.py:122-155) against the reference's own integrate_ark outputs for the
imex3 / imex4 pairs (tests/golden/make_golden.py), and check the tableau
mirror against the reference's rationals (tableaus.py:82-127)."""

import numpy as np
import pytest

import _golden as G
from oracle import oracle as O
from paper_1209_4297_b200.errors import ConfigError
from paper_1209_4297_b200.tableaus import ButcherPair, imex3_tableau, imex4_tableau

ARK, ARR = G.ark_cases()


def _tab(scheme):
    return imex3_tableau() if scheme == "imex3" else imex4_tableau()


@pytest.mark.parametrize("case", ARK, ids=[c["name"] for c in ARK])
def test_oracle_ark_matches_reference(case):
    pd = G.descriptor(case["problem"])
    t = _tab(case["scheme"])
    y = O.ark(pd, t.a_implicit, t.a_explicit, t.b_implicit, t.b_explicit, ARR[case["name"] + "/y0"],
              0.0, case["t_end"], case["steps"])
    assert G.normwise(y, ARR[case["name"] + "/final"]) <= 1e-10


def test_tableau_consistency():
    for tab, s, diag in ((imex3_tableau(), 5, [0, .5, 2 / 3, 2, 1]),
                         (imex4_tableau(), 7, [0, .5, .5, .5, .5, .5, 2 / 3])):
        assert tab.stages == s
        assert np.allclose(np.diag(tab.a_implicit), diag, atol=0, rtol=1e-15)
        assert abs(tab.b_implicit.sum() - 1.0) < 1e-14 and abs(tab.b_explicit.sum() - 1.0) < 1e-14
        assert np.abs(tab.a_implicit.sum(1) - tab.c).max() <= 1e-14
    assert imex4_tableau().shifts(0.1) == [0.05, 0.1 * 2 / 3]


def test_tableau_validation():
    c = np.array([0.0, 1.0])
    with pytest.raises(ConfigError):
        ButcherPair(c, np.array([[0.0, 1.0], [0.0, 1.0]]), np.zeros((2, 2)), np.ones(2) / 2, np.ones(2) / 2)
    with pytest.raises(ConfigError):
        ButcherPair(c, np.zeros((2, 2)), np.eye(2), np.ones(2) / 2, np.ones(2) / 2)
