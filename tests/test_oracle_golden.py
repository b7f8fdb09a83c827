"""Pin the CPU oracle against the reference's own outputs (tests/golden/).

The golden vectors were produced by running the reference implementation
(tests/golden/make_golden.py).  Bar: normwise relative error <= 1e-10
(SURVEY.md §8c); the structured restatement lands at <= 3e-12 here.
"""

import numpy as np
import pytest

import _golden as G
from oracle import oracle as O
from paper_1209_4297_b200.quadrature import pack_weight_tables

RUNS, ARR = G.run_cases()


@pytest.mark.parametrize("case", RUNS, ids=[c["name"] for c in RUNS])
def test_oracle_matches_reference_run(case):
    pd = G.descriptor(case["problem"])
    dt = case["t_end"] / case["steps"]
    r = O.run(pd, ARR[case["name"] + "/y0"], case["levels"], case["steps"], case["restarts"], dt,
              pack_weight_tables(case["levels"], dt), workers=case["workers"],
              level_finals=True, record_trajectory=case["trajectory"])
    tol = G.tolerance(case["levels"])
    assert G.normwise(r["final_state"], ARR[case["name"] + "/final"]) <= tol
    for j in range(case["levels"]):
        assert G.normwise(r["level_finals"][j], ARR[case["name"] + "/level_finals"][j]) <= tol
    if case["trajectory"]:
        assert G.normwise(r["trajectory"], ARR[case["name"] + "/trajectory"]) <= 1e-10


def test_oracle_pipelined_workers_bitwise():
    """The reference's determinism gate (engine.py:497-503) holds for the oracle."""
    c = next(c for c in RUNS if c["name"] == "ad_c1_p4")
    pd = G.descriptor(c["problem"])
    dt = c["t_end"] / c["steps"]
    w = pack_weight_tables(4, dt)
    outs = [O.run(pd, ARR["ad_c1_p4/y0"], 4, 1000, 1, dt, w, workers=k)["final_state"]
            for k in (1, 2, 4)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_oracle_kat_predict_correct(golden):
    cases, arr = golden
    kat = next(c for c in cases if c["name"] == "kat/predict")
    pd = G.descriptor(kat["problem"])
    dt = kat["dt"]
    from paper_1209_4297_b200 import problems as P
    eta = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 64, t_end=1.0)).ivp.initial_state
    e1, fs1, fn1 = O.predict_step(pd, dt, eta)
    assert G.normwise(e1, arr["kat/predict/eta_new"]) <= 1e-13
    assert np.abs(fs1 - arr["kat/predict/fs"]).max() <= 1e-9 * np.abs(arr["kat/predict/fs"]).max()
    from paper_1209_4297_b200.quadrature import steady_weights
    ec, _, _ = O.correct_step(pd, dt, eta, arr["kat/correct/fs_win"], arr["kat/correct/fn_win"],
                              0, 1, steady_weights(2, dt).weights)
    assert G.normwise(ec, arr["kat/correct/eta_new"]) <= 1e-13


def test_oracle_blowup_reports_nonfinite(golden):
    cases, _ = golden
    c = next(c for c in cases if c["name"] == "bu_n255_blowup")
    pd = G.descriptor(c["problem"])
    from paper_1209_4297_b200 import problems as P
    y0 = P.build_burgers(P.BurgersSpec(dx=1 / 256, t_end=0.5)).ivp.initial_state
    dt = c["t_end"] / c["steps"]
    with pytest.raises(O.OracleError) as ei:
        O.run(pd, y0, 1, c["steps"], 1, dt, pack_weight_tables(1, dt))
    assert ei.value.code == O.NONFINITE
    assert "step 53" in str(ei.value) and c["message"].endswith("step 53")


def test_golden_kats(golden):
    _, arr = golden
    assert abs(arr["kat/fbe_scalar"][0] - 2.0 / 3.0) <= 1e-15
    assert list(arr["kat/startup_delay"]) == [0, 1, 3, 6, 10, 15, 21, 28]
    assert arr["kat/burgers_flux"][1] == pytest.approx(-2.0 / 0.1)
