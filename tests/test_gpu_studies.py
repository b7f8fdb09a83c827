"""The reference's acceptance criteria through the device study harness
(SPEC.md:569-577): order ladder vs the IMEX4 fine reference (1), ARK design
orders (2), the paper's error-constant ordering (Fig. 4), restart trend
(Fig. 3), the speedup table's 1-GPU row and bitwise gate, and the CLI."""

import io

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1209_4297_b200 import cli, studies as S  # noqa: E402

STEPS = (100, 200, 400, 800, 1600)


@pytest.fixture(scope="module")
def desk():
    cfg = S.StudyConfig(problem="adv-diff", step_counts=STEPS)
    system = S.make_system(cfg)
    from paper_1209_4297_b200.problems import reference_solution
    ref = reference_solution(system, system.ivp.t_end, cfg.refinement, max(STEPS))
    return system, ref


@pytest.mark.parametrize("scheme,lo,hi", [("fbe", 0.8, 1.2), ("ridc-2", 1.6, 9), ("ridc-3", 2.6, 9),
                                          ("ridc4-fbe", 3.6, 9), ("imex3", 2.6, 3.4), ("imex4", 3.6, 4.4)])
def test_convergence_orders(desk, scheme, lo, hi):
    system, ref = desk
    cfg = S.StudyConfig(problem="adv-diff", scheme=scheme, step_counts=STEPS)
    rows = S.run_convergence(cfg, system=system, reference=ref)
    assert rows[0].observed_order is None
    last = rows[-1].observed_order if scheme in ("fbe", "imex3", "imex4") else rows[-2].observed_order
    assert lo <= last <= hi, [(r.steps, r.error_inf, r.observed_order) for r in rows]
    assert all(r.wall_ms > 0 for r in rows)


def test_imex4_error_constant_below_ridc4(desk):
    system, ref = desk
    e = {}
    for scheme in ("imex4", "ridc4-fbe"):
        rows = S.run_convergence(S.StudyConfig(scheme=scheme, step_counts=(200, 400)), system=system, reference=ref)
        e[scheme] = rows[-1].error_inf
    assert e["imex4"] < e["ridc4-fbe"]


def test_restart_trend_and_degenerate_partition():
    cfg = S.StudyConfig(problem="adv-diff", scheme="ridc4-fbe", step_counts=(4000,), t_end=40.0)
    rows = S.run_restart_study(cfg, [1, 2, 5, 10])
    assert rows[-1].error_inf < rows[0].error_inf
    system = S.make_system(cfg)
    a, _ = S.integrate_scheme(system, "ridc4-fbe", 4000, restarts=1)
    b, _ = S.integrate_scheme(system, "ridc4-fbe", 4000)
    assert np.array_equal(a, b)


def test_speedup_single_gpu_row():
    rows = S.run_speedup(S.StudyConfig(scheme="ridc-4", step_counts=(400,), reps=2), [1])
    assert len(rows) == 1 and rows[0].speedup == 1.0 and rows[0].wall_ms > 0


def test_cli_converge_writes_csv(tmp_path):
    out = tmp_path / "conv.csv"
    buf = io.StringIO()
    rc = cli.main(["converge", "--scheme", "ridc-3", "--steps", "100,200,400", "--out", str(out)], out=buf)
    assert rc == cli.EXIT_OK
    rows = S.read_csv(str(out))
    assert [r.steps for r in rows] == [100, 200, 400] and rows[-1].observed_order > 2.5
    assert "fitted order" in buf.getvalue()
