"""Study harness + CLI host logic (no GPU): the reference's studies.py contract
(StudyConfig validation, fit_order, the 9-column CSV with 17 significant digits
and its round trip) and the CLI's surface / exit codes."""

import io
import math

import pytest

from paper_1209_4297_b200 import cli, studies as S
from paper_1209_4297_b200.errors import ConfigError


def test_scheme_levels_and_config_validation():
    assert S.scheme_levels("fbe") == 1 and S.scheme_levels("ridc4-fbe") == 4
    assert S.scheme_levels("ridc-7") == 7 and S.scheme_levels("imex4") is None
    for bad in ("ridc-1", "ridc-13", "rk4"):
        with pytest.raises(ConfigError):
            S.scheme_levels(bad)
    with pytest.raises(ConfigError):
        S.StudyConfig(step_counts=(200, 100))
    with pytest.raises(ConfigError):
        S.StudyConfig(problem="heat")
    with pytest.raises(ConfigError):
        S.StudyConfig(norm="l1")
    with pytest.raises(ConfigError):
        S.StudyConfig(workers=0)


def _rows():
    return [S.ResultRow("ridc4-fbe", 100, 0.04, 1.2345678901234567e-05, 3.3e-06, 12.5, 1, 1, None),
            S.ResultRow("ridc4-fbe", 200, 0.02, 7.7e-07, 2.0e-07, 20.25, 1, 1, 4.003)]


def test_csv_contract_and_round_trip(tmp_path):
    p = tmp_path / "out.csv"
    S.emit_csv(_rows(), str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == S.CSV_HEADER
    assert all(len(ln.split(",")) == 9 for ln in lines)
    assert lines[1].split(",")[8] == ""                       # first row: no observed order
    assert lines[1].split(",")[3] == format(1.2345678901234567e-05, ".17g")
    assert S.read_csv(str(p)) == _rows()
    S.emit_csv([], str(p))
    assert p.read_text().splitlines() == [S.CSV_HEADER]
    with pytest.raises(OSError):
        S.emit_csv(_rows(), str(tmp_path / "missing" / "x.csv"))


def test_fit_order():
    rows = [S.ResultRow("x", n, 1.0 / n, 3.0 * (1.0 / n) ** 4, 1.0, 0.0, 1, 1) for n in (100, 200, 400)]
    assert abs(S.fit_order(rows) - 4.0) < 1e-12
    rows.append(S.ResultRow("x", 800, 1 / 800, math.nan, math.nan, math.nan, 1, 1))
    assert abs(S.fit_order(rows) - 4.0) < 1e-12
    with pytest.raises(ValueError):
        S.fit_order(rows[:1])


def test_speedup_and_restart_validation(monkeypatch):
    monkeypatch.setenv("RIDC_FORCE_PARALLELISM", "1")
    assert S.available_parallelism() == 1
    cfg = S.StudyConfig(scheme="ridc-4", step_counts=(1000,))
    with pytest.raises(ConfigError):
        S.run_speedup(cfg, [2, 4])              # must include 1
    with pytest.raises(ConfigError):
        S.run_speedup(cfg, [1, 2])              # one level per GPU: 1 or levels
    with pytest.raises(ConfigError):
        S.run_speedup(cfg, [1, 4])              # only 1 GPU available
    with pytest.raises(ConfigError):
        S.run_speedup(S.StudyConfig(scheme="imex4"), [1])
    with pytest.raises(ConfigError):
        S.run_restart_study(cfg, [3])           # 3 does not divide 1000
    with pytest.raises(ConfigError):
        S.run_restart_study(cfg, [1000])        # interval shorter than the pipeline fill
    monkeypatch.setenv("RIDC_FORCE_PARALLELISM", "zero")
    with pytest.raises(ConfigError):
        S.available_parallelism()


def test_cli_config_file_and_exit_codes(tmp_path, monkeypatch):
    cfgf = tmp_path / "study.cfg"
    cfgf.write_text("# desk run\nproblem = burgers\nscheme = ridc-3\nsteps = 100, 200\nreps = 2\n")
    args = cli.build_parser().parse_args(["converge", "--config", str(cfgf), "--scheme", "fbe"])
    cfg, extra = cli.study_config(args)
    assert (cfg.problem, cfg.scheme, cfg.step_counts, cfg.reps) == ("burgers", "fbe", (100, 200), 2)
    bad = tmp_path / "bad.cfg"
    bad.write_text("colour = blue\n")
    assert cli.main(["converge", "--config", str(bad)], out=io.StringIO()) == cli.EXIT_CONFIG
    assert cli.main(["converge", "--steps", "400,100"], out=io.StringIO()) == cli.EXIT_CONFIG
    monkeypatch.setenv("RIDC_FORCE_PARALLELISM", "1")
    assert cli.main(["speedup", "--scheme", "ridc-4", "--worker-counts", "1,4"],
                    out=io.StringIO()) == cli.EXIT_CONFIG
