"""``ridc`` command line: the study harness the reference declares but does not
ship (pyproject.toml:19-20 names ``ridc.cli:main``; SPEC.md:543-556 fixes its
surface).

    python -m paper_1209_4297_b200 converge --problem adv-diff --scheme ridc4-fbe --steps 100,200,400
    python -m paper_1209_4297_b200 restarts --restart-counts 1,2,5,10 --steps 4000
    python -m paper_1209_4297_b200 speedup  --scheme ridc-4 --worker-counts 1,4

Flags: --problem --scheme --steps --workers --restarts --dx --t-end
--paper-scale --out (CSV) --norm --refinement --reps, and --config FILE
(plain ``key = value`` lines; flags override file values).  Exit codes: 0
success, 1 configuration error, 2 solver failure, 3 determinism-gate failure.
"""

import argparse
import sys

from .errors import SOLVER_FAILURES, ConfigError, DeterminismError
from . import studies as S

EXIT_OK, EXIT_CONFIG, EXIT_SOLVER, EXIT_DETERMINISM = 0, 1, 2, 3

_KEYS = {"problem": str, "scheme": str, "steps": str, "workers": int, "restarts": int, "dx": float,
         "t_end": float, "paper_scale": lambda v: str(v).lower() in ("1", "true", "yes", "on"),
         "out": str, "norm": str, "refinement": int, "reps": int, "worker_counts": str,
         "restart_counts": str}


def _ints(text: str) -> tuple:
    try:
        return tuple(int(x) for x in str(text).replace(" ", "").split(",") if x)
    except ValueError as exc:
        raise ConfigError(f"expected a comma-separated integer list, got {text!r}") from exc


def read_config(path: str) -> dict:
    """``key = value`` lines (``#`` comments); keys as the long flags with '_' or '-'."""
    out = {}
    try:
        with open(path) as fh:
            for ln, line in enumerate(fh, 1):
                line = line.split("#", 1)[0].strip()
                if not line:
                    continue
                if "=" not in line:
                    raise ConfigError(f"{path}:{ln}: expected key = value")
                k, v = (x.strip() for x in line.split("=", 1))
                k = k.replace("-", "_")
                if k not in _KEYS:
                    raise ConfigError(f"{path}:{ln}: unknown key {k!r}")
                out[k] = _KEYS[k](v)
    except OSError as exc:
        raise ConfigError(f"cannot read config {path!r}: {exc}") from exc
    return out


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="ridc", description="RIDC / ARK studies on the B200 device engine")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("converge", "speedup", "restarts"):
        p = sub.add_parser(name)
        p.add_argument("--config")
        p.add_argument("--problem")
        p.add_argument("--scheme")
        p.add_argument("--steps", help="comma-separated step counts (the last is used by speedup/restarts)")
        p.add_argument("--workers", type=int)
        p.add_argument("--restarts", type=int)
        p.add_argument("--dx", type=float)
        p.add_argument("--t-end", dest="t_end", type=float)
        p.add_argument("--paper-scale", dest="paper_scale", action="store_true", default=None)
        p.add_argument("--out")
        p.add_argument("--norm")
        p.add_argument("--refinement", type=int)
        p.add_argument("--reps", type=int)
        if name == "speedup":
            p.add_argument("--worker-counts", dest="worker_counts")
        if name == "restarts":
            p.add_argument("--restart-counts", dest="restart_counts")
    return ap


def study_config(args) -> tuple:
    vals = read_config(args.config) if args.config else {}
    for k in _KEYS:
        v = getattr(args, k, None)
        if v is not None:
            vals[k] = v
    extra = {k: vals.pop(k) for k in ("worker_counts", "restart_counts") if k in vals}
    if "steps" in vals:
        vals["step_counts"] = _ints(vals.pop("steps"))
    return S.StudyConfig(**vals), extra


def _print_rows(rows, out):
    print(S.CSV_HEADER.replace(",", "  "), file=out)
    for r in rows:
        print(f"{r.scheme:10s} {r.steps:7d} {r.dt:11.4e} {r.error_inf:11.4e} {r.error_l2:11.4e} "
              f"{r.wall_ms:10.3f} {r.workers:3d} {r.restarts:3d} "
              f"{'' if r.observed_order is None else format(r.observed_order, '.3f')}", file=out)


def main(argv=None, out=None) -> int:
    out = out or sys.stdout
    args = build_parser().parse_args(argv)
    try:
        cfg, extra = study_config(args)
        if args.cmd == "converge":
            rows = S.run_convergence(cfg)
            _print_rows(rows, out)
            try:
                print(f"fitted order: {S.fit_order(rows, cfg.norm):.3f}", file=out)
            except ValueError:
                pass
            if cfg.out:
                S.emit_csv(rows, cfg.out)
        elif args.cmd == "restarts":
            rows = S.run_restart_study(cfg, _ints(extra.get("restart_counts", "1,2,5,10")))
            _print_rows(rows, out)
            if cfg.out:
                S.emit_csv(rows, cfg.out)
        else:
            levels = S.scheme_levels(cfg.scheme) or 1
            counts = _ints(extra.get("worker_counts", f"1,{levels}" if levels > 1 else "1"))
            rows = S.run_speedup(cfg, counts)
            print("workers  wall_ms  speedup", file=out)
            for r in rows:
                print(f"{r.workers:7d} {r.wall_ms:9.3f} {r.speedup:8.3f}", file=out)
    except ConfigError as exc:
        print(f"ridc: configuration error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except SOLVER_FAILURES as exc:
        print(f"ridc: solver failure: {exc}", file=sys.stderr)
        return EXIT_SOLVER
    except DeterminismError as exc:
        print(f"ridc: determinism gate failed: {exc}", file=sys.stderr)
        return EXIT_DETERMINISM
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
