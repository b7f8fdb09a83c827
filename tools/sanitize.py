"""Small marches of every kernel family against the CPU oracle: the tick
kernel (1-D segmented, whole-line, 2-D x-lines), the resident marches (FEBE:
halo exchange and carry exchange; all levels; the resident RIDC-2), the
streaming sweeps (1-D FEBE per warp, 2-D FEBE, 2-D levels), the carry-level
tick, the pipeline ranks, levels x row shards and the ARK comparators.

Run it under compute-sanitizer where that is available, or -- on the GPU pool,
where compute-sanitizer is closed -- against the checked build, whose kernels
assert their bounds and pipeline-protocol invariants (RIDC_CHECK, ridc_device.cuh):

    compute-sanitizer --tool memcheck python tools/sanitize.py [--cases a,b]
    RIDC_CHECKED=1 python tools/sanitize.py      # __graft_entry__.build(checked=True) first
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1209_4297_b200 import distributed as PD  # noqa: E402
from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402
from paper_1209_4297_b200.quadrature import pack_weight_tables  # noqa: E402


def _short(system, t):
    ivp = system.ivp
    return P.StructuredIVP(ivp.problem, 0.0, t, ivp.initial_state)


def c1(t=0.04):
    return _short(P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024, t_end=4.0)), t)


def seg(n=1 << 15, steps=20):
    # r ~ 110 as C2: several truncated segments with halos
    return _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)),
                  1e-4 * steps)


CASES = {
    "febe-whole": (lambda: c1(), 1, 10, {}),
    "febe-carry": (lambda: seg(), 1, 20, {}),
    "febe-halo-seg": (lambda: _short(P.build_burgers(P.BurgersSpec(dx=1 / (1 << 15))), 0.002), 1, 20, {}),
    "febe-sweep": (lambda: seg(1 << 21, 10), 1, 10, {}),
    "febe-sweep2d": (lambda: P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(
        nx=4096, ny=600, t_end=0.02 * 6 / 1000)).ivp, 1, 6, {}),
    "levels-sweep2d-p3": (lambda: P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(
        nx=4096, ny=400, t_end=0.05 * 10 / 1000)).ivp, 3, 10, {}),
    "tick-seg-p3": (lambda: seg(), 3, 20, {"tick_only": True}),
    "levels-seg-p3": (lambda: seg(), 3, 20, {}),
    "levels-whole-p4": (lambda: c1(), 4, 20, {}),
    "tick-2d-p2": (lambda: P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=256, ny=16,
                                                                                     t_end=1e-4)).ivp, 2, 8, {}),
    "burgers-p3": (lambda: _short(P.burgers_paper(), 0.02), 3, 20, {}),
    # round 2 (end): the warp sweep, the carry-level tick, the resident RIDC-2
    "febe-sweep-warp": (lambda: seg(1 << 22, 6), 1, 6, {}),
    "carry-levels-p4": (lambda: seg(1 << 19, 24), 4, 24, {}),
    "resident-res2": (lambda: seg(1 << 18, 24), 2, 24, {}),
    "febe-warp-carry": (lambda: seg(1 << 18, 20), 1, 20, {}),
}


def check(name, ivp, levels, steps, kw):
    cfg = E.RidcConfig(levels=levels, steps=steps)
    with E.Engine(ivp, cfg, **kw) as eng:
        sol = eng.run()
        path = eng.info["path_name"]
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, levels, steps, 1, dt, pack_weight_tables(levels, dt))
    err = np.abs(sol.final_state - ref["final_state"]).max() / np.abs(ref["final_state"]).max()
    print(f"{name}: path {path}, normwise err {err:.2e}", flush=True)
    assert err <= 1e-10, (name, err)


def pipe(name, resident):
    ivp = seg(steps=20)
    cfg = E.RidcConfig(levels=2, steps=20)
    sp = PD.SequentialPipeline(ivp, cfg)
    try:
        if not resident:
            for r in sp.ranks:
                pass
        fin, _ = sp.run()
    finally:
        sp.close()
    with E.Engine(ivp, cfg, tick_only=True) as eng:
        ref = eng.run().final_state
    print(f"{name}: pipeline ranks bitwise {np.array_equal(fin, ref)}", flush=True)
    assert np.array_equal(fin, ref)


def ark():
    from paper_1209_4297_b200.steppers import integrate_ark
    from paper_1209_4297_b200.tableaus import imex3_tableau
    ivp = seg(steps=4)
    tab = imex3_tableau()
    y = integrate_ark(ivp, tab, 0.0, ivp.initial_state, ivp.t_end, 4)
    ref = O.ark(ivp.problem, tab.a_implicit, tab.a_explicit, tab.b_implicit, tab.b_explicit,
                ivp.initial_state, 0.0, ivp.t_end, 4)
    err = np.abs(y - ref).max() / np.abs(ref).max()
    print(f"ark-imex3: normwise err {err:.2e}", flush=True)
    assert err <= 1e-10


def ark_carry():
    """imex4 stages on the carry-exchange tick (periodic RD, 512-point chunks)."""
    from paper_1209_4297_b200.steppers import ArkEngine
    from paper_1209_4297_b200.tableaus import imex4_tableau
    ivp = seg(1 << 17, 6)
    tab = imex4_tableau()
    with ArkEngine(ivp, tab, 0.0, ivp.t_end, 6) as eng:
        y, _ = eng.run(ivp.initial_state)
        path = eng.info["path_name"]
    ref = O.ark(ivp.problem, tab.a_implicit, tab.a_explicit, tab.b_implicit, tab.b_explicit,
                ivp.initial_state, 0.0, ivp.t_end, 6)
    err = np.abs(y - ref).max() / np.abs(ref).max()
    print(f"ark-imex4-carry: path {path}, normwise err {err:.2e}", flush=True)
    assert err <= 1e-10


def grid():
    """Levels x row shards (ridc_pipe_create_shard): 3 levels x 2 shards on one device."""
    s = P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=256, ny=20, t_end=0.002))
    cfg = E.RidcConfig(levels=3, steps=12)
    with PD.GridPipeline(s, cfg, 2, devices=[0]) as g:
        fin, _ = g.run()
    ref = E.run_serial(s, cfg).final_state
    print(f"grid-3x2: bitwise {np.array_equal(fin, ref)}", flush=True)
    assert np.array_equal(fin, ref)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(list(CASES) + ["pipe", "ark", "ark-carry", "grid"]))
    a = ap.parse_args()
    for name in a.cases.split(","):
        if name == "pipe":
            pipe("pipe-resident-p2", True)
        elif name == "ark":
            ark()
        elif name == "ark-carry":
            ark_carry()
        elif name == "grid":
            grid()
        else:
            b, levels, steps, kw = CASES[name]
            check(name, b(), levels, steps, kw)
    from paper_1209_4297_b200 import _lib
    print(f"sanitize cases done ({os.path.basename(_lib.LIB_PATH)})")


if __name__ == "__main__":
    main()
