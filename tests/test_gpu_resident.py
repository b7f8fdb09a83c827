"""The resident single-level marches against the tick kernel: RIDC order 1
(FEBE, engine.py:167-175) on 1-D lines.  The halo-exchange march
(csrc/ridc_resident.cuh) gives bitwise the same final state, level finals and
trajectory as the tick kernel -- both call the same per-chunk stencil/solve
code, only the data movement differs (registers + published segment edges vs
TMA-staged ring slots).  On periodic reaction-diffusion lines the
carry-exchange march (csrc/ridc_febe_carry.cuh) solves each tile without halos
and couples the tiles by two carries per step: the same solve to rounding
(<= 1e-13 against the tick kernel) and <= 1e-10 against the oracle."""

import numpy as np
import pytest

import _golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402
from paper_1209_4297_b200.errors import NonFiniteStateError  # noqa: E402
from paper_1209_4297_b200.quadrature import pack_weight_tables  # noqa: E402


def _short(system, t_end):
    ivp = system.ivp
    return P.StructuredIVP(ivp.problem, 0.0, t_end, ivp.initial_state)


CASES = [
    # (id, ivp builder, steps, restarts, trajectory)
    ("c1-whole-cyclic", lambda: _short(P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024)), 4.0),
     1000, 1, False),
    ("c1-restarts-traj", lambda: _short(P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024)), 0.4),
     120, 3, True),
    ("burgers-whole-dirichlet", lambda: _short(P.burgers_paper(), 0.1), 200, 1, False),
    ("burgers-segments", lambda: _short(P.build_burgers(P.BurgersSpec(dx=1 / (1 << 15))), 0.002), 100, 1, False),
    ("rd-few-segments", lambda: _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=12000, d=1e-4)), 0.01),
     100, 1, False),
    ("rd-seg-2^16", lambda: _short(P.reaction_diffusion_c2(n=1 << 16), 0.02), 200, 2, False),
    ("rd-c2-2^20", lambda: _short(P.reaction_diffusion_c2(), 0.02), 200, 1, False),
    ("rd-c2-traj", lambda: _short(P.reaction_diffusion_c2(n=1 << 18), 0.002), 20, 2, True),
]


@pytest.mark.parametrize("name,builder,steps,restarts,traj", CASES, ids=[c[0] for c in CASES])
def test_resident_equals_tick_kernel_bitwise(name, builder, steps, restarts, traj):
    ivp = builder()
    cfg = E.RidcConfig(levels=1, steps=steps, restarts=restarts, record_trajectory=traj)
    with E.Engine(ivp, cfg, resident_segments=True) as res, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert res.info["kernel_launches"] == 2, res.info          # seed + one cooperative march
        assert tick.info["kernel_launches"] == restarts + restarts * steps // restarts
        a, b = res.run(), tick.run()
        a2 = res.run()
        path = res.info["path_name"]
        assert path in ("resident_febe", "carry_febe", "warp_carry_febe") and tick.info["path_name"] == "tick"
        if ivp.problem.kind == P.KIND_REACTION_DIFFUSION_1D and res.info["items_per_level"] > 1:
            # lines of 512-point chunks: one chunk per warp; other RD lines: one tile per SM
            want = "warp_carry_febe" if ivp.dimension % 512 == 0 else "carry_febe"
            assert path == want, res.info
    assert np.array_equal(a.final_state, a2.final_state)
    if path in ("carry_febe", "warp_carry_febe"):
        # periodic RD lines: tiles exchange carries instead of halos -- the same
        # solve to rounding (the tick kernel truncates at lam^H <= 2^-60)
        assert G.normwise(a.final_state, b.final_state) <= 1e-13
        assert G.normwise(a.level_finals[0], b.level_finals[0]) <= 1e-13
        if traj:
            assert G.normwise(a.trajectory, b.trajectory) <= 1e-13
    else:
        assert np.array_equal(a.final_state, b.final_state)
        assert np.array_equal(a.level_finals[0], b.level_finals[0])
        if traj:
            assert np.array_equal(a.trajectory, b.trajectory)
    # and the oracle (the reference's algebra restated on the CPU)
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, 1, steps, restarts, dt, pack_weight_tables(1, dt))
    assert G.normwise(a.final_state, ref["final_state"]) <= 1e-10


def test_default_selection():
    """Single-level runs on 1-D lines march resident (whole lines and segmented
    lines); RIDC-2 on RD lines holds both levels per tile (one launch per
    interval); other multi-level runs on short 1-D lines use the resident
    level march (two seeds + one launch per interval, tests/test_gpu_reslevels.py)."""
    whole = _short(P.reaction_diffusion_c2(n=8192), 0.002)
    seg = _short(P.reaction_diffusion_c2(n=1 << 16), 0.002)
    with E.Engine(whole, E.RidcConfig(levels=1, steps=20)) as a, \
            E.Engine(seg, E.RidcConfig(levels=1, steps=20)) as b, \
            E.Engine(whole, E.RidcConfig(levels=2, steps=20)) as c, \
            E.Engine(whole, E.RidcConfig(levels=3, steps=20)) as d:
        assert a.info["kernel_launches"] == 2
        assert b.info["kernel_launches"] == 2
        assert c.info["path_name"] == "resident_carry_levels" and c.info["kernel_launches"] == 1
        assert d.info["path_name"] == "resident_levels" and d.info["kernel_launches"] == 3


def test_resident_device_run_and_wall():
    ivp = _short(P.reaction_diffusion_c2(n=1 << 16), 0.02)
    cfg = E.RidcConfig(levels=1, steps=200)
    y0 = torch.from_numpy(np.array(ivp.initial_state)).cuda()
    out = torch.empty_like(y0)
    with E.Engine(ivp, cfg, resident_segments=True) as eng:
        t = eng.run_device(y0, out)
        host = eng.run().final_state
    assert t > 0
    assert np.array_equal(out.cpu().numpy(), host)


SWEEP_CASES = [
    # (id, n, steps, restarts, trajectory): r ~ 110 as C2 (carry reach 438 < 512)
    ("2^21", 1 << 21, 30, 1, False),
    ("2^21-restarts-traj", 1 << 21, 24, 3, True),
    ("uneven-ranges", (1 << 21) + 16 * 1235, 20, 1, False),
    ("2^23", 1 << 23, 12, 1, False),
]


@pytest.mark.parametrize("variant", ["warp", "cta"])
@pytest.mark.parametrize("name,n,steps,restarts,traj", SWEEP_CASES, ids=[c[0] for c in SWEEP_CASES])
def test_sweep_febe_long_lines(name, n, steps, restarts, traj, variant, monkeypatch):
    """Lines too long to stay resident: the streaming sweeps (one launch per step;
    every warp sweeps a contiguous range, csrc/ridc_sweep_warp.cuh, or every
    SM, csrc/ridc_sweep.cuh with RIDC_SWEEP_CTA=1) against the tick kernel
    (<= 1e-13: same solve, different association) and the oracle."""
    if variant == "cta":
        monkeypatch.setenv("RIDC_SWEEP_CTA", "1")
    # lines the warp-chunk march holds (up to 14 x 148 x 1024 points) would take it
    monkeypatch.setenv("RIDC_NO_WCARRY", "1")
    ivp = _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)),
                 1e-4 * steps)
    cfg = E.RidcConfig(levels=1, steps=steps, restarts=restarts, record_trajectory=traj)
    with E.Engine(ivp, cfg) as sw, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert sw.info["path_name"] == {"warp": "sweep_warp_febe", "cta": "sweep_febe"}[variant], sw.info
        a, b = sw.run(), tick.run()
        a2 = sw.run()
    assert np.array_equal(a.final_state, a2.final_state)
    assert G.normwise(a.final_state, b.final_state) <= 1e-13
    if traj:
        assert G.normwise(a.trajectory, b.trajectory) <= 1e-13
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, 1, steps, restarts, dt, pack_weight_tables(1, dt))
    assert G.normwise(a.final_state, ref["final_state"]) <= 1e-10


LEVEL_SWEEP_CASES = [
    # (id, n, levels, steps, restarts): r ~ 110 as C2; at least three chunks per SM
    ("2^22-p2", 1 << 22, 2, 20, 1),
    ("2^22-p4-r2", 1 << 22, 4, 48, 2),
    ("2^22-p8", 1 << 22, 8, 40, 1),
    ("uneven-p3", (1 << 22) + 16 * 777, 3, 16, 1),
]


@pytest.mark.parametrize("name,n,levels,steps,restarts", LEVEL_SWEEP_CASES, ids=[c[0] for c in LEVEL_SWEEP_CASES])
def test_sweep_levels_long_lines(name, n, levels, steps, restarts):
    """RIDC p >= 2 on lines the resident level march cannot hold: every SM sweeps
    its range for each active level per tick (csrc/ridc_sweep_levels.cuh), every
    level's final against the tick kernel (<= 1e-12) and the oracle."""
    ivp = _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)),
                 1e-4 * steps)
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts)
    with E.Engine(ivp, cfg) as sw, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert sw.info["path_name"] == "sweep_levels", sw.info
        a, b = sw.run(), tick.run()
        a2 = sw.run()
    assert np.array_equal(a.final_state, a2.final_state)
    for j in range(levels):
        assert G.normwise(a.level_finals[j], b.level_finals[j]) <= 1e-12, j
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, levels, steps, restarts, dt, pack_weight_tables(levels, dt),
                level_finals=True)
    for j in range(levels):
        assert G.normwise(a.level_finals[j], ref["level_finals"][j]) <= 1e-10, j


CARRY_LEVEL_CASES = [
    # (id, n, levels, steps, restarts, trajectory): r ~ 110 as C2; one 512-point chunk per warp
    ("c2-p2", 1 << 20, 2, 24, 1, False),
    ("c2-p4-r2", 1 << 20, 4, 32, 2, False),
    ("c2-p3-traj", 1 << 20, 3, 20, 1, True),
    ("2^17-p8", 1 << 17, 8, 40, 1, False),
    ("uneven-p4", 512 * 1000, 4, 24, 1, False),
    ("2^18-p12", 1 << 18, 12, 80, 1, False),
]


@pytest.mark.parametrize("name,n,levels,steps,restarts,traj", CARRY_LEVEL_CASES,
                         ids=[c[0] for c in CARRY_LEVEL_CASES])
def test_carry_levels(name, n, levels, steps, restarts, traj):
    """RIDC p >= 2 on lines of 512-point chunks, one chunk per warp, the chunks'
    solves coupled by two exchanged carries (csrc/ridc_carry_levels.cuh):
    repeat runs bitwise, every level's final against the tick kernel (<= 1e-12:
    the same solve, different association) and the oracle (<= 1e-10)."""
    ivp = _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)),
                 1e-4 * steps)
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, record_trajectory=traj)
    with E.Engine(ivp, cfg) as cl, E.Engine(ivp, cfg, tick_only=True) as tick:
        # RIDC-2 without a recorded trajectory holds both levels on the SMs (ridc_carry_res2.cuh)
        want = "resident_carry_levels" if levels == 2 and not traj else "carry_levels"
        assert cl.info["path_name"] == want, cl.info
        a, b = cl.run(), tick.run()
        a2 = cl.run()
    assert np.array_equal(a.final_state, a2.final_state)
    for j in range(levels):
        assert np.array_equal(a.level_finals[j], a2.level_finals[j]), j
        # 12 levels amplify last-bit differences: tick vs this kernel 5e-12, the
        # two CPU codes 1.4e-10
        assert G.normwise(a.level_finals[j], b.level_finals[j]) <= (1e-10 if levels > 8 else 1e-12), j
    if traj:
        assert G.normwise(a.trajectory, b.trajectory) <= 1e-12
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, levels, steps, restarts, dt, pack_weight_tables(levels, dt),
                level_finals=True)
    bar = 5e-10 if levels > 8 else 1e-10
    for j in range(levels):
        assert G.normwise(a.level_finals[j], ref["level_finals"][j]) <= bar, j


def test_carry_levels_watchdog_recapture():
    """ridc_set_watchdog re-captures the carry-level graph (the limit is a kernel
    parameter of every tick): the run after it is unchanged."""
    ivp = _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=1 << 18, d=1e-6 * 16.0)), 1e-4 * 12)
    cfg = E.RidcConfig(levels=3, steps=12, watchdog_seconds=5.0)
    with E.Engine(ivp, cfg) as cl:
        assert cl.info["path_name"] == "carry_levels", cl.info
        a = cl.run()
        from paper_1209_4297_b200 import _lib
        _lib.check(_lib.lib().ridc_set_watchdog(cl._h, 11.0), cl._h)
        b = cl.run()
    assert np.array_equal(a.final_state, b.final_state)


RES2_CASES = [
    # (id, n, steps, restarts): r ~ 110 as C2
    ("c2", 1 << 20, 40, 1),
    ("c2-r4", 1 << 20, 48, 4),
    ("2^18", 1 << 18, 30, 1),
    ("uneven-tiles", (1 << 20) - 16 * 999, 30, 2),   # not whole 512-point chunks: the tile kernel
    ("two-ctas", 512 * 9, 30, 1),                     # warp chunks: a full and a 2-warp CTA
]


@pytest.mark.parametrize("name,n,steps,restarts", RES2_CASES, ids=[c[0] for c in RES2_CASES])
def test_resident_carry_res2(name, n, steps, restarts):
    """RIDC-2 with both levels held on the SMs for a whole interval: one
    512-point chunk per warp where the line divides (csrc/ridc_carry_res2w.cuh),
    else one tile per SM (ridc_carry_res2.cuh), coupled by carries and the
    predictor's end points: repeat runs bitwise, both level finals against the
    tick kernel (<= 1e-12) and the oracle (<= 1e-10)."""
    ivp = _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)),
                 1e-4 * steps)
    cfg = E.RidcConfig(levels=2, steps=steps, restarts=restarts)
    with E.Engine(ivp, cfg) as cr, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert cr.info["path_name"] == "resident_carry_levels", cr.info
        a, b = cr.run(), tick.run()
        a2 = cr.run()
    for j in range(2):
        assert np.array_equal(a.level_finals[j], a2.level_finals[j]), j
        assert G.normwise(a.level_finals[j], b.level_finals[j]) <= 1e-12, j
    assert np.array_equal(a.final_state, a.level_finals[1])
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, 2, steps, restarts, dt, pack_weight_tables(2, dt),
                level_finals=True)
    for j in range(2):
        assert G.normwise(a.level_finals[j], ref["level_finals"][j]) <= 1e-10, j


def test_resident_carry_res2_nonfinite_message():
    """A blow-up inside the resident RIDC-2 march reports the reference's
    message with the first non-finite (step, level), the same as the tick
    kernel's (engine.py:160-164)."""
    n = 1 << 18
    spec = P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)
    sysm = P.build_reaction_diffusion(spec)
    y0 = np.array(sysm.ivp.initial_state) * 1e150   # the logistic term overflows within a few steps
    ivp = P.StructuredIVP(sysm.ivp.problem, 0.0, 1e-4 * 20, y0)
    msgs = []
    for tick_only in (False, True):   # the same first (step, level) as the tick kernel reports
        with E.Engine(ivp, E.RidcConfig(levels=2, steps=20), tick_only=tick_only) as eng:
            assert (eng.info["path_name"] == "resident_carry_levels") != tick_only, eng.info
            with pytest.raises(NonFiniteStateError, match=r"level \d produced non-finite entries at step \d+") as ei:
                eng.run()
            msgs.append(str(ei.value))
    assert msgs[0] == msgs[1], msgs


@pytest.mark.parametrize("n,steps,restarts,traj", [(1 << 20, 200, 1, False), (1 << 18, 40, 2, True),
                                                    (512 * 1000, 60, 1, False), (1 << 16, 100, 1, False),
                                                    (1 << 21, 60, 1, False), (1024 * 1500, 40, 2, True)])
def test_warp_carry_vs_tile_carry(n, steps, restarts, traj, monkeypatch):
    """The warp-chunk march (k_febe_wcarry: a 512- or 1024-point chunk per warp,
    carries through shared memory inside a CTA) against the tile march
    (k_febe_carry, RIDC_NO_WCARRY=1; the tick kernel beyond its lines) and the
    oracle: the same solve to rounding."""
    ivp = _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)),
                 1e-4 * steps)
    cfg = E.RidcConfig(levels=1, steps=steps, restarts=restarts, record_trajectory=traj)
    with E.Engine(ivp, cfg) as w:
        assert w.info["path_name"] == "warp_carry_febe", w.info
        # 16 points per lane where 512-point chunks fit 14 warps per SM, else 32
        assert w.info["tile"] == (512 if n <= 14 * 148 * 512 else 1024), w.info
        a, a2 = w.run(), w.run()
    monkeypatch.setenv("RIDC_NO_WCARRY", "1")
    with E.Engine(ivp, cfg, tick_only=n > 148 * 8192) as t:   # longer lines than the tile march holds: the tick kernel
        assert t.info["path_name"] in ("carry_febe", "tick"), t.info
        b = t.run()
    assert np.array_equal(a.final_state, a2.final_state)
    assert G.normwise(a.final_state, b.final_state) <= 1e-13
    if traj:
        assert G.normwise(a.trajectory, b.trajectory) <= 1e-13
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, 1, steps, restarts, dt, pack_weight_tables(1, dt))
    assert G.normwise(a.final_state, ref["final_state"]) <= 1e-10


@pytest.mark.parametrize("levels,steps", [(3, 24), (4, 30)])
def test_carry_levels_1024_point_chunks(levels, steps):
    """A stiffer C2 line (r ~ 220: carry reach 618 > 512) runs the carry-level
    tick with 1024-point chunks (32 points per lane, csrc/ridc_carry_levels.cuh):
    against the tick kernel (<= 1e-12) and the oracle (<= 1e-10)."""
    n = 1 << 20
    ivp = _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=2e-6)), 1e-4 * steps)
    cfg = E.RidcConfig(levels=levels, steps=steps)
    with E.Engine(ivp, cfg) as cl, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert cl.info["path_name"] == "carry_levels", cl.info
        assert cl.info["r"] > 200, cl.info
        a, b = cl.run(), tick.run()
        a2 = cl.run()
    for j in range(levels):
        assert np.array_equal(a.level_finals[j], a2.level_finals[j]), j
        assert G.normwise(a.level_finals[j], b.level_finals[j]) <= 1e-12, j
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, levels, steps, 1, dt, pack_weight_tables(levels, dt),
                level_finals=True)
    for j in range(levels):
        assert G.normwise(a.level_finals[j], ref["level_finals"][j]) <= 1e-10, j
