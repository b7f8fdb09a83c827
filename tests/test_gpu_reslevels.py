"""The resident level march (csrc/ridc_levels.cuh) against the tick kernel.

RIDC order p >= 2 on a 1-D line: every level is a co-resident CTA group that
marches a whole restart interval in one launch, the lagged pipeline between
the levels driven by per-segment publish / release flags (the LevelBuffer
watermark / released protocol, engine.py:284-331) instead of one launch per
tick.  The per-chunk stencil / solve code and the node order are the tick
kernel's, so final states and every level's final must agree BITWISE with
the tick-kernel graph (RIDC_TICK_ONLY), and with the CPU oracle to 1e-10.
The same kernel, one level per launch, is the multi-GPU pipeline rank
(ridc_pipe_*): SequentialPipeline below runs it rank after rank."""

import numpy as np
import pytest

import _golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402
from paper_1209_4297_b200.distributed import SequentialPipeline  # noqa: E402
from paper_1209_4297_b200.errors import ConfigError  # noqa: E402
from paper_1209_4297_b200.quadrature import pack_weight_tables  # noqa: E402


def _short(system, t_end):
    ivp = system.ivp
    return P.StructuredIVP(ivp.problem, 0.0, t_end, ivp.initial_state)


def _c1(t_end):
    return _short(P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024)), t_end)


CASES = [
    # (id, ivp builder, levels, steps, restarts)
    ("c1-p2", lambda: _c1(0.4), 2, 100, 1),
    ("c1-p4", lambda: _c1(4.0), 4, 1000, 1),
    ("c1-p4-r10", lambda: _c1(4.0), 4, 1000, 10),
    ("c1-p8", lambda: _c1(0.4), 8, 100, 1),
    ("c1-p12", lambda: _c1(0.4), 12, 200, 1),
    ("burgers-whole-p4", lambda: _short(P.burgers_paper(), 0.1), 4, 200, 1),
    ("burgers-segments-p3", lambda: _short(P.build_burgers(P.BurgersSpec(dx=1 / (1 << 15))), 0.002), 3, 60, 1),
    ("rd-few-segments-p4", lambda: _short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=12000, d=1e-4)), 0.01),
     4, 100, 1),
    ("rd-seg-2^16-p4-r2", lambda: _short(P.reaction_diffusion_c2(n=1 << 16), 0.02), 4, 200, 2),
    ("rd-seg-2^16-p8", lambda: _short(P.reaction_diffusion_c2(n=1 << 16), 0.01), 8, 100, 1),
    ("rd-seg-2^17-p4", lambda: _short(P.reaction_diffusion_c2(n=1 << 17), 0.002), 4, 40, 1),
]


@pytest.mark.parametrize("name,builder,levels,steps,restarts", CASES, ids=[c[0] for c in CASES])
def test_resident_levels_equal_tick_kernel_bitwise(name, builder, levels, steps, restarts):
    ivp = builder()
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts)
    with E.Engine(ivp, cfg) as res, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert res.info["kernel_launches"] == 3 * restarts, res.info   # 2 seeds + 1 march per interval
        assert tick.info["kernel_launches"] > steps
        a, b = res.run(), tick.run()
        a2 = res.run()                      # fresh epoch: no flag / mailbox clearing needed
    assert np.array_equal(a.final_state, b.final_state)
    for j in range(levels):
        assert np.array_equal(a.level_finals[j], b.level_finals[j]), j
    assert np.array_equal(a.final_state, a2.final_state)
    dt = (ivp.t_end - ivp.t_start) / steps
    ref = O.run(ivp.problem, ivp.initial_state, levels, steps, restarts, dt, pack_weight_tables(levels, dt))
    # 12 levels amplify the rounding differences of any two solvers (the oracle's
    # Thomas and the reference's dense QR already differ by 1.4e-10 there:
    # _golden.tolerance); the tick kernel is bitwise this
    err = G.normwise(a.final_state, ref["final_state"])
    print(f"{name}: resident levels vs oracle {err:.3e}")
    assert err <= G.tolerance(levels)


def test_resident_levels_nonfinite_message():
    """A blow-up is reported with the reference's message (engine.py:160-164)."""
    ivp = P.build_burgers(P.BurgersSpec(dx=1 / 256, t_end=0.5))   # golden bu_n255_blowup grid
    cfg = E.RidcConfig(levels=3, steps=100)
    with E.Engine(ivp, cfg) as res, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert res.info["kernel_launches"] == 3
        msgs = []
        for eng in (res, tick):
            with pytest.raises(Exception) as ei:
                eng.run()
            msgs.append(str(ei.value))
    assert "produced non-finite entries at step" in msgs[0]
    assert msgs[0] == msgs[1]


PIPE_CASES = [
    ("c1-p4-r2", lambda: _c1(0.4), 4, 100, 2),
    ("burgers-whole-p3", lambda: _short(P.burgers_paper(), 0.1), 3, 60, 1),
    ("rd-c2-p2", lambda: _short(P.reaction_diffusion_c2(), 0.002), 2, 20, 1),
    ("rd-c2-p4-r2", lambda: _short(P.reaction_diffusion_c2(), 0.002), 4, 40, 2),
]


@pytest.mark.parametrize("name,builder,levels,steps,restarts", PIPE_CASES, ids=[c[0] for c in PIPE_CASES])
def test_resident_pipeline_ranks_bitwise(name, builder, levels, steps, restarts):
    """One level per launch, the multi-GPU rank kernel: ranks run one after
    another on this device (whole-run inboxes, so no rank waits on one that
    has not run), C2-size lines included; equal to the tick engine bitwise."""
    ivp = builder()
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, watchdog_seconds=20.0)
    with E.Engine(ivp, cfg, tick_only=True) as tick:
        ref = tick.run()
    pipe = SequentialPipeline(ivp, cfg)
    try:
        assert all(r.resident for r in pipe.ranks)
        assert all(r.kernel_launches == 2 * restarts for r in pipe.ranks)   # seed + march per interval
        assert all(r.tick_launches == restarts for r in pipe.ranks)
        final, level_finals = pipe.run()
        final2, _ = pipe.run()
    finally:
        pipe.close()
    assert np.array_equal(final, ref.final_state)
    for j in range(levels):
        assert np.array_equal(level_finals[j], ref.level_finals[j]), j
    assert np.array_equal(final2, final)


def test_pipeline_modes_must_agree():
    """The mode travels in the exported blob; neighbours that disagree are a
    configuration error, not a hang."""
    from paper_1209_4297_b200.distributed import PipelineRank
    ivp = _c1(0.4)
    cfg = E.RidcConfig(levels=2, steps=100)
    a = PipelineRank(ivp, cfg, 0, 2, 0, inbox_capacity=101, resident=True)
    b = PipelineRank(ivp, cfg, 1, 2, 0, inbox_capacity=101, resident=False)
    try:
        with pytest.raises(ConfigError):
            a.connect([a.blob, b.blob])
    finally:
        a.close()
        b.close()


def test_resident_rank_watchdog():
    """A consumer rank whose producer never publishes: the in-kernel waits give
    up after the watchdog and the rank raises PipelineProtocolError with the
    reference's message shape (engine.py:432-439) -- no hang.  Nothing else
    runs on the device, so no kernel waits on another kernel here."""
    from paper_1209_4297_b200.distributed import PipelineRank
    from paper_1209_4297_b200.errors import PipelineProtocolError
    ivp = _c1(0.4)
    cfg = E.RidcConfig(levels=2, steps=100, watchdog_seconds=0.5)
    prod = PipelineRank(ivp, cfg, 0, 2, 0)
    cons = PipelineRank(ivp, cfg, 1, 2, 0)
    try:
        assert cons.resident
        prod.connect([prod.blob, cons.blob])
        cons.connect([prod.blob, cons.blob])
        y0 = torch.from_numpy(np.array(ivp.initial_state)).cuda()
        with pytest.raises(PipelineProtocolError) as ei:
            cons.run_interval(0, y0)          # level 1 alone: level 0 never runs
        assert "made no progress" in str(ei.value)
    finally:
        prod.close()
        cons.close()


@pytest.mark.parametrize("levels,pub_every", [(4, 4), (8, 1), (8, 7)])
def test_resident_levels_tight_inboxes(monkeypatch, levels, pub_every):
    """Inbox rings at the minimum (levels + 2 slots): producers block on their
    consumers' release counters nearly every step, and must publish their
    pending steps before blocking (batched publication would otherwise
    deadlock).  Still bitwise the tick kernel."""
    monkeypatch.setenv("RIDC_LEVEL_INBOX", "1")          # clamped up to levels + 2
    monkeypatch.setenv("RIDC_PUB_EVERY", str(pub_every))
    ivp = _short(P.reaction_diffusion_c2(n=1 << 15), 0.02)
    cfg = E.RidcConfig(levels=levels, steps=200, restarts=2, watchdog_seconds=20.0)
    with E.Engine(ivp, cfg) as res, E.Engine(ivp, cfg, tick_only=True) as tick:
        assert res.info["kernel_launches"] == 3 * 2
        assert res.info["ring_vectors"] < tick.info["ring_vectors"] + 16 * (levels - 1)
        a, b = res.run(), tick.run()
    assert np.array_equal(a.final_state, b.final_state)
    for j in range(levels):
        assert np.array_equal(a.level_finals[j], b.level_finals[j]), j
