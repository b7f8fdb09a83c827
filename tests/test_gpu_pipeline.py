"""The native one-level-per-GPU pipeline (ridc_pipe_*) on one device: all
level ranks in one process, run one after another (their inbox rings hold
the whole run, so no rank waits on one that has not started).  This drives
the real data path -- mirror peer stores into the next level's inbox,
device-side watermark / release stream ops, per-interval re-seeding -- and
must reproduce the single-device engine BITWISE (engine.py:497-503 gate)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402
from paper_1209_4297_b200.distributed import ConcurrentPipeline, SequentialPipeline  # noqa: E402

CASES = [
    ("ad-c1-p2", lambda: P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024, t_end=0.4)), 2, 100, 1),
    ("ad-c1-p4-r2", lambda: P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024, t_end=0.4)), 4, 100, 2),
    ("rd-seg-p3", lambda: P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=1 << 16, t_end=0.004)), 3, 40, 1),
    ("bu-p4", lambda: P.build_burgers(P.BurgersSpec(dx=1 / 1024, t_end=0.1)), 4, 100, 1),
    ("ad2d-p2-r2", lambda: P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=512, ny=64, t_end=0.001)), 2, 20, 2),
]


@pytest.mark.parametrize("name,builder,levels,steps,restarts", CASES, ids=[c[0] for c in CASES])
def test_pipeline_equals_engine_bitwise(name, builder, levels, steps, restarts):
    s = builder()
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, watchdog_seconds=20.0)
    ref = E.run_serial(s, cfg)
    pipe = SequentialPipeline(s, cfg)
    try:
        final, level_finals = pipe.run()
        final2, _ = pipe.run()   # counters reset between runs
    finally:
        pipe.close()
    assert np.array_equal(final, ref.final_state) and np.array_equal(final2, ref.final_state)
    for j in range(levels):
        assert np.array_equal(level_finals[j], ref.level_finals[j])


@pytest.mark.parametrize("name,builder,levels,steps,restarts", CASES, ids=[c[0] for c in CASES])
def test_concurrent_pipeline_small_rings_bitwise(name, builder, levels, steps, restarts):
    """All ranks at once, one host thread and stream each, small inbox rings
    (2L+3 slots, the memop protocol's minimum for the top consumer): the
    backpressure (release counters) and watermark waits are live, as across
    GPUs; the result must still equal the engine bitwise."""
    s = builder()
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, watchdog_seconds=30.0)
    ref = E.run_serial(s, cfg)
    pipe = ConcurrentPipeline(s, cfg, inbox_capacity=2 * levels + 3)
    try:
        assert all(r.info["ring_vectors"] < steps for r in pipe.ranks[1:])
        final, level_finals = pipe.run()
        # a second run of the same ranks: the step counters are reset between
        # runs (ridc_pipe_reset), else the last run's watermarks would satisfy
        # every wait at once
        final2, _ = pipe.run()
    finally:
        pipe.close()
    assert np.array_equal(final, ref.final_state) and np.array_equal(final2, ref.final_state)
    for j in range(levels):
        assert np.array_equal(level_finals[j], ref.level_finals[j])
