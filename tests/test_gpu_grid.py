"""Levels x row shards: rank (j, s) computes level j on
row shard s of a 2-D grid (ridc_pipe_create_shard), fed by (j-1, s) plus the
ghost rows of (j-1, s-+1), its own ghost rows from (j, s-+1), every exchange a
watermark / release pair in device memory (the reference's LevelBuffer
protocol, engine.py:284-331, per neighbour).  Here all ranks share device 0
(one host thread + stream each, stream-memory waits only); the grid must
reproduce the single-device engine BITWISE: same x-tiling, same
y-neighbour values, same per-row arithmetic."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402
from paper_1209_4297_b200.distributed import GridPipeline, ShardRank  # noqa: E402
from paper_1209_4297_b200.errors import ConfigError  # noqa: E402

CASES = [
    # (id, builder, levels, steps, restarts, shards, inbox)
    ("ad2d-64x24-p2-s2", lambda: P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=64, ny=24, t_end=0.002)),
     2, 16, 1, 2, 0),
    ("ad2d-512x37-p3-s3-r2", lambda: P.build_advection_diffusion_2d(
        P.AdvectionDiffusion2DSpec(nx=512, ny=37, t_end=0.002)), 3, 24, 2, 3, 0),
    ("rd2d-2048x16-p4-s2-tight", lambda: P.build_reaction_diffusion_2d(
        P.ReactionDiffusion2DSpec(nx=2048, ny=16, t_end=0.001)), 4, 24, 1, 2, 7),
    ("rd2d-256x12-p2-s4", lambda: P.build_reaction_diffusion_2d(
        P.ReactionDiffusion2DSpec(nx=256, ny=12, t_end=0.001)), 2, 12, 1, 4, 0),
]


@pytest.mark.parametrize("name,builder,levels,steps,restarts,nshards,inbox", CASES, ids=[c[0] for c in CASES])
def test_levels_x_shards_equal_engine_bitwise(name, builder, levels, steps, restarts, nshards, inbox):
    s = builder()
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, watchdog_seconds=30.0)
    ref = E.run_serial(s, cfg)
    with GridPipeline(s, cfg, nshards, devices=[0], inbox_capacity=inbox) as g:
        a, lev_a = g.run()
        b, _ = g.run()   # a second run: the counters carry global step numbers, nothing is reset
        assert g.device_seconds > 0
    assert np.array_equal(a, ref.final_state) and np.array_equal(b, ref.final_state)
    for j in range(levels):
        assert np.array_equal(lev_a[j], ref.level_finals[j]), j


def test_levels_x_shards_rejects_1d():
    s1 = P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=1024, d=1e-3, t_end=0.01))
    cfg = E.RidcConfig(levels=2, steps=10)
    with pytest.raises(ConfigError):
        ShardRank(s1, cfg, 0, 0, 2)
    s2 = P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=64, ny=4, t_end=0.001))
    with pytest.raises(ConfigError):
        ShardRank(s2, cfg, 0, 0, 5)   # more shards than rows
