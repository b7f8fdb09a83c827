"""2-D row shards under the levels (ridc_shards_*):
S shards, each running every level on its rows plus one ghost row per side,
boundary rows of each newly written slot exchanged after every tick, must
reproduce the unsharded engine BITWISE (same x-tiling, same y-neighbour
values), incl. restarts, uneven shards and one-row shards."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402
from paper_1209_4297_b200.distributed import RowShardGroup  # noqa: E402
from paper_1209_4297_b200.errors import ConfigError  # noqa: E402

CASES = [
    ("ad2d-64x48-p1-s2", lambda: P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=64, ny=48, t_end=0.002)),
     1, 20, 1, 2),
    ("ad2d-512x37-p3-s3-r2", lambda: P.build_advection_diffusion_2d(
        P.AdvectionDiffusion2DSpec(nx=512, ny=37, t_end=0.002)), 3, 24, 2, 3),
    ("rd2d-4096x16-p4-s4", lambda: P.build_reaction_diffusion_2d(
        P.ReactionDiffusion2DSpec(nx=4096, ny=16, t_end=0.001)), 4, 20, 1, 4),
    ("rd2d-9000x8-p2-s8-rowshards", lambda: P.build_reaction_diffusion_2d(
        P.ReactionDiffusion2DSpec(nx=9000, ny=8, t_end=0.001)), 2, 10, 1, 8),
]


@pytest.mark.parametrize("name,builder,levels,steps,restarts,nshards", CASES, ids=[c[0] for c in CASES])
def test_row_shards_equal_engine_bitwise(name, builder, levels, steps, restarts, nshards):
    s = builder()
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts)
    ref = E.run_serial(s, cfg)
    with RowShardGroup(s, cfg, nshards) as g:
        final, sec = g.run()
        assert g.kernel_launches > 0
    assert sec > 0
    assert np.array_equal(final, ref.final_state)


@pytest.mark.parametrize("name,builder,levels,steps,restarts,nshards", CASES, ids=[c[0] for c in CASES])
def test_row_shards_multistream_equal_engine_bitwise(name, builder, levels, steps, restarts, nshards):
    """One stream per shard (all on device 0 here): the device-side mailbox
    protocol that runs across GPUs, with shards free to drift by a tick."""
    s = builder()
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, watchdog_seconds=30.0)
    ref = E.run_serial(s, cfg)
    with RowShardGroup(s, cfg, nshards, devices=[0]) as g:
        a, _ = g.run()
        b, sec = g.run()   # a second run: mailbox epochs, no reset
    assert sec > 0
    assert np.array_equal(a, ref.final_state) and np.array_equal(b, ref.final_state)


def test_row_shards_reject_1d_and_too_many():
    s1 = P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=1024, d=1e-3, t_end=0.01))
    with pytest.raises(ConfigError):
        RowShardGroup(s1, E.RidcConfig(levels=1, steps=10), 2)
    s2 = P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=64, ny=4, t_end=0.001))
    with pytest.raises(ConfigError):
        RowShardGroup(s2, E.RidcConfig(levels=1, steps=10), 5)
