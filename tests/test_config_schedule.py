"""Host logic: RidcConfig validation, restart partition, the device tick
schedule and its ring-buffer capacities (engine.py:50-118)."""

import pytest

from paper_1209_4297_b200 import engine as E
from paper_1209_4297_b200.errors import ConfigError
from paper_1209_4297_b200.studies import scheme_levels


def test_startup_delay():
    assert [E.startup_delay(j) for j in range(6)] == [0, 1, 3, 6, 10, 15]
    with pytest.raises(ValueError):
        E.startup_delay(-1)


@pytest.mark.parametrize("kw", [
    dict(levels=0, steps=10), dict(levels=13, steps=1000), dict(levels=2, steps=0),
    dict(levels=2, steps=10, restarts=3), dict(levels=4, steps=40, restarts=4),
    dict(levels=2, steps=10, workers=3), dict(levels=2, steps=10, workers=0),
])
def test_config_rejects(kw):
    with pytest.raises(ConfigError):
        E.RidcConfig(**kw)


def test_config_fill_guard():
    E.RidcConfig(levels=4, steps=11)          # 4*5/2 + 1 = 11
    with pytest.raises(ConfigError):
        E.RidcConfig(levels=4, steps=10)


def test_restart_partition():
    parts = E.restart_partition(0.0, 40.0, 10, 4000)
    assert len(parts) == 10 and all(p[2] == 400 for p in parts)
    assert parts[3][0] == pytest.approx(12.0) and parts[-1][1] == 40.0
    assert E.restart_partition(0.0, 1.0, 4, 100)[1][2] == 25
    with pytest.raises(ConfigError):
        E.restart_partition(0.0, 1.0, 3, 100)


@pytest.mark.parametrize("levels", [1, 2, 4, 8, 12])
def test_schedule_finish_tick(levels):
    per = 100
    sch = E.schedule(levels, per)
    assert sch[-1][0] == per + levels * (levels - 1) // 2
    done = {}
    for _k, act in sch:
        for j, t in act:
            assert done.get(j, 0) == t - 1                       # consecutive steps
            done[j] = t
    assert all(done[j] == per for j in range(levels))


@pytest.mark.parametrize("levels", [2, 3, 4, 8, 12])
def test_schedule_dependencies_and_ring_capacity(levels):
    """Simulate the device rings (capacity 2j+3, top 2) slot by slot: every
    read must see exactly the step the algebra needs, and no write may
    clobber a slot still needed in the same or a later tick."""
    per = 3 * levels * levels + 7
    cap = [2 * j + 3 for j in range(levels - 1)] + [2]
    ring = [[None] * c for c in cap]
    for j in range(levels):
        ring[j][0] = 0                                         # seed: step 0 everywhere
    for _k, act in E.schedule(levels, per):
        writes = []
        for j, t in act:
            assert ring[j][(t - 1) % cap[j]] == t - 1            # own previous state
            if j > 0:
                nodes = range(t - j, t + 1) if t >= j else range(0, j + 1)
                for s in nodes:
                    assert ring[j - 1][s % cap[j - 1]] == s, (j, t, s)
            writes.append((j, t))
        for j, t in writes:                                    # all reads of a tick precede writes
            ring[j][t % cap[j]] = t


def test_scheme_levels():
    assert scheme_levels("fbe") == 1 and scheme_levels("ridc4-fbe") == 4
    assert scheme_levels("ridc-8") == 8 and scheme_levels("imex4") is None
    for bad in ("ridc-1", "ridc-13", "rk4"):
        with pytest.raises(ConfigError):
            scheme_levels(bad)
