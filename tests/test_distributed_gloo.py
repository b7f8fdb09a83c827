"""The one-level-per-rank pipeline protocol on CPU (gloo, world_size 2-4):
the product's interval driver + oracle level ranks must reproduce the serial
oracle run BITWISE -- the reference's serial == pipelined gate
(engine.py:497-503) across processes."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, outdir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from _oracle_pipeline import OracleLevel, gloo_broadcast
    from paper_1209_4297_b200 import problems as P
    from paper_1209_4297_b200.distributed import run_levels
    sysm = case["system"]()
    ivp = sysm.ivp
    dt = (ivp.t_end - ivp.t_start) / case["steps"]
    lvl = OracleLevel(ivp.problem, world, case["steps"], case["restarts"], dt, rank, world)
    fin, sol, _ = run_levels(lvl, case["restarts"], ivp.initial_state, gloo_broadcast(world),
                             rank == world - 1)
    np.save(os.path.join(outdir, f"level{rank}.npy"), fin)
    np.save(os.path.join(outdir, f"sol{rank}.npy"), sol)
    dist.destroy_process_group()


def _ad():
    from paper_1209_4297_b200 import problems as P
    return P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 128, t_end=0.5))


def _bu():
    from paper_1209_4297_b200 import problems as P
    return P.build_burgers(P.BurgersSpec(dx=1 / 256, t_end=0.5))


def _rd2():
    from paper_1209_4297_b200 import problems as P
    return P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=32, ny=16, t_end=0.05, dxx=1e-2, dyy=1e-3))


CASES = [
    (2, dict(system=_ad, steps=40, restarts=1)),
    (3, dict(system=_bu, steps=400, restarts=2)),
    (4, dict(system=_ad, steps=60, restarts=2)),
    (3, dict(system=_rd2, steps=24, restarts=1)),
]


@pytest.mark.parametrize("world,case", CASES, ids=["ad-w2", "bu-w3-r2", "ad-w4-r2", "rd2d-w3"])
def test_pipeline_protocol_bitwise(world, case, tmp_path):
    from oracle import oracle as O
    from paper_1209_4297_b200.quadrature import pack_weight_tables
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, str(tmp_path)), nprocs=world, join=True)
    sysm = case["system"]()
    ivp = sysm.ivp
    dt = (ivp.t_end - ivp.t_start) / case["steps"]
    ref = O.run(ivp.problem, ivp.initial_state, world, case["steps"], case["restarts"], dt,
                pack_weight_tables(world, dt), level_finals=True)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"sol{r}.npy"), ref["final_state"])
        assert np.array_equal(np.load(tmp_path / f"level{r}.npy"), ref["level_finals"][r])
