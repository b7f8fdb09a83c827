"""The one-level-per-GPU pipeline across PROCESSES (torchrun's layout: one
process per rank), run here with every rank on cuda:0 so that it executes on
a one-GPU box: each rank exports its mailbox with cudaIpcGetMemHandle, its
neighbours open it with cudaIpcOpenMemHandle (csrc/ridc_engine.cu open_blob),
the tick kernels peer-store into the consumer's IPC-mapped inbox and the
stream memory operations carry the watermark / release counters between the
processes' CUDA contexts.  The re-seed broadcast runs over gloo (NCCL refuses
two ranks on one device).  Ranks sharing a device use the stream-memop path
(resident=False): no kernel spins on another process's kernel.

Each result must equal the single-device engine bitwise (the tiling depends
only on the problem and dt)."""

import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1209_4297_b200 import engine as E, problems as P  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _system(name):
    if name == "c1":
        s = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024, t_end=0.4))
        return s.ivp
    if name == "burgers":
        s = P.burgers_paper()
        ivp = s.ivp
        return P.StructuredIVP(ivp.problem, 0.0, 0.1, ivp.initial_state)
    if name == "ad2d":
        return P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=512, ny=64, t_end=0.002)).ivp
    if name == "rd-seg":
        s = P.reaction_diffusion_c2(n=1 << 16)
        ivp = s.ivp
        return P.StructuredIVP(ivp.problem, 0.0, 0.004, ivp.initial_state)
    raise ValueError(name)


def _worker(rank, world, port, name, levels, steps, restarts, outdir):
    import torch.distributed as dist
    from paper_1209_4297_b200 import distributed as PD
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ivp = _system(name)
        cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts, watchdog_seconds=60.0)

        def exchange(blob):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out

        def bcast(x, is_top):   # the top level's interval final -> every rank (gloo, host copy)
            h = x.detach().cpu().clone()
            dist.broadcast(h, src=world - 1)
            return h.cuda()

        rk = PD.PipelineRank(ivp, cfg, rank, world, 0, exchange=exchange, resident=False)
        assert not rk.resident
        y0 = torch.from_numpy(np.array(ivp.initial_state)).cuda()
        out = torch.empty_like(y0)
        sec = rk.run_device(y0, out, broadcast=bcast)
        np.save(os.path.join(outdir, f"rank{rank}.npy"), out.cpu().numpy())
        # a second run: every rank resets its step counters between two barriers
        out2 = torch.empty_like(y0)
        rk.run_device(y0, out2, broadcast=bcast)
        np.save(os.path.join(outdir, f"rank{rank}_2.npy"), out2.cpu().numpy())
        np.save(os.path.join(outdir, f"sec{rank}.npy"), np.array([sec]))
        dist.barrier()
        rk.close()
    finally:
        dist.destroy_process_group()


CASES = [
    ("c1", 2, 100, 2),
    ("c1", 4, 60, 1),
    ("burgers", 3, 60, 1),
    ("ad2d", 3, 30, 2),
    ("rd-seg", 2, 40, 1),
]


@pytest.mark.parametrize("name,levels,steps,restarts", CASES,
                         ids=[f"{c[0]}-p{c[1]}-r{c[3]}" for c in CASES])
def test_pipeline_ranks_as_processes_bitwise(name, levels, steps, restarts):
    import torch.multiprocessing as mp
    ivp = _system(name)
    cfg = E.RidcConfig(levels=levels, steps=steps, restarts=restarts)
    with E.Engine(ivp, cfg, tick_only=True) as eng:
        ref = eng.run().final_state
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(_worker, args=(levels, _free_port(), name, levels, steps, restarts, td),
                           nprocs=levels, join=True, start_method="spawn")
        outs = [np.load(os.path.join(td, f"rank{r}.npy")) for r in range(levels)]
        outs2 = [np.load(os.path.join(td, f"rank{r}_2.npy")) for r in range(levels)]
    for r in range(levels):   # every rank holds the solution (the re-seed broadcast of the last interval)
        assert np.array_equal(outs[r], ref), (r, np.abs(outs[r] - ref).max())
        assert np.array_equal(outs2[r], ref), (r, "second run", np.abs(outs2[r] - ref).max())
