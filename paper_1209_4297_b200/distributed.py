"""One RIDC level per GPU: the lagged pipeline across devices and processes.

The reference runs levels as threads sharing ``LevelBuffer`` rings
(engine.py:284-459); here level j runs on GPU j in its own process
(``torchrun``, one rank per GPU).  ``PipelineRank`` wraps the native rank
(``ridc_pipe_*`` in include/ridc_b200.h): each tick kernel stores its new
state tile into the next level's inbox over NVLink (peer stores through an
IPC-mapped mailbox), and device-side stream waits/writes carry the
watermark / release counters -- the levels form a point-to-point chain, so
there is no collective on the data path.  The only collective is the restart
re-seed (engine.py:511-514): the top level's interval final is broadcast to
every level.

``run_levels`` is the driver both backends share: the GPU ranks below and
the CPU oracle ranks of tests/_oracle_pipeline.py (gloo), so the interval /
re-seed protocol is tested on CPU with world_size > 1.
"""

import ctypes
import os
from typing import Callable, Optional

import numpy as np

from . import _lib, device as D
from .errors import ConfigError
from .problems import as_descriptor
from .quadrature import pack_weight_tables

__all__ = ["PipelineRank", "SequentialPipeline", "ConcurrentPipeline", "ShardRank", "GridPipeline", "run_levels",
           "run_pipelined_distributed"]


def run_levels(runner, restarts: int, state0, broadcast: Callable, is_top: bool):
    """Interval loop of run_pipelined (engine.py:509-515) for ONE level.

    runner.run_interval(r, state0) -> (final_of_this_level, seconds);
    broadcast(x, is_top) returns the top level's x on every rank.
    Returns (this level's final state of the last interval, the solution on
    every rank, total seconds).
    """
    s0 = state0
    total = 0.0
    fin = None
    for r in range(restarts):
        fin, sec = runner.run_interval(r, s0)
        total += sec
        s0 = broadcast(fin, is_top)   # next interval's state0 = top level's final
    return fin, s0, total


class PipelineRank:
    """The level this process owns, on its GPU.

    ``exchange(blob) -> list of blobs`` gathers every rank's mailbox handle
    (default: torch.distributed.all_gather_object).
    """

    def __init__(self, ivp, config, rank: int, world: int, device: int = 0,
                 inbox_capacity: int = 0, exchange: Optional[Callable] = None,
                 resident: bool = True):
        if config.levels != world:
            raise ConfigError(f"one level per GPU: levels ({config.levels}) must equal ranks ({world})")
        self.ivp = as_descriptor(ivp)
        self.config = config
        self.rank, self.world, self.device = rank, world, device
        self.problem = self.ivp.problem
        self.dt = (self.ivp.t_end - self.ivp.t_start) / config.steps
        self.weights = pack_weight_tables(config.levels, self.dt)
        D.require_cuda(device)
        cp = self.problem.to_c()
        h = ctypes.c_void_p()
        _lib.check_pipe(_lib.lib().ridc_pipe_create(
            ctypes.byref(cp), float(self.ivp.t_start), float(self.ivp.t_end), config.levels,
            config.steps, config.restarts, self.weights.ctypes.data, self.weights.shape[0],
            rank, device, int(inbox_capacity), float(config.watchdog_seconds), ctypes.byref(h)))
        self._h = h
        self._runs = 0
        # resident level march (one launch per interval, in-kernel flag waits)
        # where the line qualifies; every rank must choose the same (the blob
        # carries it and connect checks it)
        _lib.check_pipe(_lib.lib().ridc_pipe_set_resident(self._h, 1 if resident else 0), self._h)
        nb = _lib.lib().ridc_pipe_handle_bytes()
        blob = ctypes.create_string_buffer(nb)
        _lib.check_pipe(_lib.lib().ridc_pipe_export(self._h, blob), self._h)
        self.blob = bytes(blob.raw)
        if exchange is not None:
            blobs = exchange(self.blob)
            self.connect(blobs)

    def connect(self, blobs):
        prev = blobs[self.rank - 1] if self.rank > 0 else None
        nxt = blobs[self.rank + 1] if self.rank < self.world - 1 else None
        _lib.check_pipe(_lib.lib().ridc_pipe_connect(self._h, prev, nxt), self._h)

    @property
    def info(self) -> dict:
        inf = _lib.RidcInfo()
        _lib.check_pipe(_lib.lib().ridc_pipe_info(self._h, ctypes.byref(inf)), self._h)
        return {f: getattr(inf, f) for f, _ in inf._fields_}

    @property
    def resident(self) -> bool:
        return bool(_lib.lib().ridc_pipe_resident(self._h))

    @property
    def kernel_launches(self) -> int:
        """Our kernels per run: per interval the seed, then one resident march
        launch or one tick kernel per step."""
        return self.config.restarts + (self.config.restarts if self.resident else self.config.steps)

    @property
    def tick_launches(self) -> int:
        """Launches of the level-step kernel per run (resident: one per interval)."""
        return self.config.restarts if self.resident else self.config.steps

    def run_interval(self, r: int, state0_dev):
        out = D.torch().empty_like(state0_dev)
        # the rank runs on its own stream: state0 (e.g. the NCCL re-seed
        # broadcast of the previous interval) must be complete first
        D.torch().cuda.current_stream(state0_dev.device).synchronize()
        sec = ctypes.c_double(0.0)
        _lib.check_pipe(_lib.lib().ridc_pipe_run_interval(
            self._h, r, state0_dev.data_ptr(), out.data_ptr(), ctypes.byref(sec)), self._h)
        return out, sec.value

    def reset(self):
        """Zero this rank's mailbox counters (ridc_pipe_reset): between runs,
        after every rank finished and before any starts again."""
        _lib.check_pipe(_lib.lib().ridc_pipe_reset(self._h), self._h)

    def run_device(self, y0_dev, out_dev, broadcast=None, barrier=None) -> float:
        """All intervals; out_dev receives the solution on every rank.

        The stream-memop protocol counts global step numbers, so a run after
        the first resets every rank's counters between two barriers (every
        rank finished, every rank reset): ``barrier()`` defaults to
        torch.distributed.barrier."""
        if broadcast is None:
            broadcast = _nccl_broadcast(self.world)
        if self._runs and not self.resident:
            if barrier is None:
                import torch.distributed as dist
                barrier = dist.barrier
            barrier()
            self.reset()
            barrier()
        self._runs += 1
        _fin, sol, sec = run_levels(self, self.config.restarts, y0_dev, broadcast,
                                    self.rank == self.world - 1)
        out_dev.copy_(sol)
        return sec

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().ridc_pipe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _nccl_broadcast(world):
    import torch.distributed as dist

    def bcast(x, is_top):
        y = x.clone()
        dist.broadcast(y, src=world - 1)
        return y
    return bcast


class SequentialPipeline:
    """All levels' pipeline ranks in ONE process on ONE device, run one after
    another per interval (inbox rings sized for the whole run, so no rank ever
    waits on a rank that has not started).  Exercises the pipeline's data path
    -- peer-store mirrors, inbox watermarks, stream waits, re-seeding -- on a
    single GPU; its output must equal the single-device engine bitwise."""

    def __init__(self, ivp, config, device: int = 0):
        self.config = config
        L = config.levels
        self.ranks = [PipelineRank(ivp, config, j, L, device, inbox_capacity=config.steps + 1)
                      for j in range(L)]
        blobs = [r.blob for r in self.ranks]
        for r in self.ranks:
            r.connect(blobs)
        self.ivp = self.ranks[0].ivp
        self._runs = 0

    def run(self, y0=None):
        y0 = self.ivp.initial_state if y0 is None else y0
        if self._runs:   # every rank is idle here: zero the step counters of the last run
            for rk in self.ranks:
                if not rk.resident:
                    rk.reset()
        self._runs += 1
        s0 = D.to_device(y0, self.ranks[0].device)
        finals = [None] * len(self.ranks)
        for r in range(self.config.restarts):
            for j, rk in enumerate(self.ranks):
                finals[j], _ = rk.run_interval(r, s0)
            s0 = finals[-1]
        return D.to_host(finals[-1]), [D.to_host(f) for f in finals]

    def close(self):
        for r in self.ranks:
            r.close()


class ConcurrentPipeline:
    """All levels' pipeline ranks in one process, each driven by its own host
    thread on its own stream, with the DEFAULT (small) inbox rings: the
    producers run ahead only as far as the consumers' release counters allow,
    so the watermark / backpressure protocol is exercised exactly as across
    GPUs.  ``devices`` may list one device per rank: the ranks then run the
    resident level march (in-kernel flag waits across the GPUs).  Ranks that
    share a device run the stream-memop path instead: every wait is a
    stream-memory wait, no kernel ever spins on another rank."""

    def __init__(self, ivp, config, devices=(0,), inbox_capacity: int = 0):
        self.config = config
        L = config.levels
        devs = [devices[j % len(devices)] for j in range(L)]
        # ranks sharing a device use the stream-memop path: every wait is a
        # stream wait, so they cannot deadlock (resident ranks would spin on
        # each other); one rank per device runs the resident level march
        resident = len(set(devs)) == L
        self.ranks = [PipelineRank(ivp, config, j, L, devs[j], inbox_capacity=inbox_capacity, resident=resident)
                      for j in range(L)]
        blobs = [r.blob for r in self.ranks]
        for r in self.ranks:
            r.connect(blobs)
        self.ivp = self.ranks[0].ivp
        self._runs = 0

    def run(self, y0=None):
        import threading
        y0 = self.ivp.initial_state if y0 is None else y0
        if self._runs:   # every rank is idle here: zero the step counters of the last run
            for r in self.ranks:
                if not r.resident:
                    r.reset()
        self._runs += 1
        s0 = [D.to_device(y0, r.device) for r in self.ranks]
        finals = [None] * len(self.ranks)
        secs = [0.0] * len(self.ranks)
        for interval in range(self.config.restarts):
            errs = []

            def work(j):
                try:
                    finals[j], t = self.ranks[j].run_interval(interval, s0[j])
                    secs[j] += t
                except Exception as exc:   # surfaced below
                    errs.append(exc)
            th = [threading.Thread(target=work, args=(j,)) for j in range(len(self.ranks))]
            for t in th:
                t.start()
            for t in th:
                t.join()
            if errs:
                raise errs[0]
            s0 = [finals[-1].to(f"cuda:{r.device}") for r in self.ranks]
        self.device_seconds = max(secs)   # the slowest rank's device time (all intervals)
        return D.to_host(finals[-1]), [D.to_host(f) for f in finals]

    def close(self):
        for r in self.ranks:
            r.close()


def shard_rows(ny: int, shard: int, nshards: int):
    """Global rows [r0, r1) of row shard `shard` (ridc_pipe_create_shard's split)."""
    return ny * shard // nshards, ny * (shard + 1) // nshards


def shard_neighbours(level: int, shard: int, nshards: int, levels: int):
    """The eight (level, shard) neighbours ridc_pipe_connect_shard takes, in its
    order -- (j-1, s), (j-1, s-1), (j-1, s+1), (j+1, s), (j+1, s-1), (j+1, s+1),
    (j, s-1), (j, s+1) -- shards wrapping around (y is periodic), None where
    the level does not exist."""
    j, s, S = level, shard, nshards
    want = [(j - 1, s), (j - 1, s - 1), (j - 1, s + 1), (j + 1, s), (j + 1, s - 1), (j + 1, s + 1),
            (j, s - 1), (j, s + 1)]
    return [(a, b % S) if 0 <= a < levels else None for a, b in want]


class ShardRank:
    """Level ``level`` of row shard ``shard`` in a levels x row-shards grid
    (the layer that uses every GPU when p < #GPUs).

    The rank computes its level on its rows of a 2-D grid; per step it takes
    its window from (level-1, shard) plus the two ghost rows from
    (level-1, shard-+1), its own ghost rows from (level, shard-+1), and
    delivers its boundary rows to the same-level neighbours and to the
    diagonal consumers (ridc_pipe_create_shard, include/ridc_b200.h).  The
    watermark / release protocol is the reference's LevelBuffer
    (engine.py:284-331), per neighbour."""

    def __init__(self, ivp, config, level: int, shard: int, nshards: int, device: int = 0,
                 inbox_capacity: int = 0):
        self.ivp = as_descriptor(ivp)
        self.config = config
        self.level, self.shard, self.nshards, self.device = level, shard, nshards, device
        self.problem = self.ivp.problem
        self.dt = (self.ivp.t_end - self.ivp.t_start) / config.steps
        self.weights = pack_weight_tables(config.levels, self.dt)
        D.require_cuda(device)
        cp = self.problem.to_c()
        h = ctypes.c_void_p()
        _lib.check_pipe(_lib.lib().ridc_pipe_create_shard(
            ctypes.byref(cp), float(self.ivp.t_start), float(self.ivp.t_end), config.levels,
            config.steps, config.restarts, self.weights.ctypes.data, self.weights.shape[0],
            level, shard, nshards, device, int(inbox_capacity), float(config.watchdog_seconds),
            ctypes.byref(h)))
        self._h = h
        nb = _lib.lib().ridc_pipe_handle_bytes()
        blob = ctypes.create_string_buffer(nb)
        _lib.check_pipe(_lib.lib().ridc_pipe_export(self._h, blob), self._h)
        self.blob = bytes(blob.raw)
        self.r0, self.r1 = shard_rows(self.problem.ny, shard, nshards)

    def connect(self, blobs):
        """blobs[(level, shard)] for every rank of the grid."""
        keep = [blobs[k] if k is not None else None
                for k in shard_neighbours(self.level, self.shard, self.nshards, self.config.levels)]
        arr = (ctypes.c_void_p * 8)(*[ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p) if b is not None else None
                                      for b in keep])
        self._keep = keep
        _lib.check_pipe(_lib.lib().ridc_pipe_connect_shard(self._h, arr), self._h)

    def reset(self):
        _lib.check_pipe(_lib.lib().ridc_pipe_reset(self._h), self._h)

    def run_interval(self, r: int, state0_dev):
        """state0_dev: the GLOBAL interval state; returns this shard's rows of
        the level's final and the device seconds."""
        nx = self.problem.nx
        out = D.torch().empty((self.r1 - self.r0) * nx, dtype=state0_dev.dtype, device=state0_dev.device)
        D.torch().cuda.current_stream(state0_dev.device).synchronize()
        sec = ctypes.c_double(0.0)
        _lib.check_pipe(_lib.lib().ridc_pipe_run_interval(
            self._h, r, state0_dev.data_ptr(), out.data_ptr(), ctypes.byref(sec)), self._h)
        return out, sec.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().ridc_pipe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GridPipeline:
    """Levels x row shards in one process: rank (j, s) on
    ``devices[(j * nshards + s) % len(devices)]``, each driven by its own host
    thread on its own stream (stream-memory waits only, so ranks may share a
    device).  Per interval the top level's shards are gathered into the next
    interval's state0 (the reference's re-seed, engine.py:506-521)."""

    def __init__(self, ivp, config, nshards: int, devices=(0,), inbox_capacity: int = 0):
        self.config = config
        L, S = config.levels, nshards
        self.nshards = S
        self.ranks = {}
        for j in range(L):
            for s in range(S):
                dev = devices[(j * S + s) % len(devices)]
                self.ranks[(j, s)] = ShardRank(ivp, config, j, s, S, dev, inbox_capacity=inbox_capacity)
        blobs = {k: r.blob for k, r in self.ranks.items()}
        for r in self.ranks.values():
            r.connect(blobs)
        self.ivp = self.ranks[(0, 0)].ivp
        self._runs = 0

    def run(self, y0=None):
        """(final_state, level_finals) as host arrays; device_seconds is the
        slowest rank's device time."""
        import threading
        torch = D.torch()
        L, S = self.config.levels, self.nshards
        y0 = self.ivp.initial_state if y0 is None else y0
        if self._runs:   # every rank is idle here: zero the step counters of the last run
            for r in self.ranks.values():
                r.reset()
        self._runs += 1
        state = D.to_device(y0, self.ranks[(0, 0)].device)
        secs = {k: 0.0 for k in self.ranks}
        finals = {}
        for interval in range(self.config.restarts):
            s0 = {k: state.to(f"cuda:{r.device}") for k, r in self.ranks.items()}
            errs = []

            def work(k):
                try:
                    finals[k], t = self.ranks[k].run_interval(interval, s0[k])
                    secs[k] += t
                except Exception as exc:   # surfaced below
                    errs.append(exc)
            th = [threading.Thread(target=work, args=(k,)) for k in self.ranks]
            for t in th:
                t.start()
            for t in th:
                t.join()
            if errs:
                raise errs[0]
            dev = state.device
            state = torch.cat([finals[(L - 1, s)].to(dev) for s in range(S)])
        self.device_seconds = max(secs.values())
        levels = [torch.cat([finals[(j, s)].to(state.device) for s in range(S)]) for j in range(L)]
        return D.to_host(state), [D.to_host(x) for x in levels]

    def close(self):
        for r in self.ranks.values():
            r.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def run_pipelined_distributed(ivp, config, device: Optional[int] = None):
    """run_pipelined with one level per GPU; call on every rank (torchrun).

    Returns the RidcSolution-like tuple (final_state on every rank, this
    rank's device seconds)."""
    import torch.distributed as dist
    world = dist.get_world_size()
    rank = dist.get_rank()
    dev = int(os.environ.get("LOCAL_RANK", rank)) if device is None else device

    def exchange(blob):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out
    pr = PipelineRank(ivp, config, rank, world, dev, exchange=exchange)
    y0 = D.to_device(pr.ivp.initial_state, dev)
    out = D.torch().empty_like(y0)
    sec = pr.run_device(y0, out)
    pr.close()
    return D.to_host(out), sec


class RowShardGroup:
    """2-D row shards under the levels (``ridc_shards_*``):
    every shard runs all levels on its rows plus one ghost row per side, and
    the boundary rows of each newly written slot are exchanged after every
    tick.  ``devices=None``: all shards on ``device`` in lockstep (one graph);
    ``devices=[d0, d1, ...]``: one stream per shard on its device with
    device-side mailboxes and peer copies (devices may repeat).  Either way
    the result equals the unsharded engine bitwise."""

    def __init__(self, ivp, config, nshards: int, device: int = 0, devices=None):
        self.ivp = as_descriptor(ivp)
        self.config = config
        self.problem = self.ivp.problem
        dt = (self.ivp.t_end - self.ivp.t_start) / config.steps
        w = pack_weight_tables(config.levels, dt)
        D.require_cuda(device)
        cp = self.problem.to_c()
        h = ctypes.c_void_p()
        if devices is None:
            _lib.check_shards(_lib.lib().ridc_shards_create(
                ctypes.byref(cp), float(self.ivp.t_start), float(self.ivp.t_end), config.levels, config.steps,
                config.restarts, w.ctypes.data, w.shape[0], int(nshards), device, ctypes.byref(h)))
        else:
            devs = (ctypes.c_int32 * int(nshards))(*[int(devices[s % len(devices)]) for s in range(int(nshards))])
            for d in set(devs):
                D.require_cuda(d)
            _lib.check_shards(_lib.lib().ridc_shards_create_multi(
                ctypes.byref(cp), float(self.ivp.t_start), float(self.ivp.t_end), config.levels, config.steps,
                config.restarts, w.ctypes.data, w.shape[0], int(nshards), devs, float(config.watchdog_seconds),
                ctypes.byref(h)))
        self._h = h

    @property
    def kernel_launches(self) -> int:
        n = ctypes.c_int64(0)
        _lib.check_shards(_lib.lib().ridc_shards_info(self._h, ctypes.byref(n)), self._h)
        return n.value

    def run(self, y0=None):
        """-> (final_state, device seconds)."""
        y0 = np.ascontiguousarray(self.ivp.initial_state if y0 is None else y0, dtype=np.float64)
        out = np.empty_like(y0)
        sec = ctypes.c_double(0.0)
        _lib.check_shards(_lib.lib().ridc_shards_run(self._h, y0.ctypes.data, out.ctypes.data,
                                                     ctypes.byref(sec)), self._h)
        return out, sec.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().ridc_shards_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
