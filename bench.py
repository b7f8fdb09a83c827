"""Benchmark: order-p RIDC wall time & grid-point*steps/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4] [--order P] [--nt NT] [--points N]

One bench "step" = one full RIDC-FBE solve (all Nt time steps, all levels) of
the workload, starting from an initial state already resident in HBM.
Default workload (N=1): BASELINE.json configs[1] -- 1-D reaction-diffusion,
2^20 grid points, Nt = 10^4, order p = number of GPUs (1 GPU: FEBE, order 1);
the same line also reports orders 2 and 4 with all levels on the one GPU.

value = grid points * Nt * K / (device time of the K solves), max over ranks.
Between timed solves L2 is flushed (a 512 MiB write, untimed).  `e2e` is the
same metric through the host-buffer C-ABI call (``ridc_run``: H2D of y0,
marching, D2H of the final state).  `cpu_baseline` times the CPU oracle port
(oracle/ridc_oracle.c, one thread per level like the reference's workers) on
a bounded sample of the same workload.

`--impl reference` times only that CPU port (the reference is Python+numba
with dense O(N^2) solves and cannot run N = 2^20) and prints
the same JSON line with "impl": "reference" and the identical `config`.

Under torchrun (N > 1) every rank owns one RIDC level (order = N) on its GPU
(distributed.PipelineRank).  When fewer GPUs are visible than ranks (a
one-GPU box), the ranks share the devices round-robin: the control plane
runs over gloo, the ranks use the stream-memop pipeline (no in-kernel
cross-rank waits) and the line says so ("ranks_share_devices": true) -- a
functional run of the N > 1 path, not a scaling number.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "order-p RIDC wall time & grid-point·steps/s vs 1-GPU FEBE (p=1,2,4,8 GPUs)"
UNIT = "grid-point*steps/s"
HBM_FALLBACK = 6650.0


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def workload(name, points=None, nt=None):
    from paper_1209_4297_b200 import problems as P
    if name == "c2":
        # dt = 1e-4 (r ~ 110 at 2^20 points) whatever Nt: --nt shortens the horizon
        n = points or (1 << 20)
        nt = nt or 10000
        sysm = P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, t_end=1e-4 * nt))
        return sysm, nt, {"workload": "c2-reaction-diffusion-1d", "points": n, "nt": nt, "t_end": 1e-4 * nt}
    if name == "c5":
        # configs[4] grid-size sweep: 1-D RD, r held at C2's ~110 (d scaled with N), dt = 1e-4
        n = points or (1 << 24)
        nt = nt or 200
        sysm = P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (float(1 << 20) / n) ** 2,
                                                                  t_end=1e-4 * nt))
        return sysm, nt, {"workload": "c5-reaction-diffusion-1d", "points": n, "nt": nt, "t_end": 1e-4 * nt}
    if name == "c1":
        sysm = P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024, t_end=4.0))
        return sysm, nt or 1000, {"workload": "c1-adv-diff-1d", "points": 1024, "nt": nt or 1000}
    # 2-D workloads: the configuration's dt (T / 1000) whatever Nt (explicit y-terms)
    if name == "c3":
        n = points or 4096
        nt = nt or 1000
        sysm = P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=n, ny=n, t_end=0.02 * nt / 1000))
        return sysm, nt, {"workload": "c3-adv-diff-2d", "points": n * n, "grid": [n, n], "nt": nt}
    if name == "c4":
        n = points or 8192
        nt = nt or 1000
        sysm = P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=n, ny=n, t_end=0.05 * nt / 1000))
        return sysm, nt, {"workload": "c4-reaction-diffusion-2d", "points": n * n, "grid": [n, n], "nt": nt}
    raise SystemExit(f"unknown workload {name}")


def bytes_per_point(level):
    """Algorithmic HBM bytes per grid point of one level-step."""
    return 16 if level == 0 else 8 * (level + 3)


def bench_config(cfg, order, world):
    """The workload description both arms print (identical dicts)."""
    c = dict(cfg)
    c.update({"order": order, "levels_per_gpu": 1 if world > 1 else order,
              "parallelism": f"levels-over-gpus{world}" if world > 1 else "1gpu",
              "l2": "flushed between solves (512 MiB write); state stays resident within a solve"})
    return c


def host_cpus():
    """Host cores the CPU legs could use (os.cpu_count, affinity mask)."""
    try:
        aff = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        aff = None
    return {"host_cpu_count": os.cpu_count(), "affinity_cpus": aff}


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def cpu_sample(sysm, levels, nt, budget_s=12.0):
    """Time the CPU oracle port on a bounded number of steps of the workload."""
    from oracle import oracle as O
    from paper_1209_4297_b200.quadrature import pack_weight_tables
    ivp = sysm.ivp
    dt = (ivp.t_end - ivp.t_start) / nt
    w = pack_weight_tables(levels, dt)
    n = ivp.dimension
    probe = max(levels * (levels + 1) // 2 + 2, 4)
    r = O.run(ivp.problem, ivp.initial_state, levels, nt, 1, dt, w, workers=levels, max_steps=probe)
    per_step = r["wall_seconds"] / probe
    steps = int(min(max(probe, budget_s / max(per_step, 1e-9)), nt))
    r = O.run(ivp.problem, ivp.initial_state, levels, nt, 1, dt, w, workers=levels, max_steps=steps)
    out = {"value": n * steps / r["wall_seconds"], "unit": UNIT, "cores": levels,
           "kind": "port", "wall_seconds": r["wall_seconds"],
           "sample": f"{steps} of {nt} time steps, {n} points, order {levels}, "
                     f"{levels} thread(s) (one per level, as the reference's workers)"}
    out.update(host_cpus())
    return out


def cpu_sample_ark(sysm, tab, name, nt, budget_s=4.0):
    """The oracle's integrate_ark (numpy, one thread) on a bounded number of steps."""
    from oracle import oracle as O
    ivp = sysm.ivp
    dt = (ivp.t_end - ivp.t_start) / nt
    n = ivp.dimension
    args = (np.asarray(tab.a_implicit), np.asarray(tab.a_explicit), np.asarray(tab.b_implicit),
            np.asarray(tab.b_explicit))
    t0 = time.perf_counter()
    O.ark(ivp.problem, *args, ivp.initial_state, 0.0, dt, 1)
    per = time.perf_counter() - t0
    steps = int(min(max(1, budget_s / max(per, 1e-9)), nt))
    t0 = time.perf_counter()
    O.ark(ivp.problem, *args, ivp.initial_state, 0.0, dt * steps, steps)
    wall = time.perf_counter() - t0
    out = {"value": n * steps / wall, "unit": UNIT, "cores": 1, "kind": "port", "wall_seconds": wall,
           "sample": f"{steps} of {nt} {name} steps, {n} points, 1 thread (numpy)"}
    out.update(host_cpus())
    return out


def run_reference(args):
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    if rank != 0:
        return 0
    order = args.order or max(1, args.gpus)
    sysm, nt, cfg = workload(args.workload, args.points, args.nt)
    from oracle import oracle as O
    from paper_1209_4297_b200.quadrature import pack_weight_tables
    ivp = sysm.ivp
    dt = (ivp.t_end - ivp.t_start) / nt
    w = pack_weight_tables(order, dt)
    n = ivp.dimension
    fill = order * (order + 1) // 2 + 2
    sample = max(fill, args.sample_steps)
    for _ in range(args.warmup):
        O.run(ivp.problem, ivp.initial_state, order, nt, 1, dt, w, workers=order, max_steps=fill)
    total = 0.0
    for _ in range(args.steps):
        r = O.run(ivp.problem, ivp.initial_state, order, nt, 1, dt, w, workers=order, max_steps=sample)
        total += r["wall_seconds"]
    value = n * sample * args.steps / total
    cfg = bench_config(cfg, order, world)
    cpu = {"value": value, "unit": UNIT, "cores": order, "kind": "port",
           "sample": f"{sample} of {nt} time steps per bench step, {n} points, "
                     f"{order} thread(s) (one per level)"}
    cpu.update(host_cpus())
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "CPU oracle port of the reference path (reference itself is dense O(N^2), "
                "infeasible at this N)",
    }
    print(json.dumps(line))
    return 0


def pipeline_ranks_alone(sysm, nt, febe_step_s, orders=(2, 4), nt_sample=200):
    """The one-level-per-GPU pipeline's ranks, each timed ALONE on this GPU
    (SequentialPipeline: ranks one after another, whole-run inboxes, inputs
    already published; NVLink stores land in local HBM): per-step device time
    of every rank = a lower bound of the p-GPU step on this workload (same dt,
    nt_sample steps).  One GPU per box here, so N > 1 itself is not timed."""
    from paper_1209_4297_b200 import distributed as PD
    from paper_1209_4297_b200 import engine as E
    from paper_1209_4297_b200 import problems as P
    import torch
    ivp = sysm.ivp
    short = P.StructuredIVP(ivp.problem, ivp.t_start, ivp.t_start + (ivp.t_end - ivp.t_start) * nt_sample / nt,
                            ivp.initial_state)
    y0 = torch.from_numpy(np.array(ivp.initial_state)).cuda()
    res = {"nt_sample": nt_sample, "febe_us_per_step": febe_step_s * 1e6}
    for p in orders:
        pipe = PD.SequentialPipeline(short, E.RidcConfig(levels=p, steps=nt_sample))
        try:
            best = [1e30] * p
            for _ in range(3):
                for j, rk in enumerate(pipe.ranks):
                    _, sec = rk.run_interval(0, y0)
                    best[j] = min(best[j], sec)
            res[f"p{p}"] = {"resident": all(r.resident for r in pipe.ranks),
                            "us_per_step": [b / nt_sample * 1e6 for b in best],
                            "max_rank_vs_febe": max(best) / nt_sample / febe_step_s}
        finally:
            pipe.close()
        torch.cuda.empty_cache()
    return res


def _timed_solves(run_device, flush, reps):
    import torch
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        ts.append(run_device())
    return ts


def workload_line(name, order, flush, reps=2, nt=None, points=None, cpu_budget=3.0):
    """One extra 1-GPU workload (C3 / C4 / C5 shapes): device time of whole solves,
    the dominant kernel's roofline (algorithmic bytes of a steady tick / tick time)."""
    import torch
    from paper_1209_4297_b200 import engine as E
    sysm, nt, cfg = workload(name, points, nt)
    n = sysm.ivp.dimension
    y0 = torch.from_numpy(np.array(sysm.ivp.initial_state)).cuda()
    out = torch.empty_like(y0)
    with E.Engine(sysm, E.RidcConfig(levels=order, steps=nt)) as eng:
        eng.run_device(y0, out)
        ts = _timed_solves(lambda: eng.run_device(y0, out), flush, reps)
        info = eng.info
    t = sum(ts) / len(ts)
    ticks = nt + order * (order - 1) // 2
    bytes_tick = sum(bytes_per_point(j) for j in range(order)) * n   # steady tick, all levels active
    peak, _ = hbm_peak()
    achieved = bytes_tick * nt / ticks / (t / ticks) / 1e9 if ticks else 0.0
    del y0, out
    torch.cuda.empty_cache()
    return {"workload": cfg["workload"], "points": n, "nt": nt, "order": order, "path": info["path_name"],
            "value": n * nt / t, "unit": UNIT, "ms_per_solve": t * 1e3, "us_per_tick": t / ticks * 1e6,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "bytes_per_tick": bytes_tick},
            # the CPU oracle port beside it (one thread per level), a bounded sample
            "cpu_baseline": cpu_sample(sysm, order, nt, budget_s=cpu_budget)}


def run_ours(args):
    import torch
    from paper_1209_4297_b200 import engine as E
    from paper_1209_4297_b200 import problems as P

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    ndev = torch.cuda.device_count()
    shared = world > 1 and ndev < world   # one-GPU box: ranks share the devices round-robin
    dev = local % max(ndev, 1)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")   # NCCL refuses two ranks on one device
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))

    def reduce_max(x):
        if dist is None:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    sysm, nt, cfg = workload(args.workload, args.points, args.nt)
    n = sysm.ivp.dimension
    order = args.order or max(1, world)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    if world > 1:
        # one level per GPU (levels = ranks): the NVLink point-to-point pipeline
        from paper_1209_4297_b200 import distributed as PD
        if order != world:
            raise SystemExit("--order must equal the GPU count (one level per GPU)")

        def exchange(blob):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out

        def gloo_bcast(x, is_top):   # re-seed broadcast over the gloo control plane
            h = x.detach().cpu().clone()
            dist.broadcast(h, src=world - 1)
            return h.to(x.device)
        runner = PD.PipelineRank(sysm, E.RidcConfig(levels=order, steps=nt), rank, world, dev,
                                 exchange=exchange, resident=not shared)
        y0 = torch.from_numpy(np.array(sysm.ivp.initial_state)).cuda()
        out = torch.empty_like(y0)
        bcast = gloo_bcast if shared else None

        def solve_device():
            return runner.run_device(y0, out, broadcast=bcast, barrier=barrier)
        launches_per_step = runner.kernel_launches
        tick_launches = runner.tick_launches
        # this rank's level-step bytes per point; the producer side also writes the
        # consumer's inbox copy (8 B/pt over NVLink, counted on the consumer);
        # per launch of the level-step kernel (resident: a whole interval)
        path = runner.info["path"]
        lev_bytes = (bytes_per_point(rank) + (8 if rank < world - 1 else 0)) * nt / max(tick_launches, 1)
    else:
        eng = E.Engine(sysm, E.RidcConfig(levels=order, steps=nt))
        y0 = torch.from_numpy(np.array(sysm.ivp.initial_state)).cuda()
        out = torch.empty_like(y0)

        def solve_device():
            return eng.run_device(y0, out)
        launches_per_step = eng.info["kernel_launches"]

    for _ in range(max(args.warmup, 0)):
        solve_device()
    barrier()
    times = []
    clocks = ClockSampler(dev)
    with clocks:
        barrier()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            times.append(solve_device())
        barrier()
    t_local = float(sum(times))
    t_max = reduce_max(t_local)
    value = n * nt * args.steps / t_max
    ms_per_step = t_max / args.steps * 1e3

    if world == 1:
        # the path actually taken, read back from the engine after the timed runs
        info = eng.info
        path = info["path"]
        launches_per_step = info["kernel_launches"]
        # resident FEBE: seed + one march; resident level march: 2 seeds + one march
        # per interval; else the tick graph: seed + one launch per tick
        # resident marches (resident_febe, resident_levels, carry_febe): one march launch;
        # graph paths (tick kernel, FEBE sweeps): one launch per tick after the seed
        tick_launches = 1 if path in (1, 2, 3) else launches_per_step - 1
        lev_bytes = sum(bytes_per_point(j) for j in range(order)) * nt / max(tick_launches, 1)
    from paper_1209_4297_b200._lib import PATH_NAMES
    path_name = PATH_NAMES.get(path, "?")

    # roofline of the dominant kernel: algorithmic bytes per launch / average
    # launch duration over the timed region (CUDA events on the library's stream)
    peak, peak_kind = hbm_peak()
    per_launch_s = t_local / (args.steps * max(tick_launches, 1))
    bytes_launch = lev_bytes * n
    achieved = bytes_launch / per_launch_s / 1e9
    traffic, traffic_note = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                ent = json.load(f).get(f"{cfg['workload']}/p{order}/{path_name}")
            if isinstance(ent, dict) and ent.get("nt") == nt:
                traffic, traffic_note = ent["bytes_per_launch"], ent.get("source")
        except Exception:
            traffic = None
    kernels = {
        "resident_febe": "k_resident_febe (whole FEBE march in one launch: registers-resident chunks, "
                         "stencil + factored tridiagonal solve per step, halo edges via tagged L2 mailbox)",
        "resident_levels": ("k_resident_levels (this rank's level: whole interval in one launch, TMA-staged "
                            "window, per-segment publish/release flags, tile stores into the consumer's inbox "
                            "over NVLink)") if world > 1 else
                           ("k_resident_levels (all levels on this GPU in one launch: a co-resident CTA group "
                            "per level, registers-resident chunks, TMA-staged windows, per-segment flags)"),
        "warp_carry_febe": "k_febe_wcarry (whole FEBE march in one launch: one 512-point chunk per warp in "
                           "registers, rhs + factored tridiagonal solve per step, chunks coupled by two carries per "
                           "step -- shared memory within a CTA, L2 between CTAs -- computed from the rhs and "
                           "published before the recurrences, no block barriers)",
        "carry_febe": "k_febe_carry (whole FEBE march in one launch: one tile per SM in registers, rhs + "
                      "factored tridiagonal solve per step, tiles coupled by two tagged carries per step through L2)",
        "sweep_febe": "k_sweep_febe (one launch per step: every SM sweeps a contiguous range of the line through "
                      "TMA-staged chunks, carries along the sweep, each point read and written once)",
        "sweep_warp_febe": "k_sweep_febe_warp (one launch per step: every warp sweeps a contiguous range of the "
                           "line through its own TMA-staged 512-point chunks, no block barriers, each point read "
                           "and written once)",
        "resident_carry_levels": "k_carry_res2w / k_carry_res2 (RIDC-2: both levels in registers for a whole "
                                 "interval, one cooperative launch; one 512-point chunk per warp (or one tile per "
                                 "SM) coupled by carries and the predictor's end points)",
        "carry_levels": "k_carry_levels (one launch per tick: every warp folds and solves one 512-point chunk of "
                        "each active level, neighbouring chunks exchange two carries through L2)",
        "sweep2d_febe": "k_sweep2d_febe (one launch per step: every CTA sweeps a row block, each row read once and "
                        "folded into three right-hand sides, cyclic x-line solves)",
        "tick": "k_tick_chunk (fused level-step: stencils + factored tridiagonal solve)",
    }
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                "kernel": kernels.get(path_name, path_name), "path": path_name,
                "bytes_per_launch": bytes_launch, "launch_us": per_launch_s * 1e6,
                "steps_per_launch": nt // max(tick_launches, 1)}
    if traffic_note:
        roofline["traffic_source"] = traffic_note
    if path_name in ("warp_carry_febe", "carry_febe", "resident_febe", "resident_levels", "resident_carry_levels"):
        # the state stays on the SMs for the whole launch: `achieved` is the
        # equivalent bandwidth of the algorithmic bytes (frac may exceed 1);
        # the kernel is bound by its per-step dependency chain, not by HBM
        roofline["note"] = ("SM-resident march: DRAM traffic is one read and one write of the state per launch "
                            "(traffic); achieved/frac are the algorithmic 16 B/pt/step as equivalent bandwidth, "
                            "the bound is the per-step dependency chain (recurrences, warp scans, the neighbour "
                            "carries' L2 hop) and FP64 instruction issue")

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            # level-steps/s = p N Nt / wall (work done by all levels)
            "level_steps_per_s": order * n * nt * args.steps / t_max,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "gpu_launches": int(launches_per_step * args.steps)}
    line["config"] = bench_config(cfg, order, world)
    line["path"] = path_name
    if shared:
        line["ranks_share_devices"] = True
        line["note"] = (f"{world} ranks on {ndev} visible GPU(s): stream-memop pipeline ranks time-sliced on "
                        "shared devices -- a functional run of the N>1 path, not a scaling measurement")
    line["roofline"] = roofline
    line["clocks"] = clocks.summary()

    # e2e: the host-buffer C-ABI call (H2D y0 + marching + D2H final)
    if world == 1:
        # pinned host buffers (the contract's "from pinned host memory")
        y0p = torch.from_numpy(np.array(sysm.ivp.initial_state, dtype=np.float64, order="C")).pin_memory()
        finp = torch.empty(n, dtype=torch.float64).pin_memory()
        y0h, fin = y0p.numpy(), finp.numpy()
        from paper_1209_4297_b200 import _lib
        walls = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(_lib.lib().ridc_run(eng._h, y0h.ctypes.data, fin.ctypes.data, None, None,
                                           None), eng._h)
            walls.append(time.perf_counter() - t0)
        line["e2e"] = {"value": n * nt * len(walls) / sum(walls), "unit": UNIT,
                       "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n}
        line["cpu_baseline"] = cpu_sample(sysm, order, nt, budget_s=args.cpu_budget)
        # extra orders with all levels on this GPU (configs[1]: "RIDC order 1-4 on 1 B200"),
        # each beside the CPU oracle with one thread per level (the reference's workers)
        extra = {}
        if not args.no_extra:
            for p in (2, 3, 4):
                if p == order:
                    continue
                with E.Engine(sysm, E.RidcConfig(levels=p, steps=nt)) as e2:
                    e2.run_device(y0, out)
                    ts = _timed_solves(lambda: e2.run_device(y0, out), flush, 2)
                    t_solve = sum(ts) / len(ts)
                    # every level does nt steps of bytes_per_point(j) algorithmic bytes per point
                    alg = sum(bytes_per_point(j) for j in range(p)) * n * nt
                    extra[f"order{p}_1gpu"] = {"value": n * nt * len(ts) / sum(ts),
                                               "level_steps_per_s": p * n * nt * len(ts) / sum(ts),
                                               "ms_per_solve": t_solve * 1e3,
                                               "wall_ratio_vs_febe": t_solve / (t_max / args.steps),
                                               "roofline": {"bound": "hbm", "achieved": alg / t_solve / 1e9,
                                                            "peak": peak, "unit": "GB/s",
                                                            "frac": alg / t_solve / 1e9 / peak},
                                               "path": e2.info["path_name"],
                                               "cpu_baseline": cpu_sample(sysm, p, nt, budget_s=args.cpu_budget / 3)}
            # the paper's ARK comparators on the same grid and dt (steppers.integrate_ark)
            from paper_1209_4297_b200.steppers import ArkEngine
            from paper_1209_4297_b200.tableaus import imex3_tableau, imex4_tableau
            ivp = sysm.ivp
            for name, tab in (("imex3", imex3_tableau()), ("imex4", imex4_tableau())):
                with ArkEngine(ivp, tab, ivp.t_start, ivp.t_end, nt) as ae:
                    ae.run_device(y0, out)
                    ts = _timed_solves(lambda: ae.run_device(y0, out), flush, 2)
                    extra[f"{name}_1gpu"] = {"value": n * nt * len(ts) / sum(ts),
                                             "ms_per_solve": sum(ts) / len(ts) * 1e3,
                                             "wall_ratio_vs_febe": (sum(ts) / len(ts)) / (t_max / args.steps),
                                             "launches_per_solve": ae.info["kernel_launches"],
                                             "cpu_baseline": cpu_sample_ark(sysm, tab, name, nt)}
        line["ridc_orders_1gpu"] = extra
        if not args.no_extra:
            line["pipeline_ranks_alone"] = pipeline_ranks_alone(sysm, nt, t_max / args.steps / nt)
            eng.close()
            del y0, out
            torch.cuda.empty_cache()
            # the paper headline's shape (configs[2], C3: 2-D adv-diff 4096^2): FEBE on
            # one GPU is the denominator of "RIDC-4 on 4 GPUs <= 1.1x FEBE on 1 GPU"
            line["c3_1gpu"] = {f"order{p}": workload_line("c3", p, flush) for p in (1, 4)}
            # configs[4]: the HBM-streaming FEBE sweep at 2^24 and 2^26 points (Nt 200, dt kept)
            line["c5_1gpu"] = {f"febe_2^{e}": workload_line("c5", 1, flush, points=1 << e) for e in (24, 26)}
    else:
        # e2e at N GPUs: every rank copies y0 in from pinned host memory, the
        # pipeline marches, every rank reads the solution back; wall time of the
        # slowest rank (CUDA events around the whole sequence)
        y0h = torch.from_numpy(np.array(sysm.ivp.initial_state)).pin_memory()
        finh = torch.empty_like(y0h).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        walls = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.zero_()
            barrier()
            e0.record()
            y0.copy_(y0h, non_blocking=True)
            torch.cuda.current_stream().synchronize()   # the pipeline runs on its own stream
            runner.run_device(y0, out, broadcast=bcast, barrier=barrier)
            finh.copy_(out, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            walls.append(e0.elapsed_time(e1) * 1e-3)
        tw = reduce_max(sum(walls))
        line["e2e"] = {"value": n * nt * len(walls) / tw, "unit": UNIT,
                       "h2d_bytes_per_step": 8 * n * world, "d2h_bytes_per_step": 8 * n * world}
        runner.close()
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--order", type=int, default=0)
    ap.add_argument("--points", type=int, default=0)
    ap.add_argument("--nt", type=int, default=0)
    ap.add_argument("--sample-steps", type=int, default=100)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-extra", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
