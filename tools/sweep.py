"""C5 grid-size sweep: 1-D reaction-diffusion, N = 2^16..2^26,
orders 1/2/4/8 with all levels on one GPU (resident marches where the
line fits: FEBE up to ~2^20, all levels while levels x segments <= SMs).  The stiffness r = dt*d/dx^2 is held
at the C2 value (~110) by scaling d with N; Nt is shortened with dt kept
(so the solve geometry is the workload's).  Device time of whole solves
(CUDA events inside ridc_run_device), L2 flushed between solves.

Per tick in the steady state every level is active, so the algorithmic bytes
of one tick are sum_j bytes_per_point(j) * N (bench.bytes_per_point).

    python tools/sweep.py [--exps 16,18,20,22,24,26] [--orders 1,2,4] [--nt 200]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--exps", default="16,18,20,22,24,26")
ap.add_argument("--orders", default="1,2,4,8")
ap.add_argument("--nt", type=int, default=200)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default="")
a = ap.parse_args()

peak, peak_kind = bench.hbm_peak()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
rows = []
for ex in [int(x) for x in a.exps.split(",")]:
    n = 1 << ex
    full_nt = 10000
    spec = P.ReactionDiffusionSpec(n=n, d=1e-6 * (float(1 << 20) / n) ** 2, t_end=1.0 * a.nt / full_nt)
    sysm = P.build_reaction_diffusion(spec)
    y0 = torch.from_numpy(np.array(sysm.ivp.initial_state)).cuda()
    out = torch.empty_like(y0)
    for p in [int(x) for x in a.orders.split(",")]:
        with E.Engine(sysm, E.RidcConfig(levels=p, steps=a.nt)) as eng:
            eng.run_device(y0, out)
            ts = []
            for _ in range(a.reps):
                flush.zero_()
                torch.cuda.synchronize()
                ts.append(eng.run_device(y0, out))
            info = eng.info
        t = float(np.median(ts))
        ticks = info["ticks_per_interval"]
        tick_s = t / ticks
        bpp = sum(bench.bytes_per_point(j) for j in range(p))
        # steady ticks carry all p levels; fill ticks fewer: average bytes per tick
        gbs = bpp * n * a.nt / t / 1e9
        path = info["path_name"]   # read back from the engine after the runs
        row = {"points": n, "order": p, "nt": a.nt, "path": path, "us_per_step": t / a.nt * 1e6,
               "ms_per_solve": t * 1e3, "us_per_tick": tick_s * 1e6,
               "grid_pt_steps_per_s": n * a.nt / t, "alg_bytes_per_pt_tick": bpp,
               "achieved_gbs": gbs, "frac": gbs / peak, "items_per_level": info["items_per_level"],
               "r": info["r"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump({"peak_gbs": peak, "peak_kind": peak_kind, "rows": rows}, f, indent=1)
