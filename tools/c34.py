"""C3 / C4 (2-D) on one GPU: device time per solve at reduced Nt with the
workload's dt (shortened T), all levels on one device.  Reported beside the
C2 bench line; the multi-GPU level pipeline for these is measured when a
multi-GPU box is available."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402

out = []
peak, _ = bench.hbm_peak()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for wl, orders, nt in (("c3", (1, 4), 100), ("c4", (1, 8), 60)):
    sysm, full_nt, cfg = bench.workload(wl)
    ivp = sysm.ivp
    sysm = P.StructuredIVP(ivp.problem, 0.0, ivp.t_end * nt / full_nt, ivp.initial_state)
    n = ivp.problem.dimension
    y0 = torch.from_numpy(np.array(ivp.initial_state)).cuda()
    o = torch.empty_like(y0)
    for p in orders:
        with E.Engine(sysm, E.RidcConfig(levels=p, steps=nt)) as eng:
            eng.run_device(y0, o)
            ts = []
            for _ in range(2):
                flush.zero_()
                torch.cuda.synchronize()
                ts.append(eng.run_device(y0, o))
            info = eng.info
        t = min(ts)
        ticks = info["ticks_per_interval"]
        bpp = sum(bench.bytes_per_point(j) for j in range(p))
        row = {"workload": cfg["workload"], "grid": cfg["grid"], "order": p, "nt": nt,
               "ms_per_solve": t * 1e3, "us_per_tick": t / ticks * 1e6,
               "grid_pt_steps_per_s": n * nt / t, "achieved_gbs": bpp * n * nt / t / 1e9,
               "frac": bpp * n * nt / t / 1e9 / peak, "items_per_level": info["items_per_level"],
               "threads": info["threads"], "r": info["r"]}
        out.append(row)
        print(json.dumps(row), flush=True)
    del y0, o
    torch.cuda.empty_cache()
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
