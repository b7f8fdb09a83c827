"""Per-rank device time of the one-level-per-GPU pipeline, measured on ONE GPU
(WORKLOAD=c2|c3|c4, ORDERS, NT).

Every rank of ``SequentialPipeline`` runs alone (whole-run inbox rings, so its
watermark waits are already satisfied and nothing waits on another rank): the
time per step of rank j is a lower bound of the p-GPU pipeline's step time
(NVLink stores land in local memory here).  Printed beside the resident FEBE
march on the same workload (C2 shape, reduced Nt with C2's dt).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1209_4297_b200 import distributed as Dd  # noqa: E402
from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402

nt = int(os.environ.get("NT", "500"))
orders = [int(x) for x in os.environ.get("ORDERS", "2,4").split(",")]
sysm, full_nt, cfg = bench.workload(os.environ.get("WORKLOAD", "c2"))
ivp = sysm.ivp
sysm = P.StructuredIVP(ivp.problem, 0.0, ivp.t_end * nt / full_nt, ivp.initial_state)
n = ivp.problem.dimension
out = []
y0 = torch.from_numpy(np.array(ivp.initial_state)).cuda()
o = torch.empty_like(y0)
with E.Engine(sysm, E.RidcConfig(levels=1, steps=nt)) as eng:
    eng.run_device(y0, o)
    t = min(eng.run_device(y0, o) for _ in range(3))
febe = t / nt
out.append({"what": "febe_engine_1gpu", "us_per_step": febe * 1e6})
print(json.dumps(out[-1]), flush=True)
for p in orders:
    pipe = Dd.SequentialPipeline(sysm, E.RidcConfig(levels=p, steps=nt))
    s0 = y0.clone()
    best = [1e30] * p
    for rep in range(3):
        for j, rk in enumerate(pipe.ranks):
            _, sec = rk.run_interval(0, s0)
            best[j] = min(best[j], sec)
    for j in range(p):
        row = {"what": f"pipe_rank_alone p={p} level={j}", "workload": cfg["workload"],
               "resident": pipe.ranks[j].resident, "us_per_step": best[j] / nt * 1e6,
               "ratio_vs_febe": best[j] / nt / febe}
        out.append(row)
        print(json.dumps(row), flush=True)
    pipe.close()
    torch.cuda.empty_cache()
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
