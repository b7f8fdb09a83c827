"""All levels on one GPU: the resident level march (one launch per interval,
ridc_levels.cuh) vs the tick-kernel graph (RIDC_TICK_ONLY), device time per
solve, on the lines it covers (levels x segments <= SMs): C1 (N=1024, the
reference's own case) and segmented lines up to 2^17 points."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402


def short(system, t_end):
    ivp = system.ivp
    return P.StructuredIVP(ivp.problem, 0.0, t_end, ivp.initial_state)


cases = [
    ("c1-adv-diff-1024", short(P.build_advection_diffusion(P.AdvectionDiffusionSpec(dx=1 / 1024)), 4.0), 1000,
     (1, 2, 4, 8)),
    ("rd-2^16", short(P.reaction_diffusion_c2(n=1 << 16), 0.1), 1000, (2, 4, 8)),
    ("rd-2^17", short(P.reaction_diffusion_c2(n=1 << 17), 0.1), 1000, (2, 4)),
    ("rd-2^16-r110", short(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=1 << 16, d=1e-6 * 256.0)), 0.1),
     1000, (2, 4, 8)),
]
out = []
for name, ivp, nt, orders in cases:
    n = ivp.problem.dimension
    y0 = torch.from_numpy(np.array(ivp.initial_state)).cuda()
    o = torch.empty_like(y0)
    for p in orders:
        row = {"case": name, "points": n, "nt": nt, "order": p}
        for mode, kw in (("resident", {}), ("tick", {"tick_only": True})):
            with E.Engine(ivp, E.RidcConfig(levels=p, steps=nt), **kw) as eng:
                eng.run_device(y0, o)
                t = min(eng.run_device(y0, o) for _ in range(3))
                row[f"{mode}_launches"] = eng.info["kernel_launches"]
            row[f"{mode}_us_per_step"] = t / nt * 1e6
            row[f"{mode}_grid_pt_steps_per_s"] = n * nt / t
        row["speedup"] = row["tick_us_per_step"] / row["resident_us_per_step"]
        out.append(row)
        print(json.dumps(row), flush=True)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
