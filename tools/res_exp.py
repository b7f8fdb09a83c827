"""Resident FEBE march at C2: how much of a step is the neighbour exchange?
Times the march with RIDC_RES_EXP = 0 (production), 1 (no halo waits),
2 (no edge pushes), 3 (neither: compute only).  Variants 1-3 give WRONG
states; they only bound the exchange's share of the step.

    python tools/res_exp.py [--nt 2000] [--n 1048576]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nt", type=int, default=2000)
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--exps", default="0,1,2,3")
a = ap.parse_args()

spec = P.ReactionDiffusionSpec(n=a.n, d=1e-6 * (float(1 << 20) / a.n) ** 2, t_end=1e-4 * a.nt)
sysm = P.build_reaction_diffusion(spec)
y0 = torch.from_numpy(np.array(sysm.ivp.initial_state)).cuda()
out = torch.empty_like(y0)
res = {}
for ex in [int(x) for x in a.exps.split(",")]:
    os.environ["RIDC_RES_EXP"] = str(ex)
    with E.Engine(sysm, E.RidcConfig(levels=1, steps=a.nt)) as eng:
        assert eng.info["path_name"] == "resident_febe", eng.info
        eng.run_device(y0, out)
        ts = [eng.run_device(y0, out) for _ in range(a.reps)]
    res[ex] = min(ts) / a.nt * 1e6
    print(f"exp {ex}: {res[ex]:.3f} us/step", flush=True)
os.environ.pop("RIDC_RES_EXP", None)
print(json.dumps({"n": a.n, "nt": a.nt, "us_per_step": res}))
