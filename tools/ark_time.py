"""Time the device ARK comparators (imex3 / imex4) on C2's grid and dt:
device time of whole marches (CUDA events in ridc_ark_run_device), path read
back from the context.  python tools/ark_time.py [--steps 10000]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1209_4297_b200 import problems as P, steppers as S  # noqa: E402
from paper_1209_4297_b200.tableaus import imex3_tableau, imex4_tableau  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10000)
ap.add_argument("--exp", type=int, default=20)
a = ap.parse_args()
s = P.reaction_diffusion_c2(n=1 << a.exp)
ivp = P.StructuredIVP(s.problem, 0.0, 1e-4 * a.steps, s.ivp.initial_state)
y0 = torch.from_numpy(np.array(ivp.initial_state)).cuda()
out = torch.empty_like(y0)
for name, tab in (("imex3", imex3_tableau()), ("imex4", imex4_tableau())):
    with S.ArkEngine(ivp, tab, 0.0, ivp.t_end, a.steps) as eng:
        eng.run_device(y0, out)
        ts = [eng.run_device(y0, out) for _ in range(3)]
        inf = eng.info
    t = float(np.median(ts))
    print(json.dumps({"scheme": name, "points": 1 << a.exp, "steps": a.steps, "path": inf["path_name"],
                      "ms_per_solve": t * 1e3, "us_per_step": t / a.steps * 1e6,
                      "us_per_stage_launch": t / (a.steps * inf["items_per_step"]) * 1e6,
                      "grid_pt_steps_per_s": (1 << a.exp) * a.steps / t}), flush=True)
