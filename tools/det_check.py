"""Repeat a run and report whether the device path is deterministic (bitwise),
and where repeated results differ (diagnostics for the streaming sweeps)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 23)
ap.add_argument("--steps", type=int, default=12)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--kind", default="rd1")
ap.add_argument("--levels", type=int, default=1)
a = ap.parse_args()
if a.kind == "rd1":
    ivp = P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=a.n, d=1e-6 * (2.0 ** 20 / a.n) ** 2,
                                                             t_end=1e-4 * a.steps)).ivp
elif a.kind == "ad2":
    ivp = P.build_advection_diffusion_2d(P.AdvectionDiffusion2DSpec(nx=a.n, ny=a.n, t_end=0.02 * a.steps / 1000)).ivp
else:
    ivp = P.build_reaction_diffusion_2d(P.ReactionDiffusion2DSpec(nx=a.n, ny=a.n, t_end=0.05 * a.steps / 1000)).ivp
with E.Engine(ivp, E.RidcConfig(levels=a.levels, steps=a.steps)) as eng:
    print("path", eng.info["path_name"], flush=True)
    outs = [eng.run().final_state for _ in range(a.reps)]
for r in range(1, a.reps):
    d = np.abs(outs[r] - outs[0])
    bad = np.nonzero(d)[0]
    print(f"rep {r}: max diff {d.max():.3e}, {bad.size} points differ"
          + (f", first {bad[:8].tolist()} last {bad[-4:].tolist()}" if bad.size else ""), flush=True)
