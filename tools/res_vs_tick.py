"""Same-box comparison of the resident FEBE march and the tick kernel (no claims)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
wl = sys.argv[2] if len(sys.argv) > 2 else "c2"
pts = int(sys.argv[3]) if len(sys.argv) > 3 else None
sysm, full_nt, _ = bench.workload(wl, pts)
ivp = sysm.ivp
sysm = P.StructuredIVP(ivp.problem, 0.0, ivp.t_end * nt / full_nt, ivp.initial_state)
y0 = torch.from_numpy(np.array(sysm.initial_state)).cuda()
out = torch.empty_like(y0)
for rep in range(3):
    for tick in (False, True):
        with E.Engine(sysm, E.RidcConfig(levels=1, steps=nt), tick_only=tick, resident_segments=not tick) as eng:
            eng.run_device(y0, out)
            ts = [eng.run_device(y0, out) for _ in range(3)]
        print(f"{wl} n={sysm.problem.dimension} {'tick' if tick else 'resident'}: {min(ts) / nt * 1e6:.2f} us/step (min of 3)", flush=True)
