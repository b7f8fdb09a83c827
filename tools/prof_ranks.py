"""Small driver for ncu: the one-level-per-GPU pipeline ranks at the C2 shape,
run one after another on one device (whole-run inboxes: no rank waits on one
that has not run).  Each rank's interval is one k_resident_levels launch.
No timing claims (tools/pipe_ranks.py times them)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import bench  # noqa: E402
from paper_1209_4297_b200 import distributed as Dd  # noqa: E402
from paper_1209_4297_b200 import engine as E  # noqa: E402
from paper_1209_4297_b200 import problems as P  # noqa: E402

nt = int(os.environ.get("NT", "100"))
order = int(os.environ.get("ORDER", "4"))
sysm, full_nt, cfg = bench.workload("c2")
ivp = sysm.ivp
sysm = P.StructuredIVP(ivp.problem, 0.0, ivp.t_end * nt / full_nt, ivp.initial_state)
pipe = Dd.SequentialPipeline(sysm, E.RidcConfig(levels=order, steps=nt))
pipe.run()
pipe.close()
print("ok")
