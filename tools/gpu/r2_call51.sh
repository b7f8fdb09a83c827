set -x
RIDC_CARRY_SWEEP=1 timeout 900 python - > gpurun_out/r2c51_par.log 2>&1 <<'PY'
import sys; sys.path[:0] = ['.', 'tests']
import numpy as np, _golden as G
from oracle import oracle as O
from paper_1209_4297_b200 import engine as E, problems as P
from paper_1209_4297_b200.quadrature import pack_weight_tables
for n, p, steps in [(1 << 21, 1, 12), (1 << 21, 3, 12), (1 << 22, 2, 10), (1 << 22 + 0, 4, 14)]:
    ivp = P.StructuredIVP(P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)).problem, 0.0, 1e-4 * steps,
                          P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2)).ivp.initial_state)
    cfg = E.RidcConfig(levels=p, steps=steps)
    with E.Engine(ivp, cfg) as a, E.Engine(ivp, cfg, tick_only=True) as b:
        ra, rb = a.run(), b.run(); ra2 = a.run()
        print(n, p, a.info["path_name"], "vs tick", max(G.normwise(ra.level_finals[j], rb.level_finals[j]) for j in range(p)),
              "repeat", all(np.array_equal(ra.level_finals[j], ra2.level_finals[j]) for j in range(p)), flush=True)
PY
RIDC_CARRY_SWEEP=1 timeout 900 python tools/sweep.py --exps 21,22,23,24,26 --orders 1,2,4,8 --nt 100 > gpurun_out/r2c51_sweep.log 2>&1
cat gpurun_out/r2c51_par.log | tail -8; cut -c1-140 gpurun_out/r2c51_sweep.log
