import sys; sys.path[:0] = ['.', 'tests']
import numpy as np, _golden as G
from paper_1209_4297_b200 import engine as E, problems as P
for n, steps in [(1 << 17, 40), (1 << 20, 40), (1 << 21, 40)]:
    sysm = P.build_reaction_diffusion(P.ReactionDiffusionSpec(n=n, d=1e-6 * (2.0 ** 20 / n) ** 2, t_end=1e-4 * steps))
    cfg = E.RidcConfig(levels=1, steps=steps)
    with E.Engine(sysm, cfg) as a, E.Engine(sysm, cfg, tick_only=True) as b:
        ra, rb = a.run(), b.run(); ra2 = a.run()
        print(n, a.info["path_name"], "vs tick", G.normwise(ra.final_state, rb.final_state),
              "repeat", np.array_equal(ra.final_state, ra2.final_state), flush=True)
