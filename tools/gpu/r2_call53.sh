set -x
./tools/micro/latency > gpurun_out/r2c53_lat.log 2>&1
cat > /tmp/par53.py <<'PY'
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
PY
for E in 0 2; do RIDC_WC_EXP=$E timeout 600 python /tmp/par53.py > gpurun_out/r2c53_par$E.log 2>&1; done
for E in 0 2 1 3; do RIDC_WC_EXP=$E timeout 600 python tools/sweep.py --exps 18,19,20,21 --orders 1 --nt 2000 --reps 5 > gpurun_out/r2c53_wc$E.log 2>&1; done
RIDC_WC_EXP=2 timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "carry" > gpurun_out/r2c53_t2.log 2>&1; echo rc=$? >> gpurun_out/r2c53_t2.log
cat gpurun_out/r2c53_lat.log gpurun_out/r2c53_par*.log; for E in 0 2 1 3; do echo E=$E; cut -c1-120 gpurun_out/r2c53_wc$E.log; done; tail -2 gpurun_out/r2c53_t2.log
