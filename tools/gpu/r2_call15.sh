set -x
RIDC_CHECKED=1 python tools/sanitize.py > gpurun_out/r2c15_checked_sanitize.log 2>&1; echo rc=$? >> gpurun_out/r2c15_checked_sanitize.log
RIDC_CHECKED=1 python -m pytest tests/test_gpu_reslevels.py tests/test_gpu_pipeline.py tests/test_gpu_sweep2d.py tests/test_gpu_resident.py tests/test_gpu_parity.py tests/test_gpu_shards.py tests/test_gpu_ark.py -x -q > gpurun_out/r2c15_checked_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c15_checked_tests.log
RIDC_NO_CARRY=1 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "c2_febe" > gpurun_out/r2c15_c2_halo.log 2>&1
python - > gpurun_out/r2c15_c2_tick.log 2>&1 <<'PY'
import sys; sys.path[:0] = ['.', 'tests']
import numpy as np, _golden as G
from oracle import oracle as O
from paper_1209_4297_b200 import engine as E, problems as P
from paper_1209_4297_b200.quadrature import pack_weight_tables
ivp = P.reaction_diffusion_c2().ivp
with E.Engine(ivp, E.RidcConfig(levels=1, steps=10000), tick_only=True) as t, E.Engine(ivp, E.RidcConfig(levels=1, steps=10000)) as c:
    a = t.run().final_state; b = c.run().final_state
dt = 1e-4
ref = O.run(ivp.problem, ivp.initial_state, 1, 10000, 1, dt, pack_weight_tables(1, dt))["final_state"]
print("tick vs oracle", G.normwise(a, ref), "carry vs oracle", G.normwise(b, ref), "carry vs tick", G.normwise(b, a))
PY
tail -3 gpurun_out/r2c15_checked_sanitize.log gpurun_out/r2c15_checked_tests.log; cat gpurun_out/r2c15_c2_tick.log; grep "n=" gpurun_out/r2c15_c2_halo.log
