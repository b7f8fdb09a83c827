set -x
for cps in 2 1; do
RIDC_S2D_CPS=$cps timeout 600 python bench.py --workload c3 --order 1 --nt 200 --no-extra --steps 3 --warmup 2 --cpu-budget 1 > gpurun_out/r2c37_c3_cps$cps.json 2>&1
done
for cps in 2 1; do python -c "
import json,sys; d=json.loads(open('gpurun_out/r2c37_c3_cps$cps.json').read().strip().split('\n')[-1]); print($cps, d['ms_per_step'], d['roofline']['frac'])"; done
