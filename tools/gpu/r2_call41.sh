set -x
for cps in 2 1; do
RIDC_S2L_CPS=$cps timeout 600 python bench.py --workload c3 --order 4 --nt 200 --no-extra --steps 2 --warmup 1 --cpu-budget 1 > gpurun_out/r2c41_c3p4_cps$cps.json 2>&1
done
timeout 600 python bench.py --workload c4 --order 8 --nt 100 --no-extra --steps 2 --warmup 1 --cpu-budget 1 > gpurun_out/r2c41_c4p8.json 2>&1
timeout 900 python -m pytest tests/test_gpu_sweep2d.py tests/test_gpu_fullsize.py -x -q -k "sweep2d or c3 or c4" > gpurun_out/r2c41_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c41_tests.log
tail -n 2 gpurun_out/r2c41_tests.log; for f in c3p4_cps2 c3p4_cps1 c4p8; do python -c "
import json; d=json.loads(open('gpurun_out/r2c41_$f.json').read().strip().split('\n')[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_us'])"; done
