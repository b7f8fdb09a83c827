set -x
timeout 600 python bench.py --workload c3 --order 4 --nt 200 --no-extra --steps 2 --warmup 1 --cpu-budget 1 > gpurun_out/r2c40_c3p4.json 2>&1
timeout 600 python -m pytest tests/test_gpu_sweep2d.py -x -q > gpurun_out/r2c40_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c40_tests.log
tail -n 2 gpurun_out/r2c40_tests.log; python -c "
import json; d=json.loads(open('gpurun_out/r2c40_c3p4.json').read().strip().split('\n')[-1]); print('c3p4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_us'])"
