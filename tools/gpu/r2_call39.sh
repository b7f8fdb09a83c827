set -x
timeout 1500 python -m pytest tests/test_gpu_sweep2d.py tests/test_gpu_resident.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2c39_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c39_tests.log
timeout 600 python bench.py --workload c3 --order 4 --nt 200 --no-extra --steps 2 --warmup 1 --cpu-budget 1 > gpurun_out/r2c39_c3p4.json 2>&1
timeout 600 python tools/sweep.py --exps 22,24,26 --orders 2,4,8 --nt 100 > gpurun_out/r2c39_sweeplev.log 2>&1
RIDC_SWEEP_CTA=1 timeout 600 python tools/sweep.py --exps 24 --orders 1 --nt 200 > gpurun_out/r2c39_sweepcta.log 2>&1
tail -n 3 gpurun_out/r2c39_tests.log; python -c "
import json; d=json.loads(open('gpurun_out/r2c39_c3p4.json').read().strip().split('\n')[-1]); print('c3p4', d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_us'])"; cut -c1-160 gpurun_out/r2c39_sweeplev.log gpurun_out/r2c39_sweepcta.log
