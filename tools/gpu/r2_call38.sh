set -x
timeout 900 python -m pytest tests/test_gpu_sweep2d.py tests/test_gpu_fullsize.py -x -q -k "sweep2d or c3 or febe" > gpurun_out/r2c38_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c38_tests.log
timeout 600 python bench.py --workload c3 --order 1 --nt 200 --no-extra --steps 3 --warmup 2 --cpu-budget 1 > gpurun_out/r2c38_c3.json 2>&1
timeout 600 python bench.py --workload c4 --order 1 --nt 100 --no-extra --steps 3 --warmup 2 --cpu-budget 1 > gpurun_out/r2c38_c4.json 2>&1
tail -n 3 gpurun_out/r2c38_tests.log; for f in c3 c4; do python -c "
import json; d=json.loads(open('gpurun_out/r2c38_$f.json').read().strip().split('\n')[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_us'])"; done
