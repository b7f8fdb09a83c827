set -x
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_reslevels.py -x -q > gpurun_out/r2c29_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c29_tests.log
timeout 600 python tools/sweep.py --exps 16,17,18,19,20 --orders 2 --nt 400 > gpurun_out/r2c29_sweep.log 2>&1
RIDC_NO_RESIDENT_LEVELS=1 timeout 600 python tools/sweep.py --exps 16,17,18 --orders 2 --nt 400 > gpurun_out/r2c29_sweep_nores.log 2>&1
for f in gpurun_out/r2c29_tests.log gpurun_out/r2c29_sweep.log gpurun_out/r2c29_sweep_nores.log; do tail -n 6 $f | cut -c1-200; done
