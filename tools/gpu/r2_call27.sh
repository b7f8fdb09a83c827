set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2" > gpurun_out/r2c27_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c27_tests.log
timeout 600 python tools/sweep.py --exps 18,20 --orders 2 --nt 400 > gpurun_out/r2c27_sweep.log 2>&1
for f in gpurun_out/r2c27_tests.log gpurun_out/r2c27_sweep.log; do tail -n 4 $f | cut -c1-250; done
