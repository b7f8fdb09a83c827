set -x
timeout 1800 python -m pytest tests/test_gpu_resident.py tests/test_gpu_ark.py tests/test_gpu_studies.py -x -q > gpurun_out/r2c46_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c46_tests.log
tail -n 3 gpurun_out/r2c46_tests.log; cut -c1-200 gpurun_out/r2c46_ark.log gpurun_out/r2c46_sweep.log
