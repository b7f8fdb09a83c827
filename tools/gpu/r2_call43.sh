set -x
RIDC_CHECKED=1 timeout 1200 python tools/sanitize.py > gpurun_out/r2c43_checked_sanitize.log 2>&1; echo rc=$? >> gpurun_out/r2c43_checked_sanitize.log
RIDC_CHECKED=1 timeout 1500 python -m pytest tests/test_gpu_resident.py tests/test_gpu_sweep2d.py -x -q > gpurun_out/r2c43_checked_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c43_checked_tests.log
tail -n 25 gpurun_out/r2c43_checked_sanitize.log; tail -n 3 gpurun_out/r2c43_checked_tests.log
