set -x
RIDC_CHECKED=1 timeout 1200 python tools/sanitize.py > gpurun_out/r2c31_checked_sanitize.log 2>&1; echo rc=$? >> gpurun_out/r2c31_checked_sanitize.log
RIDC_CHECKED=1 timeout 1500 python -m pytest tests/test_gpu_resident.py tests/test_gpu_grid.py tests/test_gpu_ark.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r2c31_checked_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c31_checked_tests.log
tail -n 25 gpurun_out/r2c31_checked_sanitize.log; tail -n 3 gpurun_out/r2c31_checked_tests.log
