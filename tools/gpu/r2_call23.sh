set -x
timeout 900 python -m pytest tests/test_gpu_ark.py tests/test_gpu_studies.py -q > gpurun_out/r2c23_ark.log 2>&1; echo rc=$? >> gpurun_out/r2c23_ark.log
