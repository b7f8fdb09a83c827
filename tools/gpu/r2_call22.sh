set -x
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q > gpurun_out/r2c22_grid.log 2>&1; echo rc=$? >> gpurun_out/r2c22_grid.log
timeout 600 python -m pytest tests/test_gpu_shards.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r2c22_pipe.log 2>&1; echo rc=$? >> gpurun_out/r2c22_pipe.log
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -x -q > gpurun_out/r2c22_mp.log 2>&1; echo rc=$? >> gpurun_out/r2c22_mp.log
for f in gpurun_out/r2c22_grid.log gpurun_out/r2c22_pipe.log gpurun_out/r2c22_mp.log; do tail -n 3 $f; done
