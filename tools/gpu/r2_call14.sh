set -x
python -m pytest tests/test_gpu_resident.py tests/test_gpu_trajectory.py tests/test_gpu_edges.py -x -q > gpurun_out/r2c14_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c14_tests.log
python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "c2_febe" >> gpurun_out/r2c14_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c14_tests.log
python tools/det_check.py --n 1048576 --steps 2000 --reps 3 > gpurun_out/r2c14_det.log 2>&1
python bench.py --no-extra --steps 10 --warmup 3 > gpurun_out/r2c14_bench.log 2>&1
tail -3 gpurun_out/r2c14_tests.log; cat gpurun_out/r2c14_det.log
