set -x
python -m pytest tests/test_gpu_sweep2d.py tests/test_gpu_resident.py tests/test_gpu_trajectory.py tests/test_gpu_parity.py tests/test_gpu_reslevels.py -x -q -s > gpurun_out/r2c12_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c12_tests.log
python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "c3 or c4 or 1-2" > gpurun_out/r2c12_full.log 2>&1; echo rc=$? >> gpurun_out/r2c12_full.log
python tools/det_check.py --n 8388608 --reps 4 > gpurun_out/r2c12_det.log 2>&1
python tools/sweep.py --exps 22,24,26 --orders 1 --nt 200 > gpurun_out/r2c12_sweep.log 2>&1
python bench.py --workload c3 --order 4 --no-extra --steps 2 --warmup 1 > gpurun_out/r2c12_c3p4.log 2>&1
python bench.py --workload c4 --order 8 --nt 200 --no-extra --steps 2 --warmup 1 > gpurun_out/r2c12_c4p8.log 2>&1
tail -3 gpurun_out/r2c12_tests.log gpurun_out/r2c12_full.log; cat gpurun_out/r2c12_det.log
