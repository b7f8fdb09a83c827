set -x
python -m pytest tests/test_gpu_sweep2d.py tests/test_gpu_resident.py -x -q > gpurun_out/r2c8_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c8_tests.log
RIDC_SWEEP_NT=256 python tools/det_check.py --n 8388608 --reps 4 > gpurun_out/r2c8_det.log 2>&1
RIDC_SWEEP_NT=256 python tools/sweep.py --exps 20,22,24,26 --orders 1 --nt 200 > gpurun_out/r2c8_sweep256.log 2>&1
RIDC_SWEEP_NT=512 python tools/sweep.py --exps 22,24,26 --orders 1 --nt 200 > gpurun_out/r2c8_sweep512.log 2>&1
python bench.py --workload c3 --no-extra --steps 3 --warmup 2 > gpurun_out/r2c8_c3.log 2>&1
python bench.py --workload c4 --no-extra --steps 3 --warmup 2 > gpurun_out/r2c8_c4.log 2>&1
python bench.py --no-extra --steps 5 --warmup 3 > gpurun_out/r2c8_c2.log 2>&1
tail -3 gpurun_out/r2c8_tests.log; cat gpurun_out/r2c8_det.log
