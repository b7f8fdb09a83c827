set -x
RIDC_SWEEP_NT=256 python tools/det_check.py --n 8388608 > gpurun_out/r2c6_det256.log 2>&1
RIDC_SWEEP_NT=512 python tools/det_check.py --n 8388608 > gpurun_out/r2c6_det512.log 2>&1
python tools/det_check.py --kind ad2 --n 4096 --steps 10 --reps 3 > gpurun_out/r2c6_det_ad2.log 2>&1
python -m pytest tests/test_gpu_resident.py tests/test_gpu_fullsize.py -x -q -k "sweep or c3 or c4" > gpurun_out/r2c6_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c6_tests.log
cat gpurun_out/r2c6_det256.log gpurun_out/r2c6_det512.log gpurun_out/r2c6_det_ad2.log; tail -3 gpurun_out/r2c6_tests.log
