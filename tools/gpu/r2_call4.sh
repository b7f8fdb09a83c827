set -x
python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/r2c4_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c4_tests.log
python tools/sweep.py --exps 20,21,22,24,26 --orders 1 --nt 200 > gpurun_out/r2c4_sweep.log 2>&1
RIDC_NO_SWEEP=1 python tools/sweep.py --exps 22,24,26 --orders 1 --nt 200 > gpurun_out/r2c4_sweep_tick.log 2>&1
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c5_sweep_sizes and 1-2" >> gpurun_out/r2c4_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c4_tests.log
tail -3 gpurun_out/r2c4_tests.log
