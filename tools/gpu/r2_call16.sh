set -x
python -m pytest tests/test_gpu_resident.py -x -q -k "sweep_levels" > gpurun_out/r2c16_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c16_tests.log
python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "c2_orders or 4-2" >> gpurun_out/r2c16_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c16_tests.log
python tools/sweep.py --exps 20,22,24,26 --orders 2,4,8 --nt 200 > gpurun_out/r2c16_sweep.log 2>&1
tail -3 gpurun_out/r2c16_tests.log
