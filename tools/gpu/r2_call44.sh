set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "warp_carry or equals_tick or default_selection" > gpurun_out/r2c44_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c44_tests.log
timeout 600 python tools/sweep.py --exps 20,21 --orders 1 --nt 1000 > gpurun_out/r2c44_sweep.log 2>&1
RIDC_NO_WCARRY=1 timeout 600 python tools/sweep.py --exps 21 --orders 1 --nt 1000 > gpurun_out/r2c44_sweep_nowc.log 2>&1
tail -n 3 gpurun_out/r2c44_tests.log; cut -c1-160 gpurun_out/r2c44_sweep.log gpurun_out/r2c44_sweep_nowc.log
