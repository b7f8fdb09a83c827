set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "warp_carry or equals_tick or res2 or carry_levels" > gpurun_out/r2c36_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c36_tests.log
timeout 600 python tools/sweep.py --exps 18,20 --orders 1,2,4 --nt 1000 > gpurun_out/r2c36_sweep.log 2>&1
RIDC_NO_WCARRY=1 timeout 600 python tools/sweep.py --exps 20 --orders 1 --nt 1000 > gpurun_out/r2c36_sweep_tile.log 2>&1
for f in gpurun_out/r2c36_tests.log gpurun_out/r2c36_sweep.log gpurun_out/r2c36_sweep_tile.log; do tail -n 7 $f | cut -c1-160; done
