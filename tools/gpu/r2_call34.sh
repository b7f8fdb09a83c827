set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "warp_carry or equals_tick" > gpurun_out/r2c34_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c34_tests.log
timeout 600 python tools/sweep.py --exps 16,18,19,20 --orders 1 --nt 2000 > gpurun_out/r2c34_sweep.log 2>&1
RIDC_NO_WCARRY=1 timeout 600 python tools/sweep.py --exps 16,18,19,20 --orders 1 --nt 2000 > gpurun_out/r2c34_sweep_tile.log 2>&1
python bench.py --no-extra --steps 5 --warmup 3 > gpurun_out/r2c34_bench.json 2>&1
for f in gpurun_out/r2c34_tests.log gpurun_out/r2c34_sweep.log gpurun_out/r2c34_sweep_tile.log; do tail -n 5 $f | cut -c1-200; done; cut -c1-400 gpurun_out/r2c34_bench.json
