set -x
python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2c11_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c11_gpu_tests.log
python bench.py > gpurun_out/r2c11_bench.log 2>&1; echo rc=$? >> gpurun_out/r2c11_bench.log
python tools/sweep.py --exps 16,18,20,22,24,26 --orders 1,2,4,8 --nt 200 --out gpurun_out/r2c11_sweep.json > gpurun_out/r2c11_sweep.log 2>&1
tail -3 gpurun_out/r2c11_gpu_tests.log
