set -x
timeout 1200 python -m pytest tests/test_gpu_resident.py tests/test_gpu_ark.py -x -q > gpurun_out/r2c71_t.log 2>&1; echo rc=$? >> gpurun_out/r2c71_t.log
for i in 1 2; do timeout 900 python tools/sweep.py --exps 18,19,20 --orders 3,4,8 --nt 200 > gpurun_out/r2c71_sweep$i.log 2>&1; done
timeout 600 python bench.py > gpurun_out/r2c71_bench.log 2>&1
tail -n 2 gpurun_out/r2c71_t.log
