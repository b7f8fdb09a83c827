set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2 or default" > gpurun_out/r2c67_t.log 2>&1; echo rc=$? >> gpurun_out/r2c67_t.log
timeout 600 python tools/sweep.py --exps 16,17,18,19,20 --orders 2 --nt 2000 --reps 5 > gpurun_out/r2c67_res2.log 2>&1
timeout 600 python bench.py > gpurun_out/r2c67_bench.log 2>&1
tail -n 2 gpurun_out/r2c67_t.log
