set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2 or default" > gpurun_out/r2c61_t.log 2>&1; echo rc=$? >> gpurun_out/r2c61_t.log
for T in 0 1; do RIDC_RES2_TILE=$T timeout 600 python tools/sweep.py --exps 16,17,18,19,20 --orders 2 --nt 2000 --reps 5 > gpurun_out/r2c61_res2_tile$T.log 2>&1; done
tail -15 gpurun_out/r2c61_t.log
