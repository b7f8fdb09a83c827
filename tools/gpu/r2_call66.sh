set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2 or default" > gpurun_out/r2c66_t.log 2>&1; echo rc=$? >> gpurun_out/r2c66_t.log
RIDC_RES2W_WARPS=14 timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2" > gpurun_out/r2c66_t14.log 2>&1; echo rc=$? >> gpurun_out/r2c66_t14.log
for V in "RIDC_RES2_TILE=1" "RIDC_RES2W_WARPS=7" "RIDC_RES2W_WARPS=14"; do env $V timeout 600 python tools/sweep.py --exps 16,18,19,20 --orders 2 --nt 2000 --reps 5 > gpurun_out/r2c66_res2_$V.log 2>&1; done
tail -n 2 gpurun_out/r2c66_t.log; tail -n 2 gpurun_out/r2c66_t14.log
