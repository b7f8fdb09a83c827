set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2 or default" > gpurun_out/r2c62_t.log 2>&1; echo rc=$? >> gpurun_out/r2c62_t.log
RIDC_RES2W_EARLY=1 timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2" > gpurun_out/r2c62_t1.log 2>&1; echo rc=$? >> gpurun_out/r2c62_t1.log
RIDC_RES2W_EARLY=0 timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2" > gpurun_out/r2c62_t0.log 2>&1; echo rc=$? >> gpurun_out/r2c62_t0.log
for V in "RIDC_RES2_TILE=1" "RIDC_RES2W_EARLY=1" "RIDC_RES2W_EARLY=0" "RIDC_RES2_TILE=0"; do env $V timeout 600 python tools/sweep.py --exps 16,17,18,19,20 --orders 2 --nt 2000 --reps 5 > gpurun_out/r2c62_res2_$V.log 2>&1; done
tail -2 gpurun_out/r2c62_t.log gpurun_out/r2c62_t1.log gpurun_out/r2c62_t0.log
