set -x
timeout 1500 python tools/sweep.py --exps 16,17,18,19,20,21,22,23,24,25,26 --orders 1,2,4,8 --nt 200 --out gpurun_out/r2_sweep_c5_final.json > gpurun_out/r2c48_sweep.log 2>&1; echo rc=$? >> gpurun_out/r2c48_sweep.log
tail -n 3 gpurun_out/r2c48_sweep.log
