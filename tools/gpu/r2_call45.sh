RIDC_WCARRY_K=32 timeout 600 python tools/sweep.py --exps 18,19,20 --orders 1 --nt 2000 > gpurun_out/r2c45_k32.log 2>&1
timeout 600 python tools/sweep.py --exps 18,19,20 --orders 1 --nt 2000 > gpurun_out/r2c45_k16.log 2>&1
cut -c1-130 gpurun_out/r2c45_k32.log gpurun_out/r2c45_k16.log
