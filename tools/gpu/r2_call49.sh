RIDC_SWEEPLEV_CHUNKS=1 timeout 600 python tools/sweep.py --exps 20,21 --orders 2,4,8 --nt 200 > gpurun_out/r2c49_sl1.log 2>&1
cut -c1-140 gpurun_out/r2c49_sl1.log
