set -x
python tools/sweep.py --exps 20 --orders 2,4 --nt 400 > gpurun_out/r2c24_cl.log 2>&1
RIDC_CL_EXP=1 python tools/sweep.py --exps 20 --orders 2,4 --nt 400 > gpurun_out/r2c24_cl_exp1.log 2>&1
cut -c1-200 gpurun_out/r2c24_cl.log gpurun_out/r2c24_cl_exp1.log
