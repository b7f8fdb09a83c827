set -x
cp tools/gpu/par53.py /tmp/par53.py
RIDC_WC_EXP=16 timeout 600 python /tmp/par53.py > gpurun_out/r2c68_par16.log 2>&1
for E in 0 16 0 16; do RIDC_WC_EXP=$E timeout 600 python tools/sweep.py --exps 18,20 --orders 1 --nt 10000 --reps 5 > gpurun_out/r2c68_wc$E.log 2>&1; cat gpurun_out/r2c68_wc$E.log | cut -c1-100 >> gpurun_out/r2c68_all.log; echo "E=$E" >> gpurun_out/r2c68_all.log; done
cat gpurun_out/r2c68_par16.log | grep tick; cat gpurun_out/r2c68_all.log
