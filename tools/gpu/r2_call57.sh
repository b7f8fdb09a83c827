set -x
cp tools/gpu/par53.py /tmp/par53.py
for E in 8; do RIDC_WC_EXP=$E timeout 600 python /tmp/par53.py > gpurun_out/r2c57_par$E.log 2>&1; done
RIDC_WCARRY_K=32 timeout 600 python /tmp/par53.py > gpurun_out/r2c57_park32.log 2>&1
for E in 0 8 1 9; do RIDC_WC_EXP=$E timeout 600 python tools/sweep.py --exps 17,18,19,20 --orders 1 --nt 2000 --reps 5 > gpurun_out/r2c57_wc$E.log 2>&1; done
for E in 0 8 1; do RIDC_WCARRY_K=32 RIDC_WC_EXP=$E timeout 600 python tools/sweep.py --exps 18,19,20 --orders 1 --nt 2000 --reps 5 > gpurun_out/r2c57_k32_wc$E.log 2>&1; done
for E in 0 8; do RIDC_WC_EXP=$E timeout 600 python tools/sweep.py --exps 20 --orders 1 --nt 10000 --reps 5 > gpurun_out/r2c57_c2_wc$E.log 2>&1; done
cat gpurun_out/r2c57_par*.log
