set -x
cp tools/gpu/par53.py /tmp/par53.py
for E in 0 4 6; do RIDC_WC_EXP=$E timeout 600 python /tmp/par53.py > gpurun_out/r2c54_par$E.log 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_resident.py -x -q -k "carry or res2" > gpurun_out/r2c54_t.log 2>&1; echo rc=$? >> gpurun_out/r2c54_t.log
for E in 0 4 2 6 1; do RIDC_WC_EXP=$E timeout 600 python tools/sweep.py --exps 18,19,20,21 --orders 1 --nt 2000 --reps 5 > gpurun_out/r2c54_wc$E.log 2>&1; done
timeout 900 python tools/sweep.py --exps 18,19,20 --orders 2,3,4,8 --nt 400 --reps 3 > gpurun_out/r2c54_lev.log 2>&1
cat gpurun_out/r2c54_par*.log; tail -2 gpurun_out/r2c54_t.log
