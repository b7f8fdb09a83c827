set -x
cp tools/gpu/par53.py /tmp/par53.py
timeout 600 python /tmp/par53.py > gpurun_out/r2c59_par.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q > gpurun_out/r2c59_t.log 2>&1; echo rc=$? >> gpurun_out/r2c59_t.log
for E in 0 2 1; do RIDC_WC_EXP=$E timeout 600 python tools/sweep.py --exps 16,17,18,19,20,21 --orders 1 --nt 2000 --reps 5 > gpurun_out/r2c59_wc$E.log 2>&1; done
for L in 0 1 2; do RIDC_RES2_LATE=$L timeout 600 python tools/sweep.py --exps 16,17,18,19,20 --orders 2 --nt 2000 --reps 5 > gpurun_out/r2c59_res2_$L.log 2>&1; done
timeout 600 python bench.py > gpurun_out/r2c59_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_febe_wcarry -s 1 -c 1 -o gpurun_out/r2_ncu_wcarry_pred python tools/sweep.py --exps 20 --orders 1 --nt 1000 --reps 1 > gpurun_out/r2c59_ncu.log 2>&1
cat gpurun_out/r2c59_par.log | grep tick; tail -2 gpurun_out/r2c59_t.log; tail -c 300 gpurun_out/r2c59_bench.log
