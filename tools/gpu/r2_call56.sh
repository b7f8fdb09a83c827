set -x
cp tools/gpu/par53.py /tmp/par53.py
for E in 0 4; do RIDC_WC_EXP=$E timeout 600 python /tmp/par53.py > gpurun_out/r2c56_par$E.log 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q > gpurun_out/r2c56_t.log 2>&1; echo rc=$? >> gpurun_out/r2c56_t.log
for E in 0 4 2 1; do RIDC_WC_EXP=$E timeout 600 python tools/sweep.py --exps 16,17,18,19,20,21 --orders 1 --nt 2000 --reps 5 > gpurun_out/r2c56_wc$E.log 2>&1; done
timeout 600 python bench.py > gpurun_out/r2c56_bench.log 2>&1
cat gpurun_out/r2c56_par*.log; tail -2 gpurun_out/r2c56_t.log; tail -c 400 gpurun_out/r2c56_bench.log
