set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "res2 or carry_levels" > gpurun_out/r2c26_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c26_tests.log
timeout 600 python tools/sweep.py --exps 18,20 --orders 1,2 --nt 400 > gpurun_out/r2c26_sweep.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_carry_res2 -c 1 -o gpurun_out/r2_ncu_res2_c2 python tools/sweep.py --exps 20 --orders 2 --nt 100 --reps 1 > gpurun_out/r2c26_ncu.log 2>&1
for f in gpurun_out/r2c26_tests.log gpurun_out/r2c26_sweep.log; do tail -n 8 $f | cut -c1-250; done
