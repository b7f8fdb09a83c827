set -x
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -k "carry_levels" > gpurun_out/r2c20_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c20_tests.log
timeout 600 python tools/sweep.py --exps 17,18,19,20 --orders 2,3,4,8 --nt 200 > gpurun_out/r2c20_sweep_cl.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_carry_levels -s 30 -c 1 -o gpurun_out/r2_ncu_carrylev2_c2p4 python tools/sweep.py --exps 20 --orders 4 --nt 40 --reps 1 > gpurun_out/r2c20_ncu.log 2>&1
tail -4 gpurun_out/r2c20_tests.log; cat gpurun_out/r2c20_sweep_cl.log | cut -c1-150
