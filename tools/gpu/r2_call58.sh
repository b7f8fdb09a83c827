set -x
timeout 1200 python -m pytest tests/test_gpu_resident.py -x -q -k "res2 or carry or default" > gpurun_out/r2c58_t.log 2>&1; echo rc=$? >> gpurun_out/r2c58_t.log
for L in 0 1 0; do RIDC_RES2_LATE=$L timeout 600 python tools/sweep.py --exps 16,17,18,19,20 --orders 2 --nt 2000 --reps 5 > gpurun_out/r2c58_res2_late$L.log 2>&1; done
timeout 600 python tools/sweep.py --exps 20 --orders 1 --nt 2000 --reps 5 > gpurun_out/r2c58_wc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_febe_wcarry -s 1 -c 1 -o gpurun_out/r2_ncu_wcarry_early python tools/sweep.py --exps 20 --orders 1 --nt 1000 --reps 1 > gpurun_out/r2c58_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_carry_res2 -s 1 -c 1 -o gpurun_out/r2_ncu_res2_early python tools/sweep.py --exps 20 --orders 2 --nt 1000 --reps 1 > gpurun_out/r2c58_ncu2.log 2>&1
tail -2 gpurun_out/r2c58_t.log; ls gpurun_out/*.ncu-rep
