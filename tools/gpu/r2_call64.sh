set -x
RIDC_CHECKED=1 timeout 1500 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q > gpurun_out/r2c64_checked_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c64_checked_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_febe_wcarry -c 1 -o gpurun_out/r2_ncu_wcarry_bench python bench.py --steps 1 --warmup 0 --no-extra --cpu-budget 1 > gpurun_out/r2c64_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_carry_res2w -s 1 -c 1 -o gpurun_out/r2_ncu_res2w_c2 python tools/sweep.py --exps 20 --orders 2 --nt 1000 --reps 1 > gpurun_out/r2c64_ncu2.log 2>&1
tail -n 3 gpurun_out/r2c64_checked_tests.log; ls gpurun_out/*.ncu-rep
