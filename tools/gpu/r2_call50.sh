set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep2d_febe -s 5 -c 1 -o gpurun_out/r2_ncu_sweep2d_c3_final python bench.py --workload c3 --nt 20 --no-extra --steps 1 --warmup 0 --cpu-budget 1 > gpurun_out/r2c50_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep2d_levels -s 12 -c 1 -o gpurun_out/r2_ncu_sweeplev_c3p4_final python bench.py --workload c3 --order 4 --nt 20 --no-extra --steps 1 --warmup 0 --cpu-budget 1 > gpurun_out/r2c50_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_levels -s 12 -c 1 -o gpurun_out/r2_ncu_sweeplev1d_2p24 python tools/sweep.py --exps 24 --orders 4 --nt 20 --reps 1 > gpurun_out/r2c50_ncu3.log 2>&1
ls gpurun_out/*final* gpurun_out/*1d_2p24*
