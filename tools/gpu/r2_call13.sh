set -x
python bench.py --workload c4 --order 8 --nt 200 --no-extra --steps 2 --warmup 1 > gpurun_out/r2c13_c4p8.log 2>&1
python bench.py --workload c4 --order 1 --no-extra --steps 3 --warmup 2 > gpurun_out/r2c13_c4p1.log 2>&1
python tools/sweep.py --exps 22,24,26 --orders 1 --nt 200 > gpurun_out/r2c13_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_febe_carry -c 1 -o gpurun_out/r2_ncu_carry_c2 python bench.py --no-extra --steps 1 --warmup 0 --cpu-budget 1 > gpurun_out/r2c13_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_febe -s 5 -c 1 -o gpurun_out/r2_ncu_sweep_2p24 python tools/sweep.py --exps 24 --orders 1 --nt 20 --reps 1 > gpurun_out/r2c13_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep2d_febe -s 5 -c 1 -o gpurun_out/r2_ncu_sweep2d_c3 python bench.py --workload c3 --nt 20 --no-extra --steps 1 --warmup 0 --cpu-budget 1 > gpurun_out/r2c13_ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep2d_levels -s 12 -c 1 -o gpurun_out/r2_ncu_sweeplev_c3p4 python bench.py --workload c3 --order 4 --nt 20 --no-extra --steps 1 --warmup 0 --cpu-budget 1 > gpurun_out/r2c13_ncu4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-extra --cpu-budget 1 > gpurun_out/r2c13_ncu5.log 2>&1
ls -la gpurun_out | tail -12
