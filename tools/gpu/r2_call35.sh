set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_febe_wcarry -c 1 -o gpurun_out/r2_ncu_wcarry_c2 python bench.py --no-extra --steps 1 --warmup 0 --cpu-budget 1 > gpurun_out/r2c35_ncu1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c2_wcarry.csv python bench.py --steps 2 --warmup 1 --no-extra --cpu-budget 1 > gpurun_out/r2c35_ncu2.log 2>&1
tail -n 3 gpurun_out/r2c35_ncu1.log gpurun_out/r2c35_ncu2.log; head -5 gpurun_out/r2_launches_c2_wcarry.csv
