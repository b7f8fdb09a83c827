set -x
timeout 900 python bench.py --workload c4 --order 8 --nt 200 --no-extra --steps 2 --warmup 1 --cpu-budget 4 > gpurun_out/r2c25_c4p8.json 2> gpurun_out/r2c25_c4p8.err
timeout 900 python bench.py --workload c4 --order 1 --nt 200 --no-extra --steps 3 --warmup 2 --cpu-budget 4 > gpurun_out/r2c25_c4p1.json 2> gpurun_out/r2c25_c4p1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep2d_levels -s 40 -c 1 -o gpurun_out/r2_ncu_sweeplev_c4p8 python bench.py --workload c4 --order 8 --nt 40 --no-extra --steps 1 --warmup 0 --cpu-budget 1 > gpurun_out/r2c25_ncu.log 2>&1
cut -c1-1500 gpurun_out/r2c25_c4p8.json gpurun_out/r2c25_c4p1.json; tail -n 3 gpurun_out/r2c25_c4p8.err
