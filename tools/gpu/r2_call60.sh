set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2c60_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c60_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c60_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2c60_bench.log 2>&1
timeout 900 python tools/sweep.py --exps 16,17,18,19,20,21 --orders 1,2,4,8 --nt 200 > gpurun_out/r2c60_sweep.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c60_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2c60_ncu.log 2>&1
tail -3 gpurun_out/r2c60_tests.log; tail -1 gpurun_out/r2c60_smoke.log; tail -c 300 gpurun_out/r2c60_bench.log
