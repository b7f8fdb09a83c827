set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2c72_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c72_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c72_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2c72_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c72_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2c72_ncu.log 2>&1
tail -n 3 gpurun_out/r2c72_tests.log; tail -n 1 gpurun_out/r2c72_smoke.log
