set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2c52_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c52_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c52_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2c52_bench.log 2>&1
tail -3 gpurun_out/r2c52_tests.log; tail -1 gpurun_out/r2c52_smoke.log; tail -c 600 gpurun_out/r2c52_bench.log
