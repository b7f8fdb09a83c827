set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2c47_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2c47_gputests.log
python bench.py > gpurun_out/r2c47_bench.json 2> gpurun_out/r2c47_bench.err; echo rc=$? >> gpurun_out/r2c47_bench.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c47_smoke.log 2>&1
tail -n 3 gpurun_out/r2c47_gputests.log; tail -n 2 gpurun_out/r2c47_bench.err; cut -c1-300 gpurun_out/r2c47_bench.json
