set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2c17_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2c17_gputests.log
python bench.py > gpurun_out/r2c17_bench.json 2> gpurun_out/r2c17_bench.err; echo rc=$? >> gpurun_out/r2c17_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2c17_ref.json 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c17_smoke.log 2>&1
tail -3 gpurun_out/r2c17_gputests.log; tail -2 gpurun_out/r2c17_bench.err; cut -c1-600 gpurun_out/r2c17_bench.json
