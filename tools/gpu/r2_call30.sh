set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2c30_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2c30_gputests.log
python bench.py > gpurun_out/r2c30_bench.json 2> gpurun_out/r2c30_bench.err; echo rc=$? >> gpurun_out/r2c30_bench.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c30_smoke.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_carry_res2 -c 1 -o gpurun_out/r2_ncu_res2c_c2 python tools/sweep.py --exps 20 --orders 2 --nt 100 --reps 1 > gpurun_out/r2c30_ncu.log 2>&1
tail -n 3 gpurun_out/r2c30_gputests.log; tail -n 2 gpurun_out/r2c30_bench.err; cut -c1-300 gpurun_out/r2c30_bench.json
