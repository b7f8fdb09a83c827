set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2c63_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c63_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c63_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2c63_bench.log 2>&1
for V in "RIDC_RES2_TILE=1" "RIDC_RES2_TILE=0"; do env $V timeout 600 python tools/sweep.py --exps 16,17,18,19,20 --orders 2 --nt 2000 --reps 5 > gpurun_out/r2c63_res2_$V.log 2>&1; done
tail -n 3 gpurun_out/r2c63_tests.log; tail -n 1 gpurun_out/r2c63_smoke.log
