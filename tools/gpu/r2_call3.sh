set -x
python -m pytest tests/test_gpu_resident.py tests/test_gpu_edges.py -x -q > gpurun_out/r2c3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c3_tests.log
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2_febe or c5_sweep_sizes and 1-2" >> gpurun_out/r2c3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c3_tests.log
RIDC_NO_CARRY=1 python tools/res_exp.py --nt 2000 > gpurun_out/r2c3_resexp.log 2>&1
python bench.py --no-extra --steps 5 --warmup 3 > gpurun_out/r2c3_bench.log 2>&1
python tools/sweep.py --exps 16,18,20 --orders 1 --nt 2000 > gpurun_out/r2c3_sweep.log 2>&1
tail -3 gpurun_out/r2c3_tests.log; cat gpurun_out/r2c3_resexp.log
