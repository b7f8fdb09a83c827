set -x
python -m pytest tests/test_gpu_resident.py -x -q -k sweep > gpurun_out/r2c5_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c5_tests.log
RIDC_SWEEP_NT=256 python tools/sweep.py --exps 22,24,26 --orders 1 --nt 200 > gpurun_out/r2c5_sweep256.log 2>&1
RIDC_SWEEP_NT=512 python tools/sweep.py --exps 22,24,26 --orders 1 --nt 200 > gpurun_out/r2c5_sweep512.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_febe -s 3 -c 1 -o gpurun_out/r2_sweep256 python tools/sweep.py --exps 24 --orders 1 --nt 20 --reps 1 > gpurun_out/r2c5_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_febe_carry -s 1 -c 1 -o gpurun_out/r2_carry python tools/sweep.py --exps 20 --orders 1 --nt 200 --reps 1 > gpurun_out/r2c5_ncu2.log 2>&1
ls -la gpurun_out/
