set -x
python -m pytest tests/test_gpu_resident.py -x -q -k "sweep_febe" > gpurun_out/r2c18_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c18_tests.log
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c5" >> gpurun_out/r2c18_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c18_tests.log
python tools/sweep.py --exps 20,21,22,23,24,26 --orders 1 --nt 200 > gpurun_out/r2c18_sweep_warp.log 2>&1
RIDC_SWEEP_CTA=1 python tools/sweep.py --exps 22,24,26 --orders 1 --nt 200 > gpurun_out/r2c18_sweep_cta.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_febe_warp -s 5 -c 1 -o gpurun_out/r2_ncu_sweepwarp_2p24 python tools/sweep.py --exps 24 --orders 1 --nt 20 --reps 1 > gpurun_out/r2c18_ncu.log 2>&1
tail -3 gpurun_out/r2c18_tests.log; cat gpurun_out/r2c18_sweep_warp.log gpurun_out/r2c18_sweep_cta.log | cut -c1-200
