for x in 0 16 64 80 5; do echo "== exp $x"; RIDC_SWEEP_EXP=$x RIDC_SWEEP_NT=256 python tools/det_check.py --n 8388608 --reps 4 2>&1 | tail -3; done > gpurun_out/r2c10_det.log 2>&1
echo "== steps 2"; RIDC_SWEEP_NT=256 python tools/det_check.py --n 8388608 --reps 6 --steps 2 >> gpurun_out/r2c10_det.log 2>&1
cat gpurun_out/r2c10_det.log
