for x in 0 1 2 4 3; do echo "== exp $x"; RIDC_SWEEP_EXP=$x RIDC_SWEEP_NT=256 python tools/det_check.py --n 8388608 --reps 4 2>&1 | tail -3; done > gpurun_out/r2c9_det.log 2>&1
cat gpurun_out/r2c9_det.log
