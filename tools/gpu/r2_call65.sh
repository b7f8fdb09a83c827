set -x
for n in 1048576 262144 4608 528896; do timeout 600 python tools/det_check.py --levels 2 --n $n --steps 300 --reps 8 > gpurun_out/r2c65_det2_$n.log 2>&1; done
for n in 1048576 2097152 65536; do timeout 600 python tools/det_check.py --levels 1 --n $n --steps 1000 --reps 6 > gpurun_out/r2c65_det1_$n.log 2>&1; done
RIDC_WCARRY_K=32 timeout 600 python tools/det_check.py --levels 1 --n 1048576 --steps 1000 --reps 6 > gpurun_out/r2c65_det1_k32.log 2>&1
cat gpurun_out/r2c65_det*.log
