set -x
nproc; free -g | head -2
python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2c2_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c2_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c2_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2c2_smoke.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/r2c2_memcheck.log 2>&1; echo rc=$? >> gpurun_out/r2c2_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py > gpurun_out/r2c2_synccheck.log 2>&1; echo rc=$? >> gpurun_out/r2c2_synccheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py --cases febe-whole,febe-seg,tick-seg-p3,levels-seg-p3,tick-2d-p2 > gpurun_out/r2c2_racecheck.log 2>&1; echo rc=$? >> gpurun_out/r2c2_racecheck.log
python bench.py > gpurun_out/r2c2_bench.log 2>&1; echo rc=$? >> gpurun_out/r2c2_bench.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --nt 200 --no-extra > gpurun_out/r2c2_bench_g2.log 2>&1; echo rc=$? >> gpurun_out/r2c2_bench_g2.log
tail -3 gpurun_out/r2c2_gpu_tests.log
