set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --nt 400 > gpurun_out/r2c32_n2.json 2> gpurun_out/r2c32_n2.err; echo rc=$? >> gpurun_out/r2c32_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 2 --warmup 1 --nt 400 > gpurun_out/r2c32_n4.json 2> gpurun_out/r2c32_n4.err; echo rc=$? >> gpurun_out/r2c32_n4.err
timeout 300 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/r2c32_ref.json 2>&1
cut -c1-600 gpurun_out/r2c32_n2.json gpurun_out/r2c32_n4.json; tail -n 2 gpurun_out/r2c32_n2.err gpurun_out/r2c32_n4.err
