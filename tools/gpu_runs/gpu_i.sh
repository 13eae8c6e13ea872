#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --serve --gpus 4 > gpurun_out/serve4.json 2> gpurun_out/serve4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
