#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/f_bench_n4.json 2> gpurun_out/f_bench_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/f_bench_n2.json 2> gpurun_out/f_bench_n2.err
timeout 900 python bench.py --serve --gpus 4 > gpurun_out/f_serve4.json 2> gpurun_out/f_serve4.err
timeout 900 python bench.py --serve --gpus 2 > gpurun_out/f_serve2.json 2> gpurun_out/f_serve2.err
timeout 900 python bench.py --serve --gpus 1 > gpurun_out/f_serve1.json 2> gpurun_out/f_serve1.err
timeout 900 python bench.py --impl reference --gpus 4 --steps 5 --warmup 3 > gpurun_out/f_ref_n4.json 2> gpurun_out/f_ref_n4.err
