#!/bin/bash
# 2-GPU box: real-time serving at 1 and 2 replicas, torchrun N=2 bench,
# configs[3] batch sweep (MT-WND fixed sizes), configs[2] threshold sweep.
mkdir -p gpurun_out
timeout 900 python bench.py --serve --gpus 1 --serve-inputs device > gpurun_out/serve1_dev.json 2> gpurun_out/serve.err
timeout 900 python bench.py --serve --gpus 2 > gpurun_out/serve2.json 2>> gpurun_out/serve.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
for B in 16 32 64 128 256 512 1024; do
  timeout 600 python bench.py --workload mt-wnd --size-fixed $B --max-query 1024 --no-cpu --steps 10 --warmup 3 > gpurun_out/bsweep_$B.json 2>> gpurun_out/bsweep.err
done
RS_B200_ROWS=10000000 timeout 2400 python tools/cfg3_sweep.py > gpurun_out/r2_cfg3_threshold_sweep.json 2> gpurun_out/cfg3_sweep.err
