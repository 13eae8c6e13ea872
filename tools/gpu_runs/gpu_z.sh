#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 8 "RS_X=0" > gpurun_out/pz_d8.json 2>> gpurun_out/pz.err
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 16 "RS_X=0" > gpurun_out/pz_d16.json 2>> gpurun_out/pz.err
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 12 "RS_X=0" > gpurun_out/pz_d12.json 2>> gpurun_out/pz.err
timeout 900 python bench.py --steps 20 --warmup 5 --depth 8 --no-cpu > gpurun_out/bench_z8.json 2> gpurun_out/bench_z.err
