#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 8 "RS_X=0" > gpurun_out/ab_on_$r.json 2>> gpurun_out/ab.err
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 8 "RS_CARVEOUT=0" > gpurun_out/ab_off_$r.json 2>> gpurun_out/ab.err
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 8 "RS_CARVEOUT=0,RS_DISCARD=0" > gpurun_out/ab_r1_$r.json 2>> gpurun_out/ab.err
done
