#!/bin/bash
mkdir -p gpurun_out
for C in 50 58 72 86; do
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 8 "RS_CARVEOUT=$C" > gpurun_out/ac_c$C.json 2>> gpurun_out/ac.err
done
