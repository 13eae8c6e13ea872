#!/bin/bash
mkdir -p gpurun_out
for W in mt-wnd wnd ncf; do
for C in 0 100; do
timeout 900 python tools/env_sweep.py --workload $W --reps 2 --n 2048 "RS_CARVEOUT=$C" > gpurun_out/ad_${W}_c$C.json 2>> gpurun_out/ad.err
done
done
