#!/bin/bash
mkdir -p gpurun_out
for W in cfg3-rmc2 mt-wnd ncf rmc1 cfg5-dien; do
  timeout 900 python tools/env_sweep.py --workload $W --reps 2 --n 1024 --depth 8 "RS_X=0" > gpurun_out/depth8_$W.json 2>> gpurun_out/depth.err
  timeout 900 python tools/env_sweep.py --workload $W --reps 2 --n 1024 --depth 16 "RS_X=0" > gpurun_out/depth16_$W.json 2>> gpurun_out/depth.err
done
