#!/bin/bash
mkdir -p gpurun_out
for W in cfg3-rmc3 rmc1 rmc2 rmc3 cfg1-rmc1 cfg5-din ncf wnd mt-wnd cfg5-dien; do
  timeout 900 python tools/env_sweep.py --workload $W --reps 2 --n 2048 "RS_X=0" > gpurun_out/cv_base_$W.json 2>> gpurun_out/cv.err
  timeout 900 python tools/env_sweep.py --workload $W --reps 2 --n 2048 "RS_CARVEOUT=50,RS_TC_CFG=0" > gpurun_out/cv_c50_$W.json 2>> gpurun_out/cv.err
done
