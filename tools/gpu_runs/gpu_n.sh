#!/bin/bash
mkdir -p gpurun_out
for S in 16 256; do
  timeout 900 python tools/env_sweep.py --workload mt-wnd --size-fixed $S --reps 2 --n 1024 "RS_X=0" "RS_TC_CFG=0" "RS_TC_CFG=1" "RS_TC_CFG=2" "RS_TC_CFG=3" > gpurun_out/env_mtwnd_$S.json 2>> gpurun_out/env_mtwnd.err
  timeout 900 python tools/env_sweep.py --workload mt-wnd --fc bf16 --size-fixed $S --reps 2 --n 1024 "RS_X=0" "RS_TC_CFG=0" "RS_TC_CFG=1" "RS_TC_CFG=2" "RS_TC_CFG=3" > gpurun_out/env_mtwnd_bf16_$S.json 2>> gpurun_out/env_mtwnd.err
done
timeout 900 python tools/env_sweep.py --workload mt-wnd --size-fixed 16 --reps 2 --n 1024 --depth 16 "RS_X=0" > gpurun_out/env_mtwnd_16_d16.json 2>> gpurun_out/env_mtwnd.err
