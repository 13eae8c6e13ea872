#!/bin/bash
mkdir -p gpurun_out
run() { timeout 900 python tools/env_sweep.py --reps 2 --n 4096 "$1" > gpurun_out/carve_$2.json 2>> gpurun_out/carve.err; }
run "RS_X=0" base
run "RS_TC_CFG=0" cfg0
run "RS_CARVEOUT=50" c50
run "RS_CARVEOUT=50,RS_TC_CFG=0" c50_cfg0
run "RS_CARVEOUT=58,RS_TC_CFG=0" c58_cfg0
run "RS_CARVEOUT=100" c100
