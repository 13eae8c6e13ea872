#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 8 "RS_X=0" > gpurun_out/aa_base.json 2>> gpurun_out/aa.err
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 8 "RS_CARVEOUT_FUNC=50" > gpurun_out/aa_func50.json 2>> gpurun_out/aa.err
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 --depth 8 "RS_CARVEOUT=0,RS_CARVEOUT_FUNC=50,RS_TC_CFG=0" > gpurun_out/aa_func50_cfg0.json 2>> gpurun_out/aa.err
timeout 900 python -c "
import sys; sys.path.insert(0,'.')
import ctypes, os
import torch
os.environ['RS_CARVEOUT_FUNC']='50'
" 2>/dev/null
