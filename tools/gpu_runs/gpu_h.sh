#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python tools/env_sweep.py --reps 3 "RS_INTER_TC=0,RS_STAGE_CTAS=1000" "RS_INTER_TC=0" "RS_INTER_TC=0,RS_SLS_EF=1" "RS_INTER_TC=1,RS_SLS_EF=1" "RS_INTER_TC=0,RS_PRIO=0" "RS_INTER_TC=0,RS_PDL=0" "RS_INTER_TC=0,RS_TC_WIDE=1" > gpurun_out/env_h.json 2> gpurun_out/env_h.err
