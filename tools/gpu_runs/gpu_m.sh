#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/sls_iso.py "RS_SLS_WAVES=1" "RS_SLS_WAVES=2" "RS_SLS_WAVES=3" "RS_SLS_WAVES=4" "RS_SLS_WAVES=6" "RS_SLS_WAVES=2,RS_SLS_UB=8" "RS_SLS_WPC=4" > gpurun_out/sls_iso_m.json 2> gpurun_out/sls_iso_m.err
timeout 1200 python tools/env_sweep.py --reps 2 "RS_SLS_WAVES=2" "RS_SLS_WAVES=4" "RS_SLS_WAVES=6" > gpurun_out/env_m.json 2> gpurun_out/env_m.err
for B in 16 64 256 1024; do
  timeout 600 python bench.py --workload mt-wnd --fc bf16 --size-fixed $B --max-query 1024 --no-cpu --steps 10 --warmup 3 > gpurun_out/bsweep_bf16_$B.json 2>> gpurun_out/bsweep_bf16.err
done
