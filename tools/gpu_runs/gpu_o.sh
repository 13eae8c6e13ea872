#!/bin/bash
mkdir -p gpurun_out
for TL in "32 80" "64 40" "128 20" "16 160"; do
  set -- $TL
  timeout 600 python tools/sls_micro.py --T $1 --L $2 --variants 2:0:4 --sizes 64,330,1000 --rows 2000000 > gpurun_out/slsL_$1_$2.json 2>> gpurun_out/slsL.err
done
