#!/bin/bash
# Wide graph (CTA-pair FC tiles): parity, then per-size / stream A/B against RS_TC2=0
mkdir -p gpurun_out/tc2
timeout 900 python -m pytest tests/test_gpu_parity_benched.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/tc2/parity.log
for w in mt-wnd wnd; do for fc in auto bf16; do
  for S in 0 256 640 700 1000; do
    extra=""; [ $S -gt 0 ] && extra="--size-fixed $S"
    timeout 200 python tools/env_sweep.py --workload $w --fc $fc --reps 3 $extra "RS_TC2=0" "RS_X=1" 2>&1 | tail -1 | sed "s/^/$w $fc S=$S /"
  done
done; done | tee gpurun_out/tc2/ab.log
