#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v.log
timeout 1200 python tools/env_sweep.py --reps 3 --n 4096 "RS_DISCARD=0" "RS_DISCARD=1" > gpurun_out/env_discard2.json 2> gpurun_out/env_discard2.err
timeout 900 ncu --replay-mode app-range --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum python tools/range_traffic.py --n 256 > gpurun_out/range_discard2.csv 2> gpurun_out/range_discard2.err
for W in rmc1 mt-wnd cfg5-din; do
timeout 900 python tools/env_sweep.py --workload $W --reps 2 --n 2048 "RS_DISCARD=0" "RS_DISCARD=1" > gpurun_out/env_discard_$W.json 2>> gpurun_out/env_discard2.err
done
