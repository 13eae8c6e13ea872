#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "cfg3 or benched or zoo or tf32" > gpurun_out/pytest_u.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_u.log
timeout 1200 python tools/env_sweep.py --reps 3 --n 4096 "RS_DISCARD=0" "RS_DISCARD=1" > gpurun_out/env_discard.json 2> gpurun_out/env_discard.err
timeout 900 ncu --replay-mode app-range --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum python tools/range_traffic.py --n 256 > gpurun_out/range_discard.csv 2> gpurun_out/range_discard.err
