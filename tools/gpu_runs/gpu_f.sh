#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "tf32 or benched or auto or hybrid or cfg1 or zoo_fp32" > gpurun_out/pytest_f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f.log
RS_INTER_TC=0 timeout 600 python tools/timeline.py --n 128 --pool 128 --trace gpurun_out/tl_skip0.json > gpurun_out/tl_skip0.sum 2>&1
RS_INTER_TC=0 RS_DIAG_SKIP=2 timeout 600 python tools/timeline.py --n 128 --pool 128 --trace gpurun_out/tl_skip2.json > gpurun_out/tl_skip2.sum 2>&1
RS_INTER_TC=0 RS_DIAG_SKIP=7 timeout 600 python tools/timeline.py --n 128 --pool 128 --trace gpurun_out/tl_skip7.json > gpurun_out/tl_skip7.sum 2>&1
