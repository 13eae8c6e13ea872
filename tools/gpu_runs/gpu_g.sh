#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "tf32 or benched" > gpurun_out/pytest_g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g.log
timeout 1500 python tools/env_sweep.py "RS_INTER_TC=0" "RS_INTER_CTAS=4" "RS_INTER_CTAS=8" "RS_INTER_CTAS=16" "RS_INTER_CTAS=32" "RS_INTER_CTAS=148" "RS_DIAG_SKIP=2" > gpurun_out/env_inter.json 2> gpurun_out/env_inter.err
