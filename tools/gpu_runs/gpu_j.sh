#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "sls or bit_exact or cfg3 or benched or l2_hot or forward_many or merged or queue" > gpurun_out/pytest_j.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_j.log
timeout 900 python tools/sls_iso.py "RS_SLS_DYN=0" "RS_SLS_DYN=1" "RS_SLS_DYN=1,RS_SLS_WAVES=2" > gpurun_out/sls_iso_j.json 2> gpurun_out/sls_iso_j.err
timeout 1200 python tools/env_sweep.py --reps 3 "RS_SLS_DYN=0" "RS_SLS_DYN=1" "RS_SLS_DYN=1,RS_SLS_WAVES=2" > gpurun_out/env_j.json 2> gpurun_out/env_j.err
