#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "zoo or tf32 or benched" > gpurun_out/ae_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ae_pytest.log
timeout 1800 python tools/sweep.py --out gpurun_out/ae_sweep --steps 10 --warmup 3 --workloads rmc3,cfg3-rmc3 > gpurun_out/ae_sweep.log 2>&1
