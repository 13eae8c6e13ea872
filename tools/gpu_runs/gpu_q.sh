#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_q.log 2>&1; echo "all rc=$?" >> gpurun_out/pytest_q.log
timeout 3000 python tools/sweep.py --out gpurun_out/r2_sweep --steps 10 --warmup 3 > gpurun_out/sweep.log 2>&1
timeout 1500 python tools/sweep.py --out gpurun_out/r2_sweep_bf16 --steps 10 --warmup 3 --workloads mt-wnd,wnd,ncf,cfg5-din,cfg5-dien,cfg3-rmc3 --extra "--fc bf16 --no-cpu" > gpurun_out/sweep_bf16.log 2>&1
