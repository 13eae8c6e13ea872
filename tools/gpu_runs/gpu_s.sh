#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "tf32 or benched or bf16 or zoo" > gpurun_out/pytest_s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_s.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err
timeout 3600 python tools/sweep.py --out gpurun_out/r2_sweep_final --steps 10 --warmup 3 > gpurun_out/sweep_final.log 2>&1
