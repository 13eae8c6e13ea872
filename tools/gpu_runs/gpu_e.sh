#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "tf32 or benched or auto or hybrid or cfg1 or zoo_fp32" > gpurun_out/pytest_e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e.log
timeout 900 python tools/pipe_diag.py --depths 8 --skips 0,2,7 > gpurun_out/pipe_diag_e.json 2> gpurun_out/pipe_diag_e.err
RS_INTER_TC=0 timeout 900 python tools/pipe_diag.py --depths 8 --skips 0 > gpurun_out/pipe_diag_e0.json 2>> gpurun_out/pipe_diag_e.err
timeout 900 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
