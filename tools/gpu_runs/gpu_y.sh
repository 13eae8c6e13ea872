#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_y.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_y.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_y.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_y.json 2> gpurun_out/bench_y.err
for W in rmc2 cfg5-din cfg5-dien mt-wnd; do
  timeout 900 python tools/env_sweep.py --workload $W --reps 2 --n 2048 "RS_X=0" > gpurun_out/pol_$W.json 2>> gpurun_out/pol.err
done
