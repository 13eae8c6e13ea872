#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 3 --warmup 3 --queries-per-step 32 --no-cpu > gpurun_out/f_ncu.log 2>&1
timeout 3600 python tools/sweep.py --out gpurun_out/f_sweep --steps 10 --warmup 3 > gpurun_out/f_sweep.log 2>&1
