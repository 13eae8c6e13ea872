#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "all rc=$?" >> gpurun_out/pytest_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 3 --warmup 3 --queries-per-step 32 --no-cpu > gpurun_out/ncu_launch.log 2>&1
TP_FC=bf16 timeout 1200 python tools/tensor_profile.py > gpurun_out/r2_tensor_pipe_bf16.json 2> gpurun_out/tensor_bf16.err
timeout 900 python bench.py --serve --gpus 1 --workload rmc1 --size-median 30 --hybrid-threshold 32 --cpu-batch 16 --serve-n 20000 > gpurun_out/hybrid_rmc1_t32.json 2> gpurun_out/hybrid.err
timeout 900 python bench.py --serve --gpus 1 --workload rmc1 --size-median 30 --serve-n 20000 > gpurun_out/hybrid_rmc1_gpu.json 2>> gpurun_out/hybrid.err
