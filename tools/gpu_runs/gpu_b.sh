#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -k "breakdown or adapter or reference" > gpurun_out/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.log
timeout 900 python bench.py --workload mt-wnd --no-cpu --steps 20 --warmup 5 > gpurun_out/bench_mtwnd.json 2> gpurun_out/bench_mtwnd.err
timeout 900 python bench.py --workload mt-wnd --no-cpu --fc fp32 --steps 20 --warmup 5 > gpurun_out/bench_mtwnd_fp32.json 2>> gpurun_out/bench_mtwnd.err
timeout 900 python bench.py --no-cpu --fc fp32 --steps 20 --warmup 5 > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err
timeout 1500 python tools/tensor_profile.py > gpurun_out/r2_tensor_pipe.json 2> gpurun_out/tensor_profile.err
