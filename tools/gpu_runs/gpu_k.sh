#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -k "bf16" > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 900 python tools/parity_report.py > gpurun_out/parity_r2.json 2> gpurun_out/parity_r2.err
timeout 600 python bench.py --workload mt-wnd --fc bf16 --no-cpu --steps 20 --warmup 5 > gpurun_out/bench_mtwnd_bf16.json 2> gpurun_out/bench_mtwnd_bf16.err
timeout 600 python bench.py --workload mt-wnd --no-cpu --steps 20 --warmup 5 > gpurun_out/bench_mtwnd_auto.json 2>> gpurun_out/bench_mtwnd_bf16.err
timeout 600 python bench.py --fc bf16 --no-cpu --steps 20 --warmup 5 > gpurun_out/bench_cfg3_bf16.json 2>> gpurun_out/bench_mtwnd_bf16.err
timeout 600 python bench.py --workload wnd --fc bf16 --no-cpu --steps 20 --warmup 5 > gpurun_out/bench_wnd_bf16.json 2>> gpurun_out/bench_mtwnd_bf16.err
