#!/bin/bash
# One GPU-box session: full GPU test suite, smoke, 1-GPU bench, real-time serve,
# reference arm. Outputs land in gpurun_out/ (merged back by gpurun).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "all rc=$?" >> gpurun_out/pytest_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --serve --gpus 1 > gpurun_out/serve1.json 2> gpurun_out/serve1.err; echo "serve rc=$?" >> gpurun_out/serve1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?" >> gpurun_out/ref.err
