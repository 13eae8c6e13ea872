#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "all rc=$?" >> gpurun_out/pytest_all.log
timeout 900 python bench.py --serve --gpus 2 > gpurun_out/serve2.json 2> gpurun_out/serve2.err
timeout 900 python tools/pipe_diag.py --depths 8,16 --skips 0,1,2,4,7 > gpurun_out/pipe_diag.json 2> gpurun_out/pipe_diag.err
for B in 16 64 256; do
  for SK in 2 4; do
    RS_LIB_VARIANT=exp RS_SPLITK=$SK timeout 600 python bench.py --workload mt-wnd --size-fixed $B --max-query 1024 --no-cpu --steps 10 --warmup 3 > gpurun_out/bsweep_sk${SK}_$B.json 2>> gpurun_out/bsweep_sk.err
  done
done
