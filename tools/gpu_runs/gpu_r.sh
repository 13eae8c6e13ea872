#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 "RS_DIAG_SKIP=0" "RS_DIAG_SKIP=7" "RS_DIAG_SKIP=2" > gpurun_out/env_power.json 2> gpurun_out/env_power.err
for S in 256 1024; do
  timeout 900 python tools/env_sweep.py --workload mt-wnd --size-fixed $S --reps 2 --n 1024 "RS_X=0" "RS_TC_CFG=4" > gpurun_out/env_cfg4_$S.json 2>> gpurun_out/env_cfg4.err
  timeout 900 python tools/env_sweep.py --workload mt-wnd --fc bf16 --size-fixed $S --reps 2 --n 1024 "RS_X=0" "RS_TC_CFG=4" > gpurun_out/env_cfg4_bf16_$S.json 2>> gpurun_out/env_cfg4.err
done
timeout 900 python tools/env_sweep.py --workload mt-wnd --reps 2 --n 1024 "RS_X=0" "RS_TC_CFG=4" > gpurun_out/env_cfg4_ln.json 2>> gpurun_out/env_cfg4.err
timeout 900 python bench.py --workload cfg5-dien --rnn augru --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_dien_augru.json 2> gpurun_out/bench_dien_augru.err
timeout 900 python bench.py --workload cfg5-dien --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_dien_gru.json 2>> gpurun_out/bench_dien_augru.err
timeout 900 python bench.py --serve --gpus 1 --workload ncf --size-fixed 1 --serve-inputs device --serve-n 100000 > gpurun_out/serve_dispatch_ncf1.json 2> gpurun_out/serve_dispatch.err
timeout 900 python tools/env_sweep.py --reps 2 --n 4096 "RS_DIAG_SKIP=2" "RS_DIAG_SKIP=2,RS_DIAG_EMPTY=1,RS_DIAG_EMPTY_CTAS=1" "RS_DIAG_SKIP=2,RS_DIAG_EMPTY=1,RS_DIAG_EMPTY_CTAS=296" "RS_DIAG_SKIP=2,RS_DIAG_EMPTY=3,RS_DIAG_EMPTY_CTAS=1" > gpurun_out/env_empty.json 2> gpurun_out/env_empty.err
