mkdir -p gpurun_out/fuse
timeout 600 python tools/env_sweep.py --workload cfg3-rmc2 --depth 16 --reps 3 "RS_DIAG_SKIP=0" "RS_DIAG_SKIP=2" "RS_DIAG_SERIAL=1" "RS_DIAG_SERIAL=1,RS_DIAG_SKIP=2" "RS_DIAG_SKIP=7" > gpurun_out/fuse/diag.log 2>&1
tail -1 gpurun_out/fuse/diag.log
