mkdir -p gpurun_out/waves
timeout 600 python tools/sls_iso.py --sizes 128,322,500,1000 "RS_SLS_WAVES=2" "RS_SLS_WAVES=1" "RS_SLS_WAVES=3" "RS_SLS_WAVES=4" 2>&1 | tail -6 | tee gpurun_out/waves/iso.log
timeout 600 python tools/env_sweep.py --workload cfg3-rmc2 --depth 16 --reps 3 "RS_SLS_WAVES=2" "RS_SLS_WAVES=1" 2>&1 | tail -1 | tee gpurun_out/waves/pipe.log
