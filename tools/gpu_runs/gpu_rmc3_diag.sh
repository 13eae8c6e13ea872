timeout 600 python tools/env_sweep.py --workload cfg3-rmc3 --depth 16 --reps 3 "RS_X=default" "RS_CARVEOUT=0" "RS_DIAG_SKIP=1" "RS_DIAG_SKIP=4" "RS_DIAG_SKIP=7" "RS_DIAG_SKIP=8" 2>&1 | tail -1
