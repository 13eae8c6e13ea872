timeout 600 python tools/env_sweep.py --workload cfg3-rmc2 --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_DIAG_SKIP=7" "RS_DIAG_SKIP=2" 2>&1 | tail -1
