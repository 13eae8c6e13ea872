timeout 600 python tools/env_sweep.py --workload cfg3-rmc2 --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_SLS_UB=8" "RS_SLS_UB=2" "RS_SLS_WPC=4" 2>&1 | tail -1
