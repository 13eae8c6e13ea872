timeout 600 python tools/env_sweep.py --workload cfg3-rmc3 --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_PDL=0" "RS_DIAG_SERIAL=1" 2>&1 | tail -1
