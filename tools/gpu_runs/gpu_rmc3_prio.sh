timeout 900 python tools/env_sweep.py --workload cfg3-rmc3 --depth 16 --reps 3 "RS_X=default" "RS_PRIO=0" "RS_PDL=0" 2>&1 | tail -1
timeout 900 python tools/env_sweep.py --workload cfg3-rmc3 --depth 8 --reps 3 "RS_X=default" 2>&1 | tail -1
