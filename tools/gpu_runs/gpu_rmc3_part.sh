export RS_LIB_VARIANT=exp
timeout 900 python tools/env_sweep.py --workload cfg3-rmc3 --depth 16 --reps 2 "RS_X=default" "RS_CARVEOUT=0" "RS_CARVEOUT=0,RS_DENSE_SMS=80" "RS_CARVEOUT=0,RS_DENSE_SMS=96" "RS_CARVEOUT=0,RS_DENSE_SMS=112" "RS_CARVEOUT=0,RS_DENSE_SMS=80,RS_TC2_CAPPED=0" 2>&1 | tail -1
