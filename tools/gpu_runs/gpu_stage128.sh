for w in cfg3-rmc2 rmc2; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_X=default" "RS_STAGE_THREADS=128" "RS_STAGE_THREADS=128,RS_STAGE_CTAS=148" "RS_DIAG_SKIP=1" "RS_DIAG_SKIP=4" "RS_DIAG_SKIP=7" 2>&1 | tail -1 | sed "s/^/$w /"
done
