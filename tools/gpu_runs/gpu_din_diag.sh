for w in cfg5-din din cfg1-rmc1 rmc1; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_X=default" "RS_DIAG_SKIP=4" "RS_DIAG_SKIP=7" "RS_PRIO=0" 2>&1 | tail -1 | sed "s/^/$w /"
done
