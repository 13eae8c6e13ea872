for w in cfg3-rmc2 rmc2 cfg3-rmc3; do
  timeout 300 python tools/env_sweep.py --workload $w --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_INTER_PER_SM=1" "RS_INTER_PER_SM=4" 2>&1 | tail -1 | sed "s/^/$w /"
done
