for w in cfg3-rmc2 cfg3-rmc3 cfg1-rmc1; do for d in 8 12 16; do
  timeout 300 python tools/env_sweep.py --workload $w --depth $d --reps 3 --n 1024 "RS_X=d$d" 2>&1 | tail -1 | sed "s/^/$w depth=$d /"
done; done
