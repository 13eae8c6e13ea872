for w in cfg1-rmc1 cfg3-rmc2 rmc1 ncf; do for d in 16 24 32; do
  timeout 300 python tools/env_sweep.py --workload $w --depth $d --reps 3 --n 1024 "RS_X=d$d" 2>&1 | tail -1 | sed "s/^/$w depth=$d /"
done; done
