for st in "RS_PRIO=0" "RS_PDL=0"; do
  echo "== $st"; timeout 240 python tools/env_sweep.py --workload cfg3-rmc3 --depth 16 --reps 1 --n 512 "$st" 2>&1 | tail -2; echo "rc=$?"
done
echo "== cfg3-rmc2 RS_PDL=0"; timeout 240 python tools/env_sweep.py --workload cfg3-rmc2 --depth 16 --reps 1 --n 512 "RS_PDL=0" 2>&1 | tail -1
