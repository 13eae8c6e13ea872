for w in mt-wnd wnd rmc3 cfg3-rmc3; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_X=default" "RS_TC2=2" 2>&1 | tail -1 | sed "s/^/$w /"
done
for w in mt-wnd; do
  timeout 400 python tools/env_sweep.py --workload $w --fc bf16 --depth 16 --reps 3 "RS_X=default" "RS_TC2=2" 2>&1 | tail -1 | sed "s/^/$w bf16 /"
done
