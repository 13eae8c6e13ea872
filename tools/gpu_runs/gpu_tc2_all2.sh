for w in mt-wnd wnd; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_X=default" "RS_TC2=2" "RS_TC2=2,RS_TC2_STAGES=4" "RS_TC2=1" 2>&1 | tail -1 | sed "s/^/$w /"
done
