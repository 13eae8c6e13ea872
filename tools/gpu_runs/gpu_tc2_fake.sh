for w in mt-wnd wnd; do
  timeout 400 python tools/env_sweep.py --workload $w --reps 4 "RS_TC2=0" "RS_TC2=1" "RS_TC2=1,RS_TC2_FAKE=1" 2>&1 | tail -1 | sed "s/^/$w /"
done
