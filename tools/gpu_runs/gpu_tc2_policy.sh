for w in mt-wnd wnd; do
  timeout 400 python tools/env_sweep.py --workload $w --reps 3 "RS_TC2=0" "RS_TC2=1" "RS_TC2=1,RS_TC2_POLICY=1" "RS_TC2=1,RS_TC2_POLICY=2" 2>&1 | tail -1 | sed "s/^/$w /"
done
timeout 400 python tools/env_sweep.py --workload mt-wnd --reps 2 --size-fixed 1000 "RS_TC2=0" "RS_TC2=1" "RS_TC2=1,RS_TC2_POLICY=2" 2>&1 | tail -1 | sed "s/^/mt-wnd S=1000 /"
