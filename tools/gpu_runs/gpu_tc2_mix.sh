for w in mt-wnd wnd; do for fc in auto bf16; do
  timeout 300 python tools/env_sweep.py --workload $w --fc $fc --reps 4 "RS_TC2=0" "RS_X=1" "RS_TC2_MIN=100000" "RS_TC2_MIN=640" 2>&1 | tail -1 | sed "s/^/$w $fc /"
done; done | tee gpurun_out/tc2/mix.log
