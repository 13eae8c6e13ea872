mkdir -p gpurun_out/tc2
for w in mt-wnd wnd; do for S in 300 400 700 1000; do
  timeout 200 python tools/env_sweep.py --workload $w --reps 2 --size-fixed $S "RS_TC2=0" "RS_TC2=1" 2>&1 | tail -1 | sed "s/^/$w S=$S /"
done; done | tee gpurun_out/tc2/sizes2.log
