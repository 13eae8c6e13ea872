mkdir -p gpurun_out/tc2
for fc in tf32 bf16; do for S in 256 512 640 768 896; do
  timeout 200 python tools/env_sweep.py --workload mt-wnd --fc $fc --reps 2 --size-fixed $S "RS_TC2=0" "RS_TC2=1" 2>&1 | tail -1 | sed "s/^/$fc S=$S /"
done; done | tee gpurun_out/tc2/sizes.log
for S in 512 1024; do timeout 200 python tools/env_sweep.py --workload wnd --reps 2 --size-fixed $S "RS_TC2=0" "RS_TC2=1" 2>&1 | tail -1 | sed "s/^/wnd S=$S /"; done | tee -a gpurun_out/tc2/sizes.log
