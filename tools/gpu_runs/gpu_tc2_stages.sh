RS_TC2=2 TP_CASES="mt-wnd:1024,wnd:1024" TP_TAG=_pair6 timeout 900 python tools/tensor_profile.py > gpurun_out/tp_pair6.json 2> gpurun_out/tp_pair6.err
cat gpurun_out/tp_pair6.err | tail -2
RS_TC2=2 timeout 300 python -m pytest tests/test_gpu_parity_benched.py -m gpu -x -q -k "cta_pair or zoo_at" 2>&1 | tail -2
for w in mt-wnd wnd; do for S in 0 1000; do
  extra=""; [ $S -gt 0 ] && extra="--size-fixed $S"
  timeout 300 python tools/env_sweep.py --workload $w --reps 3 $extra "RS_TC2=0" "RS_TC2=1,RS_TC2_STAGES=4" "RS_TC2=1" 2>&1 | tail -1 | sed "s/^/$w S=$S /"
done; done
