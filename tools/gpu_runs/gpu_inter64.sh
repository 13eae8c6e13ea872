mkdir -p gpurun_out/inter64
RS_INTER_THREADS=64 timeout 900 python -m pytest tests/test_gpu_parity_benched.py -m gpu -x -q -k "cfg3" 2>&1 | tail -2
for w in cfg3-rmc2 cfg3-rmc3 rmc2; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_INTER_THREADS=256" "RS_INTER_THREADS=64" "RS_INTER_THREADS=64,RS_INTER_PER_SM=2" 2>&1 | tail -1 | sed "s/^/$w /"
done | tee gpurun_out/inter64/sweep.log
