RS_TC2_CAPPED=1 timeout 900 python -m pytest tests/test_gpu_parity_benched.py tests/test_gpu_parity.py -m gpu -x -q -k "cfg3 or RMC or DLRM or coresident" 2>&1 | tail -2
for w in cfg3-rmc3 cfg3-rmc2 rmc2 cfg1-rmc1 rmc1; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_TC2_CAPPED=0" "RS_TC2_CAPPED=1" 2>&1 | tail -1 | sed "s/^/$w /"
done
