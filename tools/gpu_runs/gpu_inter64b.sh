timeout 900 python -m pytest tests/test_gpu_parity_benched.py tests/test_gpu_parity.py -m gpu -x -q -k "cfg3 or RMC or DLRM or forward_many" 2>&1 | tail -2
for w in cfg3-rmc2 cfg3-rmc3 rmc2 cfg1-rmc1; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_X=default" "RS_INTER_THREADS=256" 2>&1 | tail -1 | sed "s/^/$w /"
done
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/inter64_bench.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/inter64_bench.json') if l.startswith('{')][-1]); print('bench value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), d['clocks'])"
