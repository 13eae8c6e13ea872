timeout 900 python -m pytest tests/test_gpu_parity_benched.py -m gpu -x -q -k "cfg3" 2>&1 | tail -2
for w in cfg3-rmc3 cfg3-rmc2; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_X=default" "RS_TC2_CAPPED=0" 2>&1 | tail -1 | sed "s/^/$w /"
done
timeout 600 python bench.py --workload cfg3-rmc3 --steps 10 --warmup 3 --no-cpu > gpurun_out/rmc3_bench.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/rmc3_bench.json') if l.startswith('{')][-1]); print('cfg3-rmc3 value', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks'])"
