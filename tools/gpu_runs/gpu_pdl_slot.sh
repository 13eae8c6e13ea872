timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in cfg3-rmc2 cfg3-rmc3 rmc3 cfg5-din; do
  timeout 300 python tools/env_sweep.py --workload $w --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_PDL=1" 2>&1 | tail -1 | sed "s/^/$w /"
done
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/pdl_bench.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/pdl_bench.json') if l.startswith('{')][-1]); print('bench value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), d['clocks'])"
