mkdir -p gpurun_out/rep
for r in 1 2; do
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/rep/bench_$r.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/rep/bench_$r.json') if l.startswith('{')][-1]); print('rep $r value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), 'cpu', round(d['cpu_baseline']['value'],1), d['clocks'])"
done
