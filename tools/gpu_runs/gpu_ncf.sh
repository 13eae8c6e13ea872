for rep in 1 2; do for d in 0 2; do
  RS_D2H_STREAMS=$d timeout 300 python bench.py --workload ncf --no-cpu --steps 10 --warmup 3 > gpurun_out/ncf_$d.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/ncf_$d.json') if l.startswith('{')][-1]); print('ncf d2h=$d value', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks'])"
done; done
