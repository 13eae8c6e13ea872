mkdir -p gpurun_out/tc2c
timeout 600 python -m pytest tests/test_gpu_parity_benched.py -m gpu -x -q -k "cta_pair" 2>&1 | tail -2
for w in mt-wnd wnd; do for B in 1024; do for cp in off on; do
  timeout 200 python bench.py --workload $w --size-fixed $B --max-query 1024 --no-cpu --cta-pairs $cp --steps 10 --warmup 3 > gpurun_out/tc2c/${w}_${B}_${cp}.json 2>/dev/null
  python -c "
import json,sys; d=json.loads([l for l in open('gpurun_out/tc2c/${w}_${B}_${cp}.json') if l.startswith('{')][-1]); r=d['roofline']
print('$w $B $cp', round(d['value']), r['kernel'], round(r['achieved'],1), r['frac'], d['gpu_launches'])"
done; done; done
