timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_benched.py -m gpu -x -q -k "forward_many or packed or e2e or queue or merged or serve" 2>&1 | tail -2
for w in mt-wnd cfg3-rmc2 wnd rmc3 ncf; do for d in 0 2; do
  RS_D2H_STREAMS=$d timeout 300 python bench.py --workload $w --no-cpu --steps 10 --warmup 3 > gpurun_out/d2h_${w}_$d.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/d2h_${w}_$d.json') if l.startswith('{')][-1]); print('$w d2h=$d value', round(d['value']), 'e2e', round(d['e2e']['value']), 'h2d GB/s', round(d['e2e']['h2d_gbs'],1))"
done; done
