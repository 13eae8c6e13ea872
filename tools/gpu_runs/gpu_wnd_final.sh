timeout 600 python -m pytest tests/test_gpu_parity_benched.py tests/test_gpu_parity.py -m gpu -q -k "WND or wnd or cta_pair" 2>&1 | tail -1
timeout 300 python bench.py --workload wnd --steps 10 --warmup 3 --no-cpu > gpurun_out/wnd_final.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/wnd_final.json') if l.startswith('{')][-1]); print('wnd value', round(d['value']), 'svc us', round(d['sla']['mean_service_ms']*1e3,2))"
