for st in default pdl1; do
  if [ $st = pdl1 ]; then export RS_PDL=1; fi
  timeout 300 python bench.py --workload wnd --steps 10 --warmup 3 --no-cpu > gpurun_out/wnd_$st.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/wnd_$st.json') if l.startswith('{')][-1]); print('wnd $st value', round(d['value']), 'svc us', round(d['sla']['mean_service_ms']*1e3,2), d['clocks'])"
done
unset RS_PDL
timeout 300 python tools/env_sweep.py --workload wnd --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_PDL=1" 2>&1 | tail -1
