run() { tag=$1; shift; env "$@" timeout 300 python bench.py --workload wnd --steps 10 --warmup 3 --no-cpu > gpurun_out/wnd_$tag.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/wnd_$tag.json') if l.startswith('{')][-1]); print('wnd $tag value', round(d['value']), 'svc us', round(d['sla']['mean_service_ms']*1e3,2), 'sat', round(d['sla']['saturated_qps']))"; }
run default RS_X=1
run pdl1 RS_PDL=1
run nopairs RS_TC2_ALL=0
run nopairs_pdl1 RS_TC2_ALL=0 RS_PDL=1
run default2 RS_X=1
