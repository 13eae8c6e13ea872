run() { tag=$1; w=$2; shift 2; env "$@" timeout 300 python bench.py --workload $w --size-fixed 1024 --max-query 1024 --steps 10 --warmup 3 --no-cpu $CP > gpurun_out/pp_${w}_$tag.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/pp_${w}_$tag.json') if l.startswith('{')][-1]); print('$w $tag value', round(d['value']), 'svc us', round(d['sla']['mean_service_ms']*1e3,2))"; }
for w in mt-wnd wnd; do
  CP="--cta-pairs off" run off $w RS_X=1
  CP="--cta-pairs on" run on $w RS_X=1
  CP="--cta-pairs on" run on_pdl1 $w RS_PDL=1
  CP="--cta-pairs off" run off_pdl1 $w RS_PDL=1
done
