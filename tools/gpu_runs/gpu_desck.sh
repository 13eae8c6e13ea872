for w in mt-wnd rmc3 ncf cfg3-rmc2; do for d in 0 1; do
  RS_DESC_KERNEL=$d timeout 300 python bench.py --workload $w --no-cpu --steps 10 --warmup 3 > gpurun_out/desck_${w}_$d.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/desck_${w}_$d.json') if l.startswith('{')][-1]); print('$w desc_kernel=$d value', round(d['value']), 'e2e', round(d['e2e']['value']), 'h2d GB/s', round(d['e2e']['h2d_gbs'],1))"
done; done
RS_DESC_KERNEL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "forward_many or packed or queue or merged or serve or edges" 2>&1 | tail -2
