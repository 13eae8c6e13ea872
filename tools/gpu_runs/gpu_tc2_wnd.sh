timeout 900 python -m pytest tests/test_gpu_parity_benched.py tests/test_gpu_parity.py -m gpu -x -q -k "WND or wnd or cta_pair" 2>&1 | tail -2
for w in wnd mt-wnd; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_X=default" "RS_TC2_ALL=0" 2>&1 | tail -1 | sed "s/^/$w /"
done
timeout 400 python tools/env_sweep.py --workload wnd --fc bf16 --depth 16 --reps 3 "RS_X=default" "RS_TC2_ALL=0" 2>&1 | tail -1 | sed "s/^/wnd bf16 /"
for S in 256 1000; do timeout 400 python tools/env_sweep.py --workload wnd --depth 16 --reps 2 --size-fixed $S "RS_X=default" "RS_TC2_ALL=0" 2>&1 | tail -1 | sed "s/^/wnd S=$S /"; done
timeout 600 python bench.py --workload wnd --steps 10 --warmup 3 --no-cpu > gpurun_out/wnd_bench.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/wnd_bench.json') if l.startswith('{')][-1]); print('wnd bench value', round(d['value']), 'e2e', round(d['e2e']['value']))"
