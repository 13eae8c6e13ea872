#!/bin/bash
# RS_OPT_CTA_PAIRS: parity, then the configs[3] MT-WND batch sweep and WND with the option on / off
mkdir -p gpurun_out/tc2d
timeout 600 python -m pytest tests/test_gpu_parity_benched.py -m gpu -x -q -k "cta_pair or zoo_at" 2>&1 | tail -3 | tee gpurun_out/tc2d/parity.log
for w in mt-wnd wnd; do for fc in auto bf16; do for B in 256 512 1024; do for cp in off on; do
  timeout 200 python bench.py --workload $w --fc $fc --size-fixed $B --max-query 1024 --no-cpu --cta-pairs $cp --steps 10 --warmup 3 > gpurun_out/tc2d/${w}_${fc}_${B}_${cp}.json 2> gpurun_out/tc2d/${w}_${fc}_${B}_${cp}.err
  python - "$w" "$fc" "$B" "$cp" gpurun_out/tc2d/${w}_${fc}_${B}_${cp}.json <<'PY'
import json, sys
w, fc, B, cp, f = sys.argv[1:]
try:
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    r = d["roofline"]
    print(w, fc, B, cp, "value", round(d["value"]), "ms/q", round(d["sla"]["mean_service_ms"] * 1e3, 2), "roof", r["kernel"], round(r["achieved"], 1), r["unit"], round(r["frac"], 3))
except Exception as e:
    print(w, fc, B, cp, "ERR", e)
PY
done; done; done; done | tee gpurun_out/tc2d/summary.txt
