timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import bench
import paper_2001_02772_b200 as rs
for w in ("cfg3-rmc2", "cfg3-rmc3", "cfg5-din", "cfg5-dien", "rmc2"):
    for env in ({}, {"RS_CARVEOUT_SINGLE": "1"}):
        os.environ.pop("RS_CARVEOUT_SINGLE", None)
        os.environ.update(env)
        spec, rows, _ = bench.workload_spec(rs, w)
        acc = rs.Accelerator(spec, rows, seed=1, max_query_size=1000, fc_mode=rs.FC_AUTO)
        out = {S: round(acc.service_time(S) * 1e3, 4) for S in (1, 64, 322, 1000)}
        print(w, env or "default", "service_time ms", out, flush=True)
        acc.close()
PY
timeout 600 python tools/sls_iso.py --sizes 322,1000 "RS_X=default" "RS_CARVEOUT_SINGLE=1" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/cs_bench.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/cs_bench.json') if l.startswith('{')][-1]); r=d['roofline']; print('bench value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(r['frac'],3), 'other TF/s', round(r['other']['achieved'],1), d['clocks'])"
