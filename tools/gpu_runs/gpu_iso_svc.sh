python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import bench
import paper_2001_02772_b200 as rs
for w in ("cfg3-rmc2", "cfg3-rmc3"):
    for env in ({}, {"RS_CARVEOUT": "0"}, {"RS_SLS_WAVES": "1"}):
        for k in ("RS_CARVEOUT", "RS_SLS_WAVES"):
            os.environ.pop(k, None)
        os.environ.update(env)
        spec, rows, _ = bench.workload_spec(rs, w)
        acc = rs.Accelerator(spec, rows, seed=1, max_query_size=1000, fc_mode=rs.FC_AUTO)
        out = {S: round(acc.service_time(S) * 1e3, 4) for S in (1, 64, 322, 1000)}
        print(w, env or "default", "service_time ms", out, flush=True)
        acc.close()
PY
