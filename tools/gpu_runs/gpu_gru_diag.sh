python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2001_02772_b200 as rs
for v in ("0", "-2"):
    os.environ["RS_GRU_DIAG"] = v
    spec = rs.builtin_model("DIEN"); spec.embeddings.lookups_per_table = 100
    acc = rs.Accelerator(spec, 1_000_000, seed=1, max_query_size=1000, fc_mode=rs.FC_AUTO)
    d, i = rs.fill_query(spec, 1_000_000, 5, 0, 300)
    ts = []
    for k in range(8):
        t = acc.pooled_timed(i) if hasattr(acc, "pooled_timed") else None
    print("RS_GRU_DIAG", v, "service_time(300) ms", acc.service_time(300) * 1e3, flush=True)
    acc.close()
PY
for v in 0 -2; do RS_GRU_DIAG=$v timeout 300 python tools/env_sweep.py --workload cfg5-dien --depth 16 --reps 2 "RS_X=$v" 2>&1 | tail -1; done
