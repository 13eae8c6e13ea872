mkdir -p gpurun_out/gru2g
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_group" 2>&1 | tail -2
for w in cfg5-dien dien; do
  timeout 400 python tools/env_sweep.py --workload $w --depth 16 --reps 3 "RS_GRU_2G=0" "RS_GRU_2G=1" 2>&1 | tail -1 | sed "s/^/$w /"
done
timeout 300 python tools/run_once.py --model DIEN --L 100 --S 300 --fc tf32 --reps 1 >/dev/null 2>&1
python - <<'PY'
import time, numpy as np, os, sys
sys.path.insert(0, ".")
import paper_2001_02772_b200 as rs
for v in ("0", "1"):
    os.environ["RS_GRU_2G"] = v
    spec = rs.builtin_model("DIEN"); spec.embeddings.lookups_per_table = 100
    acc = rs.Accelerator(spec, 1_000_000, seed=1, max_query_size=1000, fc_mode=rs.FC_AUTO)
    d, i = rs.fill_query(spec, 1_000_000, 5, 0, 300)
    for _ in range(3): acc.forward(d, i)
    t = []
    for k in range(10):
        acc.forward(d, i, timing=True) if False else None
    st = [acc.service_time(300) for _ in range(1)]
    print("RS_GRU_2G", v, "service_time(300) ms", st[0] * 1e3)
    acc.close()
PY
