"""Per-query device time of the pipelined queue (rs_forward_many, device
inputs) for a list of environment settings read at graph capture — the knob
sweeps behind DESIGN.md's tuning tables.

  python tools/env_sweep.py --workload cfg3-rmc2 "RS_INTER_TC=0" "RS_INTER_CTAS=8" ...
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3-rmc2")
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--pool", type=int, default=256)
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--size-fixed", type=int, default=0)
    ap.add_argument("--fc", default="auto", choices=["auto", "tf32", "fp32", "bf16"])
    ap.add_argument("settings", nargs="+")
    args = ap.parse_args()
    import torch
    import bench
    import paper_2001_02772_b200 as rs
    spec, rows, _ = bench.workload_spec(rs, args.workload)
    _, sizes = rs.gen_trace(42, 1000.0, rs.SizeDistribution.log_normal(math.log(300), 0.5),
                            args.pool)
    sizes = np.minimum(sizes, 1000)
    if args.size_fixed:
        sizes = np.full(args.pool, args.size_fixed, dtype=np.int64)
    dq, iq = [], []
    for q in range(args.pool):
        d, i = rs.fill_query(spec, rows, 42, q, int(sizes[q]))
        dq.append(torch.from_numpy(d).cuda())
        iq.append(torch.from_numpy(i).cuda())
    qs = [k % args.pool for k in range(args.n)]
    out = []
    for rep in range(args.reps):
        for setting in args.settings:
            saved = {}
            for kv in setting.split(","):
                if not kv:
                    continue
                k, v = kv.split("=")
                saved[k] = os.environ.get(k)
                os.environ[k] = v
            fc = {"auto": rs.FC_AUTO, "tf32": rs.FC_TF32, "fp32": rs.FC_FP32,
                  "bf16": rs.FC_BF16}[args.fc]
            acc = rs.Accelerator(spec, rows, seed=1, max_query_size=max(1000, args.size_fixed),
                                 fc_mode=fc, queue_depth=args.depth)
            o = torch.empty((max(1000, args.size_fixed), acc.output_dim), device="cuda")
            b = acc.batch([int(sizes[q]) for q in qs], [dq[q].data_ptr() for q in qs],
                          [iq[q].data_ptr() for q in qs], [o.data_ptr()] * len(qs),
                          rs.MEM_DEVICE)
            acc.forward_many(None, prepared=b)
            import time as _t
            with bench.ClockSampler(0) as clk:
                _t.sleep(0.6)  # nvidia-smi start-up
                t0 = _t.time()
                svc = np.concatenate([acc.forward_many(None, prepared=b) for _ in range(4)])
                clk.mark(t0, _t.time())
            c = clk.summary()
            pw = [float(ln.split(",")[2]) for ts, ln in clk.lines
                  if t0 - 0.03 <= ts <= clk.window[1] + 0.03 and len(ln.split(",")) >= 3
                  and ln.split(",")[2].strip() not in ("", "[N/A]")]
            rec = {"setting": setting, "rep": rep, "us_per_query": float(svc.mean() * 1e3),
                   "sm_mhz": c["sm_mhz"], "reasons": c["reasons"],
                   "power_w_median": float(np.median(pw)) if pw else None}
            out.append(rec)
            print(json.dumps(rec), flush=True)
            acc.close()
            del acc
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    summary = {}
    for r in out:
        summary.setdefault(r["setting"], []).append(r["us_per_query"])
    print(json.dumps({"workload": args.workload, "median_us_per_query":
                      {k: float(np.median(v)) for k, v in summary.items()}}))


if __name__ == "__main__":
    main()
