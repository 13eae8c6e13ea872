"""Pipelined-queue diagnostic: per-query device time of rs_forward_many for the
whole forward vs the embedding stage alone (RS_MANY_POOL_ONLY=1), per queue
depth, next to the isolated (one query at a time) graph times.

  python tools/pipe_micro.py [--workload cfg3-rmc2] [--depths 1,2,4,8] [--n 2048]
"""
import argparse
import json
import math
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3-rmc2")
    ap.add_argument("--depths", default="1,2,4,8")
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--pool", type=int, default=128, help="distinct queries")
    ap.add_argument("--max-query", type=int, default=1000)
    ap.add_argument("--fc", default="auto")
    args = ap.parse_args()
    import torch
    import bench
    import paper_2001_02772_b200 as rs
    spec, rows, _ = bench.workload_spec(rs, args.workload)
    _, sizes = rs.gen_trace(11, 1000.0, rs.SizeDistribution.log_normal(math.log(300), 0.5),
                            args.pool)
    sizes = np.minimum(sizes, args.max_query)
    dq, iq = [], []
    for q in range(args.pool):
        d, i = rs.fill_query(spec, rows, 11, q, int(sizes[q]))
        dq.append(torch.from_numpy(d).cuda())
        iq.append(torch.from_numpy(i).cuda())
    mode = {"fp32": rs.FC_FP32, "tf32": rs.FC_TF32, "auto": rs.FC_AUTO}[args.fc]
    per_item = bench.sls_bytes_per_item(spec)
    res = {"workload": args.workload, "mean_items": float(np.mean(sizes)), "rows": []}
    for depth in [int(x) for x in args.depths.split(",")]:
        acc = rs.Accelerator(spec, rows, seed=1, max_query_size=args.max_query, fc_mode=mode,
                             queue_depth=depth)
        out = torch.empty((args.max_query, max(acc.pooled_dim, acc.output_dim)), device="cuda")
        row = {"depth": depth}
        # isolated graphs, one query at a time (median over the pool)
        if depth == 1:
            iso_f, iso_p = [], []
            for q in range(args.pool):
                S = int(sizes[q])
                iso_f.append(acc.forward_ptr(S, dq[q].data_ptr(), iq[q].data_ptr(),
                                             out.data_ptr(), rs.MEM_DEVICE, timed=True).compute_ms)
                iso_p.append(acc.pooled_ptr(S, iq[q].data_ptr(), out.data_ptr(), rs.MEM_DEVICE,
                                            timed=True).compute_ms)
            res["isolated_forward_us"] = statistics.mean(iso_f) * 1e3
            res["isolated_pooled_us"] = statistics.mean(iso_p) * 1e3
        qs = [k % args.pool for k in range(args.n)]
        for m in ("full", "pool"):
            os.environ["RS_MANY_POOL_ONLY"] = "1" if m == "pool" else "0"
            b = acc.batch([int(sizes[q]) for q in qs], [dq[q].data_ptr() for q in qs],
                          [iq[q].data_ptr() for q in qs], [out.data_ptr()] * len(qs),
                          rs.MEM_DEVICE)
            acc.forward_many(None, prepared=b)  # warm
            svc = acc.forward_many(None, prepared=b)
            us = float(svc.sum() / len(qs) * 1e3)
            items = float(np.mean([sizes[q] for q in qs]))
            row[m + "_us_per_query"] = us
            row[m + "_sls_TBps"] = items * per_item / (us * 1e-6) / 1e12
        os.environ["RS_MANY_POOL_ONLY"] = "0"
        res["rows"].append(row)
        print(json.dumps(row), flush=True)
        acc.close()
        del acc
    print(json.dumps(res))


if __name__ == "__main__":
    main()
