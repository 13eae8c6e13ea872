"""Where the pipelined step goes (cfg3 RMC2): per-query device time of
rs_forward_many at queue depth d with stages of the forward graph dropped by
the diagnostic RS_DIAG_SKIP bits (1 bottom MLP, 2 interaction, 4 predict
stack, 8 embedding stage; outputs invalid) — read when a graph is captured, so
each setting builds its own handle.

  python tools/pipe_diag.py [--workload cfg3-rmc2] [--depths 8,16] [--skips 0,1,2,4,7]
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
    ap.add_argument("--depths", default="8")
    ap.add_argument("--skips", default="0,1,2,4,6,7")
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--pool", type=int, default=256)
    args = ap.parse_args()
    import torch
    import bench
    import paper_2001_02772_b200 as rs
    spec, rows, _ = bench.workload_spec(rs, args.workload)
    _, sizes = rs.gen_trace(42, 1000.0, rs.SizeDistribution.log_normal(math.log(300), 0.5),
                            args.pool)
    sizes = np.minimum(sizes, 1000)
    dq, iq = [], []
    for q in range(args.pool):
        d, i = rs.fill_query(spec, rows, 42, q, int(sizes[q]))
        dq.append(torch.from_numpy(d).cuda())
        iq.append(torch.from_numpy(i).cuda())
    qs = [k % args.pool for k in range(args.n)]
    out = []
    for depth in [int(x) for x in args.depths.split(",")]:
        for skip in [int(x) for x in args.skips.split(",")]:
            os.environ["RS_DIAG_SKIP"] = str(skip)
            acc = rs.Accelerator(spec, rows, seed=1, max_query_size=1000, fc_mode=rs.FC_AUTO,
                                 queue_depth=depth)
            o = torch.empty((1000, max(acc.pooled_dim, acc.output_dim)), device="cuda")
            b = acc.batch([int(sizes[q]) for q in qs], [dq[q].data_ptr() for q in qs],
                          [iq[q].data_ptr() for q in qs], [o.data_ptr()] * len(qs), rs.MEM_DEVICE)
            acc.forward_many(None, prepared=b)
            svc = acc.forward_many(None, prepared=b)
            rec = {"depth": depth, "skip": skip, "us_per_query": float(svc.mean() * 1e3),
                   "qps": 1.0 / float(svc.mean() * 1e-3)}
            out.append(rec)
            print(json.dumps(rec), flush=True)
            acc.close()
            del acc
    os.environ["RS_DIAG_SKIP"] = "0"
    print(json.dumps({"workload": args.workload, "rows": out}))


if __name__ == "__main__":
    main()
