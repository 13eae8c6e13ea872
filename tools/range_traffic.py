"""DRAM traffic of the WHOLE pipelined queue (not per kernel): one
rs_forward_many call over N queries inside a cudaProfilerStart/Stop range,
for `ncu --replay-mode range --profile-from-start off` (the range is replayed
as a unit, kernels overlapping as in the application). Prints the algorithmic
gather bytes of the range so ncu's dram__bytes_{read,write}.sum can be read
against them.

  ncu --replay-mode range --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      python tools/range_traffic.py --n 256 [--skip 7]
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
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--skip", type=int, default=0, help="RS_DIAG_SKIP for the captured graph")
    ap.add_argument("--depth", type=int, default=16)
    args = ap.parse_args()
    if args.skip:
        os.environ["RS_DIAG_SKIP"] = str(args.skip)
    import torch
    import bench
    import paper_2001_02772_b200 as rs
    spec, rows, _ = bench.workload_spec(rs, args.workload)
    _, sizes = rs.gen_trace(42, 1000.0, rs.SizeDistribution.log_normal(math.log(300), 0.5), args.n)
    sizes = np.minimum(sizes, 1000)
    dq, iq = [], []
    for q in range(args.n):
        d, i = rs.fill_query(spec, rows, 42, q, int(sizes[q]))
        dq.append(torch.from_numpy(d).cuda())
        iq.append(torch.from_numpy(i).cuda())
    acc = rs.Accelerator(spec, rows, seed=1, max_query_size=1000, fc_mode=rs.FC_AUTO,
                         queue_depth=args.depth)
    o = torch.empty((1000, acc.output_dim), device="cuda")
    b = acc.batch([int(s) for s in sizes], [t.data_ptr() for t in dq], [t.data_ptr() for t in iq],
                  [o.data_ptr()] * args.n, rs.MEM_DEVICE)
    acc.forward_many(None, prepared=b)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    acc.forward_many(None, prepared=b, timed=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    alg = float(np.sum(sizes)) * bench.sls_bytes_per_item(spec)
    print(json.dumps({"workload": args.workload, "queries": args.n, "skip": args.skip,
                      "items": int(np.sum(sizes)), "algorithmic_gather_bytes": alg}))
    acc.close()


if __name__ == "__main__":
    main()
