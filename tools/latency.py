"""Single-query latency by FC path: one query alone on the GPU (device-resident
inputs, rs_forward with timing = CUDA events around the graph launch), median
over reps, for each fc_mode and query size. Complements bench.py's pipelined
throughput when choosing the FC_AUTO rule.

  python tools/latency.py [--workload cfg3-rmc2] [--sizes 1,8,32,64,127,128,300]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3-rmc2")
    ap.add_argument("--sizes", default="1,8,32,64,127,128,300")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import torch
    import bench
    import paper_2001_02772_b200 as rs
    spec, rows, _ = bench.workload_spec(rs, args.workload)
    sizes = [int(x) for x in args.sizes.split(",")]
    res = {"workload": args.workload, "unit": "ms (median, rs_forward compute_ms)", "rows": []}
    res["rows"] = [{"S": S} for S in sizes]
    for m, v in (("fp32", rs.FC_FP32), ("tf32", rs.FC_TF32), ("auto", rs.FC_AUTO)):
        acc = rs.Accelerator(spec, rows, seed=1, max_query_size=max(sizes), fc_mode=v)
        for k, S in enumerate(sizes):
            d, i = rs.fill_query(spec, rows, 5, S, S)
            td, ti = torch.from_numpy(d).cuda(), torch.from_numpy(i).cuda()
            out = torch.empty((S, acc.output_dim), device="cuda")
            for _ in range(5):
                acc.forward_ptr(S, td.data_ptr(), ti.data_ptr(), out.data_ptr(), rs.MEM_DEVICE)
            acc.sync()
            t = [acc.forward_ptr(S, td.data_ptr(), ti.data_ptr(), out.data_ptr(), rs.MEM_DEVICE,
                                 timed=True).compute_ms for _ in range(args.reps)]
            res["rows"][k][m] = float(np.median(t))
        acc.close()
        torch.cuda.empty_cache()
    for r in res["rows"]:
        print(json.dumps(r), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
