"""Isolated-launch SLS roofline (the bench's roofline.achieved method): the
embedding kernel alone, event nodes around it in the embedding-stage graph,
cfg3 RMC2 tables (32 x 10M x 64), per query size, for environment settings
read at graph capture.

  python tools/sls_iso.py "RS_SLS_DYN=0" "RS_SLS_DYN=1"
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3-rmc2")
    ap.add_argument("--sizes", default="64,128,330,500,1000")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("settings", nargs="+")
    args = ap.parse_args()
    import torch
    import bench
    import paper_2001_02772_b200 as rs
    spec, rows, _ = bench.workload_spec(rs, args.workload)
    per_item = bench.sls_bytes_per_item(spec)
    sizes = [int(x) for x in args.sizes.split(",")]
    qs = {S: [torch.from_numpy(rs.fill_query(spec, rows, 3, 100 * S + r, S)[1]).cuda()
              for r in range(args.reps)] for S in sizes}
    res = {}
    for setting in args.settings:
        for kv in setting.split(","):
            k, v = kv.split("=")
            os.environ[k] = v
        acc = rs.Accelerator(spec, rows, seed=1, max_query_size=1000, fc_mode=rs.FC_AUTO)
        out = torch.empty((1000, acc.pooled_dim), device="cuda")
        row = {}
        for S in sizes:
            ms = []
            for r, ix in enumerate(qs[S]):
                t = acc.pooled_ptr(S, ix.data_ptr(), out.data_ptr(), rs.MEM_DEVICE, timed=True)
                if r:
                    ms.append(t.embed_ms)
            row[S] = S * per_item / (statistics.median(ms) * 1e-3) / 1e9
        res[setting] = row
        print(json.dumps({"setting": setting, "GBps": row}), flush=True)
        acc.close()
        del acc
        for kv in setting.split(","):
            os.environ.pop(kv.split("=")[0], None)
    print(json.dumps({"workload": args.workload, "GBps": res}))


if __name__ == "__main__":
    main()
