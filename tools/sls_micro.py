"""SLS microbenchmark: achieved HBM GB/s of the embedding stage (rs_pooled graph,
CUDA-event timed on its stream) for the cfg3 RMC2 shape at several query sizes,
for each SLS kernel variant (RS_SLS_VARIANT / RS_SLS_HINT / RS_SLS_UB knobs;
variant 3 also takes RS_SLS_NBUF / RS_SLS_WARPS: "var:hint:ub:nbuf:warps").

  python tools/sls_micro.py [--rows 10000000] [--variants "0:1:16,1:1:16,2:1:8"]
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
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--variants", default="0:0:0,1:0:0")
    ap.add_argument("--sizes", default="16,64,128,323,500,1000")
    ap.add_argument("--D", type=int, default=64)
    ap.add_argument("--L", type=int, default=80)
    ap.add_argument("--T", type=int, default=32)
    args = ap.parse_args()
    import torch
    import paper_2001_02772_b200 as rs
    spec = rs.ModelSpec("sls-micro", dense_fc=rs.LayerStack([256, 128, args.D]),
                        predict_fc=rs.LayerStack([1]),
                        embeddings=rs.EmbeddingConfig(args.T, args.L, args.D, "Sum"),
                        dense_input_dim=256)
    sizes = [int(x) for x in args.sizes.split(",")]
    per_item = args.T * args.L * (args.D * 4 + 8) + args.T * args.D * 4
    queries = []
    for i, S in enumerate(sizes):
        _, idx = rs.fill_query(spec, args.rows, 7, i, S)
        queries.append((S, torch.from_numpy(idx).cuda()))
    out = torch.empty((max(sizes), args.T * args.D), device="cuda")
    results = {}
    for v in args.variants.split(","):
        parts = v.split(":") + ["2", "16"]
        var, hint, ub, nbuf, warps = parts[:5]
        os.environ["RS_SLS_VARIANT"], os.environ["RS_SLS_HINT"], os.environ["RS_SLS_UB"] = var, hint, ub
        os.environ["RS_SLS_NBUF"], os.environ["RS_SLS_WARPS"] = nbuf, warps
        acc = rs.Accelerator(spec, args.rows, seed=1, max_query_size=max(sizes))
        row = {}
        same = True
        for S, idx in queries:
            ts = []
            for rep in range(7):
                t = acc.pooled_ptr(S, idx.data_ptr(), out.data_ptr(), rs.MEM_DEVICE, timed=True)
                if rep >= 2:
                    ts.append(t.compute_ms)
            ms = statistics.median(ts)
            row[S] = round(S * per_item / (ms * 1e-3) / 1e9, 1)
            got = out[:S].cpu()
            key = ("ref", S)
            if key not in results:
                results[key] = got
            elif not torch.equal(results[key], got):
                same = False
        results[v] = row
        print(json.dumps({"variant": v, "GBps_by_S": row,
                          "bitwise_equal_to_first_variant": same}), flush=True)
        acc.close()
        del acc
    print(json.dumps({"summary": {k: v for k, v in results.items() if isinstance(k, str)}}))


if __name__ == "__main__":
    main()
