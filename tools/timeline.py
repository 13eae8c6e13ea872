"""Kernel timeline of the pipelined forward (rs_forward_many) from CUPTI via
torch.profiler: per-kernel durations INSIDE the overlapped pipeline (which
ncu's serialised replay cannot show), concurrency, and the SLS kernels'
back-to-back coverage.

  python tools/timeline.py [--workload cfg3-rmc2] [--n 64] [--depth 8] [--trace out.json]
"""
import argparse
import collections
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def summarize(events):
    ks = [e for e in events if e.get("cat") == "kernel"]
    if not ks:
        return {"kernels": 0}
    t0 = min(e["ts"] for e in ks)
    t1 = max(e["ts"] + e["dur"] for e in ks)
    by = collections.defaultdict(list)
    for e in ks:
        name = e["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        by[name].append(e["dur"])
    # union of SLS-kernel intervals: how much of the window an SLS grid is live
    sls = sorted((e["ts"], e["ts"] + e["dur"]) for e in ks if "sls_" in e["name"])
    cover, cur_s, cur_e = 0.0, None, None
    for s, e in sls:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                cover += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        cover += cur_e - cur_s
    out = {"window_us": t1 - t0, "kernels": len(ks), "sls_live_fraction": cover / (t1 - t0),
           "per_kernel": []}
    # host-link activity (--host): H2D copy durations, GB/s per copy, and the
    # fraction of the window with at least one H2D copy in flight
    cps = [e for e in events if e.get("cat") == "gpu_memcpy" and "HtoD" in e.get("name", "")]
    big = [e for e in cps if e.get("args", {}).get("bytes", 0) >= (1 << 20)]
    if big:
        iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in big)
        lo, hi = iv[0][0], max(b for _, b in iv)
        cov, cs, ce = 0.0, None, None
        for a, b in iv:
            if ce is None or a > ce:
                if ce is not None:
                    cov += ce - cs
                cs, ce = a, b
            else:
                ce = max(ce, b)
        cov += ce - cs
        out["h2d"] = {"copies": len(big), "small_h2d_copies": len(cps) - len(big),
                      "mean_us": float(np.mean([e["dur"] for e in big])),
                      "mean_gbs_per_copy": float(np.mean([e["args"]["bytes"] / e["dur"] / 1e3
                                                          for e in big])),
                      "busy_fraction": cov / (hi - lo),
                      "overall_gbs": sum(e["args"]["bytes"] for e in big) / (hi - lo) / 1e3}
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        out["per_kernel"].append({"kernel": k, "launches": len(v), "mean_us": float(np.mean(v)),
                                  "p50_us": float(np.median(v)), "max_us": float(np.max(v)),
                                  "sum_us": float(np.sum(v))})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3-rmc2")
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--pool", type=int, default=64)
    ap.add_argument("--max-query", type=int, default=1000)
    ap.add_argument("--trace", default="")
    ap.add_argument("--host", action="store_true", help="pinned host inputs (e2e path)")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
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
    acc = rs.Accelerator(spec, rows, seed=1, max_query_size=args.max_query, fc_mode=rs.FC_AUTO,
                         queue_depth=args.depth)
    out = torch.empty((args.max_query, acc.output_dim), device="cuda")
    qs = [k % args.pool for k in range(args.n)]
    if args.host:  # one packed pinned buffer per query, as bench.py's e2e
        keep, dp, ip = [], [], []
        for q in range(args.pool):
            d, i = dq[q].cpu().numpy(), iq[q].cpu().numpy()
            hb = rs.PinnedBuffer(d.nbytes + i.nbytes)
            hb.view(np.uint8, (d.nbytes + i.nbytes,))[...] = np.concatenate(
                [d.reshape(-1).view(np.uint8), i.reshape(-1).view(np.uint8)])
            keep.append(hb)
            dp.append(hb.ptr)
            ip.append(hb.ptr + d.nbytes)
        ob = rs.PinnedBuffer(args.max_query * acc.output_dim * 4)
        b = acc.batch([int(sizes[q]) for q in qs], [dp[q] for q in qs], [ip[q] for q in qs],
                      [ob.ptr] * len(qs), rs.MEM_HOST)
    else:
        b = acc.batch([int(sizes[q]) for q in qs], [dq[q].data_ptr() for q in qs],
                      [iq[q].data_ptr() for q in qs], [out.data_ptr()] * len(qs), rs.MEM_DEVICE)
    acc.forward_many(None, prepared=b)
    acc.forward_many(None, prepared=b)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        svc = acc.forward_many(None, prepared=b)
        torch.cuda.synchronize()
    path = args.trace or "/tmp/rs_timeline.json"
    prof.export_chrome_trace(path)
    with open(path) as f:
        ev = json.load(f)["traceEvents"]
    res = summarize(ev)
    res["svc_us_per_query"] = float(svc.sum() / len(qs) * 1e3)
    res["mean_items"] = float(np.mean([sizes[q] for q in qs]))
    print(json.dumps(res, indent=1))
    acc.close()


if __name__ == "__main__":
    main()
