"""Real-time validation of the QPS@SLA methodology: serve a Poisson stream on
the clock through rs_serve (real execution, queueing included) and compare
the measured p50/p95 with the replay that bench.py uses (Lindley recursion
over the CUDA-event service gaps of rs_forward_many, sim.cpp's FIFO server).

  python tools/realtime.py [--workload cfg3-rmc2] [--n 20000] [--loads 0.5,0.8,0.9,1.0]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def replay(arrival, service, extra):
    """FIFO single server: finish_i = max(a_i, finish_{i-1}) + s_i."""
    fin = np.empty_like(arrival)
    f = 0.0
    for i in range(len(arrival)):
        f = max(arrival[i], f) + service[i]
        fin[i] = f
    return fin - arrival + extra


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3-rmc2")
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--pool", type=int, default=256)
    ap.add_argument("--loads", default="0.5,0.8,0.9,1.0")
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--host", action="store_true", help="pinned host inputs (end to end)")
    ap.add_argument("--replicas", type=int, default=1, help="K GPUs (one handle each)")
    args = ap.parse_args()
    import torch
    import bench
    import paper_2001_02772_b200 as rs
    spec, rows, _ = bench.workload_spec(rs, args.workload)
    _, sizes = rs.gen_trace(5, 1000.0, rs.SizeDistribution.log_normal(math.log(300), 0.5),
                            args.pool)
    sizes = np.minimum(sizes, 1000)
    acc = rs.Accelerator(spec, rows, seed=1, max_query_size=1000, queue_depth=args.depth)
    reps = [acc] + [rs.Accelerator(spec, rows, seed=1, device=k, max_query_size=1000,
                                   queue_depth=args.depth) for k in range(1, args.replicas)]
    if args.replicas > 1 and not args.host:
        raise SystemExit("--replicas > 1 needs --host (device inputs live on one GPU)")
    dp, ip = [], []
    keep = []
    for q in range(args.pool):
        d, i = rs.fill_query(spec, rows, 5, q, int(sizes[q]))
        if args.host:
            bd, bi = rs.PinnedBuffer(max(d.nbytes, 16)), rs.PinnedBuffer(i.nbytes)
            bd.view(np.float32, d.shape)[...] = d
            bi.view(np.int64, i.shape)[...] = i
            keep += [bd, bi]
            dp.append(bd.ptr)
            ip.append(bi.ptr)
        else:
            td, ti = torch.from_numpy(d).cuda(), torch.from_numpy(i).cuda()
            keep += [td, ti]
            dp.append(td.data_ptr())
            ip.append(ti.data_ptr())
    if args.host:
        ob = rs.PinnedBuffer(1000 * acc.output_dim * 4)
        optr = ob.ptr
    else:
        ot = torch.empty((1000, acc.output_dim), device="cuda")
        optr = ot.data_ptr()
    loc = rs.MEM_HOST if args.host else rs.MEM_DEVICE
    qs = [k % args.pool for k in range(args.n)]
    b = acc.batch([int(sizes[q]) for q in qs], [dp[q] for q in qs], [ip[q] for q in qs],
                  [optr] * len(qs), loc)
    # service gaps of the pipelined queue (what bench.py replays)
    acc.forward_many(None, prepared=b)
    svc, res = acc.forward_many(None, prepared=b, residence=True)
    svc_s, extra_s = svc * 1e-3, np.maximum(res - svc, 0.0) * 1e-3
    cap = args.replicas / float(np.mean(svc_s))
    out = {"workload": args.workload, "inputs": "host pinned" if args.host else "device",
           "replicas": args.replicas,
           "n": args.n, "capacity_qps": cap, "rows": []}
    rng = np.random.default_rng(11)
    for f in [float(x) for x in args.loads.split(",")]:
        lam = f * cap
        arrival = np.cumsum(rng.exponential(1.0 / lam, size=args.n))
        arrival -= arrival[0]
        lat_real = rs.serve(reps, b, arrival) * 1e-3
        # K-server replay: query i to the earliest-free server (FIFO per server)
        if args.replicas == 1:
            lat_rep = replay(arrival, svc_s, extra_s)
        else:
            free = np.zeros(args.replicas)
            lat_rep = np.empty(args.n)
            for i2 in range(args.n):
                k = int(np.argmin(free))
                fin = max(arrival[i2], free[k]) + svc_s[i2]
                free[k] = fin
                lat_rep[i2] = fin - arrival[i2] + extra_s[i2]
        w = args.n // 10  # warm-up excluded, as sim.cpp
        row = {"load": f, "lambda_qps": lam,
               "real_p50_ms": float(np.percentile(lat_real[w:], 50) * 1e3),
               "real_p95_ms": float(np.percentile(lat_real[w:], 95) * 1e3),
               "replay_p50_ms": float(np.percentile(lat_rep[w:], 50) * 1e3),
               "replay_p95_ms": float(np.percentile(lat_rep[w:], 95) * 1e3),
               "real_throughput_qps": args.n / float(arrival[-1] + lat_real[-1])}
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps(out))
    for r in reps:
        r.close()


if __name__ == "__main__":
    main()
