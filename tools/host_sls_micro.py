"""Throughput of rs_host_sls and rs_host_fc (host-core SparseLengthsSum) on a
cfg3-RMC2-like bag shape: T tables x rows x D=64, L=80 lookups, uniform
indices, tables larger than the host's last-level cache. Algorithmic bytes
per bag = L*D*4 (rows read) + L*8 (indices) + D*4 (pooled written), the same
per-bag accounting as the device SLS roofline.

  python tools/host_sls_micro.py [--tables 8] [--rows 1000000] [--S 300]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_02772_b200 as rs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tables", type=int, default=8)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=64)
    ap.add_argument("--lookups", type=int, default=80)
    ap.add_argument("--S", type=int, default=300)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    tab = rng.standard_normal((a.tables, a.rows, a.dim), dtype=np.float32)
    bag_bytes = a.lookups * a.dim * 4 + a.lookups * 8 + a.dim * 4
    out = {"shape": vars(a), "bytes_per_bag": bag_bytes, "cores": os.cpu_count(), "runs": []}
    for threads in sorted({1, 4, 16, os.cpu_count() or 1}):
        idxs = [rng.integers(0, a.rows, (a.S, a.tables, a.lookups), dtype=np.int64)
                for _ in range(4)]
        rs.host_sls(tab, idxs[0], threads)  # warm
        t0 = time.perf_counter()
        for i in range(a.reps):
            rs.host_sls(tab, idxs[i % 4], threads)
        dt = (time.perf_counter() - t0) / a.reps
        bags = a.S * a.tables
        out["runs"].append({"threads": threads, "ms_per_query": dt * 1e3,
                            "GBps": bags * bag_bytes / dt / 1e9,
                            "items_per_s": a.S / dt})
    # host FC at a predict-layer shape: x[S, 512] @ W[256, 512]^T, bias + ReLU
    x = rng.standard_normal((a.S, 512), dtype=np.float32)
    w = rng.standard_normal((256, 512), dtype=np.float32)
    bias = np.zeros(256, np.float32)
    out["fc"] = {"shape": [a.S, 512, 256], "runs": []}
    for threads in sorted({1, 4, 16, os.cpu_count() or 1}):
        rs.host_fc(x, w, bias, True, threads)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            rs.host_fc(x, w, bias, True, threads)
        dt = (time.perf_counter() - t0) / a.reps
        out["fc"]["runs"].append({"threads": threads, "ms": dt * 1e3,
                                  "GFLOPs": 2 * a.S * 512 * 256 / dt / 1e9})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
