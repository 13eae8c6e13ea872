"""Per-query stage latencies inside the pipelined queue from a tools/timeline.py
chrome trace: for every SLS launch, the dependent interaction / predict-stack
kernels on the same stream, the gaps between them, and how many SLS grids run
concurrently.

  python tools/tl_analyze.py gpurun_out/tl_skip0.json
"""
import collections
import json
import sys

import numpy as np


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "")
    return n.split("(")[0].split("<")[0].split("::")[-1]


def main(path):
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel"]
    t0 = min(e["ts"] for e in ks)
    by_stream = collections.defaultdict(list)
    for e in ks:
        by_stream[e["args"].get("stream")].append((e["ts"] - t0, e["dur"], short(e["name"])))
    names = collections.Counter(short(e["name"]) for e in ks)
    res = {"streams": len(by_stream), "kernel_counts": dict(names)}
    # per stream: after each sls, the next kernels until the next sls
    gaps = collections.defaultdict(list)
    durs = collections.defaultdict(list)
    for st, lst in by_stream.items():
        lst.sort()
        for i, (ts, du, nm) in enumerate(lst):
            durs[nm].append(du)
            if i + 1 < len(lst):
                nts, ndu, nnm = lst[i + 1]
                gaps[f"{nm} -> {nnm}"].append(nts - (ts + du))
    res["dur_us"] = {k: {"mean": float(np.mean(v)), "p50": float(np.median(v)), "n": len(v)}
                     for k, v in durs.items()}
    res["gap_us"] = {k: {"mean": float(np.mean(v)), "p50": float(np.median(v)), "n": len(v)}
                     for k, v in gaps.items() if len(v) > 3}
    # concurrency of SLS grids
    sls = sorted((e["ts"] - t0, e["ts"] - t0 + e["dur"]) for e in ks if "sls" in e["name"])
    pts = sorted([(a, 1) for a, _ in sls] + [(b, -1) for _, b in sls])
    cur, last, hist = 0, 0.0, collections.Counter()
    for t, d in pts:
        hist[cur] += t - last
        cur += d
        last = t
    tot = sum(hist.values())
    res["sls_concurrency_time_fraction"] = {k: v / tot for k, v in sorted(hist.items())}
    res["window_us"] = max(e["ts"] + e["dur"] for e in ks) - t0
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
