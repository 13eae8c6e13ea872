"""Summarise ncu outputs into profiles/: per-kernel launch-list shares (csv from
--metrics gpu__time_duration.sum) and key metrics of a --set full report."""
import collections
import csv
import json
import subprocess
import sys


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name")
    agg = collections.defaultdict(list)
    for r in data:
        if r[mi] != "gpu__time_duration.sum":  # other --metrics columns
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                 "ms": 1e3}.get(r[ui], 1.0)
        agg[r[ki].split("(")[0].replace("(anonymous namespace)::", "")].append(v * scale)
    tot = sum(sum(v) for k, v in agg.items() if "init_tables" not in k)
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        if "init_tables" in k:
            continue
        out.append({"kernel": k, "launches": len(v), "mean_us": round(sum(v) / len(v), 2),
                    "total_ms": round(sum(v) / 1e3, 3), "share": round(sum(v) / tot, 4)})
    return out


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
           "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active"]


def full_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                d[m] = r[hdr.index(m)] + " " + units[hdr.index(m)]
        out.append(d)
    return out


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    res = launch_shares(path) if kind == "launches" else full_report(path)
    print(json.dumps(res, indent=1))
