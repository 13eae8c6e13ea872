"""Tensor-pipe evidence for the tcgen05 kernels.

Runs ncu (one GPU, --clock-control none) on tools/run_once.py for each case and
reads per-launch tensor-pipe counters of every fc_tc_kernel / gru_tc_kernel
launch, plus the algorithmic flops of that launch, into one JSON:

  python tools/tensor_profile.py > profiles/r2_tensor_pipe.json

Cases: MT-WND (zoo, 4 predict stacks, 1640-1024-512-256) at S in {16, 64,
256, 1024} — BASELINE configs[3]'s batch sweep; cfg3 DLRM-RMC2 at S=330 (the
headline's mean query); cfg5 DIEN (L=100) at S=300 — the tensor-core GRU.
Flops per launch: 2*M*N*K per stack (M = S rows of the tile grid) for an FC
layer; 2*S*T*L*(D+H)*4H for the GRU (x- and h-projections of all gates,
gru_tcgen05.cu). Peak: tf32 = 0.5 x measured bf16 (MEASURED_PEAKS.json).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "launch__grid_size",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_tensor_subpipe_hmma.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__bytes_read.sum", "dram__bytes_write.sum"]

CASES = [("mt-wnd", 16), ("mt-wnd", 64), ("mt-wnd", 256), ("mt-wnd", 1024),
         ("cfg3-rmc2", 330), ("cfg5-dien", 300)]
if os.environ.get("TP_CASES"):  # e.g. "mt-wnd:1024,wnd:1024"
    CASES = [(c.split(":")[0], int(c.split(":")[1])) for c in os.environ["TP_CASES"].split(",")]


def layer_flops(workload, S):
    """Algorithmic flops of each tcgen05 launch in graph order."""
    sys.path.insert(0, ROOT)
    import paper_2001_02772_b200 as rs
    import bench
    spec, rows, _ = bench.workload_spec(rs, workload)
    out = []
    e = spec.embeddings
    if e.pooling == "AttentionRNN":
        H, D = spec.recurrent_hidden_dim, e.embedding_dim
        out.append(("gru_tc", 2.0 * S * e.num_tables * e.lookups_per_table * (D + H) * 4 * H))
    if spec.dense_fc is not None:
        k = spec.dense_input_dim
        for n in spec.dense_fc.dims:
            out.append(("dense_fc", 2.0 * S * k * n))
            k = n
    k = rs.predict_input_dim(spec)
    z = spec.num_parallel_predict_stacks
    for n in spec.predict_fc.dims:
        out.append(("predict_fc", 2.0 * S * k * n * z))
        k = n
    return out


FC = os.environ.get("TP_FC", "auto")  # auto (tf32) | bf16
TAG = os.environ.get("TP_TAG", "")


def run_case(workload, S):
    rep = os.path.join(ROOT, "gpurun_out", f"tp_{FC}{TAG}_{workload}_{S}.csv")
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "--csv",
           "-k", "regex:fc_tc|gru_tc", "--log-file", rep,
           sys.executable, os.path.join(ROOT, "tools", "run_once.py"), "--workload", workload,
           "--S", str(S), "--fc", FC, "--reps", "2"]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
    rows = list(csv.reader(open(rep)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value",
                                             "Metric Unit"))
    ii = hdr.index("ID")
    launches = {}
    for r in data:
        d = launches.setdefault(int(r[ii]), {"kernel": r[ki].split("(")[0].replace(
            "(anonymous namespace)::", "")})
        d[r[mi]] = (float(r[vi].replace(",", "")) if r[vi] not in ("", "n/a") else None, r[ui])
    return [launches[k] for k in sorted(launches)]


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    tf32 = 0.5 * peaks["bf16_tflops"] if FC != "bf16" else peaks["bf16_tflops"]
    out = {"fc": FC, "peak_tflops": tf32,
           "peak_source": ("0.5 x MEASURED_PEAKS bf16_tflops (tf32 rate)" if FC != "bf16"
                           else "MEASURED_PEAKS bf16_tflops"),
           "ncu": "--metrics " + ",".join(METRICS) + " --clock-control none (cold, serialised "
                  "launches; second forward of two)", "cases": []}
    for workload, S in CASES:
        launches = run_case(workload, S)
        flops = layer_flops(workload, S)
        per_fwd = len(launches) // 2
        second = launches[per_fwd:]           # the second forward (warm weights)
        tc_flops = [f for f in flops]
        res = []
        # the last predict layer may be fused into the previous epilogue
        for j, L in enumerate(second):
            t_ns = L["gpu__time_duration.sum"][0] * {"nsecond": 1, "usecond": 1e3,
                                                     "msecond": 1e6}.get(
                L["gpu__time_duration.sum"][1], 1)
            fl = tc_flops[j][1] if j < len(tc_flops) else None
            if j == len(second) - 1 and len(tc_flops) > len(second):
                fl = sum(f for _, f in tc_flops[j:])    # fused narrow last layer
            rec = {"kernel": L["kernel"], "layer": tc_flops[j][0] if j < len(tc_flops) else "?",
                   "time_us": t_ns / 1e3, "flops": fl,
                   "tflops": fl / (t_ns * 1e-9) / 1e12 if fl else None}
            rec["frac_of_tf32_peak"] = rec["tflops"] / tf32 if rec["tflops"] else None
            for m in METRICS[1:]:
                rec[m] = L.get(m, (None,))[0]
            # executed MMA flops from the tensor-pipe instruction count: each
            # tcgen05.mma kind::tf32 is M=128 x N=BN x K=8 (padding included)
            name = L["kernel"]
            inst = rec.get("sm__inst_executed_pipe_tensor_subpipe_hmma.sum")
            if "fc_tc_kernel<" in name and inst:
                bn = int(name.split("fc_tc_kernel<")[1].split(",")[0])
                rec["executed_mma_flops"] = inst * 2 * 128 * bn * (16 if FC == "bf16" else 8)
                rec["executed_over_algorithmic"] = rec["executed_mma_flops"] / fl if fl else None
            elif "fc_tc2_kernel<" in name and inst:
                # cta_group::2: one instruction (leader SM) = M 256 x N 256 x K 8
                rec["executed_mma_flops"] = inst * 2 * 256 * 256 * (16 if FC == "bf16" else 8)
                rec["executed_over_algorithmic"] = rec["executed_mma_flops"] / fl if fl else None
            res.append(rec)
        tot_f = sum(r["flops"] or 0 for r in res)
        tot_t = sum(r["time_us"] for r in res) * 1e-6
        out["cases"].append({"workload": workload, "S": S, "launches": res,
                             "stack_tflops": tot_f / tot_t / 1e12 if tot_t else None,
                             "stack_frac_of_tf32_peak": tot_f / tot_t / 1e12 / tf32
                             if tot_t else None})
        print(workload, S, json.dumps(out["cases"][-1]["stack_tflops"]), file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
