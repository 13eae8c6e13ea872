"""Run a few forwards of one model through the C-ABI (profiling driver for ncu).

  python tools/run_once.py --model DIEN --L 100 --S 300 --fc tf32 --reps 3
  python tools/run_once.py --workload cfg3-rmc2 --S 300 --pooled --reps 3

--workload takes bench.py's workload names (same spec and table rows), so an
`ncu --set full` capture of the SLS kernel here has the bench's shape with a
known item count S (dram bytes per launch / S = traffic per item).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="DIEN")
    ap.add_argument("--workload", default="", help="a bench.py workload name")
    ap.add_argument("--L", type=int, default=0, help="override lookups_per_table")
    ap.add_argument("--S", type=int, default=300)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--fc", choices=["fp32", "tf32", "auto", "bf16"], default="tf32")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--pooled", action="store_true", help="embedding stage only (rs_pooled)")
    args = ap.parse_args()
    import paper_2001_02772_b200 as rs
    if args.workload:
        import bench
        spec, rows, _ = bench.workload_spec(rs, args.workload)
    else:
        spec, rows = rs.builtin_model(args.model), args.rows
    if args.L:
        spec.embeddings.lookups_per_table = args.L
    mode = {"fp32": rs.FC_FP32, "tf32": rs.FC_TF32, "auto": rs.FC_AUTO, "bf16": rs.FC_BF16}[args.fc]
    acc = rs.Accelerator(spec, rows, max_query_size=max(args.S, 1), fc_mode=mode)
    dense, idx = rs.fill_query(spec, rows, 5, 0, args.S)
    for r in range(args.reps):
        # distinct indices per rep so no launch re-reads the previous one's rows from L2
        if r:
            dense, idx = rs.fill_query(spec, rows, 5, r, args.S)
        if args.pooled:
            acc.pooled(idx)
        else:
            acc.forward(dense, idx)
    print("ok", acc.info.kernels_per_forward, "S", args.S)


if __name__ == "__main__":
    main()
