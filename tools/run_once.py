"""Run a few forwards of one model through the C-ABI (profiling driver for ncu).

  python tools/run_once.py --model DIEN --L 100 --S 300 --fc tf32 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="DIEN")
    ap.add_argument("--L", type=int, default=0, help="override lookups_per_table")
    ap.add_argument("--S", type=int, default=300)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--fc", choices=["fp32", "tf32", "auto"], default="tf32")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import paper_2001_02772_b200 as rs
    spec = rs.builtin_model(args.model)
    if args.L:
        spec.embeddings.lookups_per_table = args.L
    mode = {"fp32": rs.FC_FP32, "tf32": rs.FC_TF32, "auto": rs.FC_AUTO}[args.fc]
    acc = rs.Accelerator(spec, args.rows, max_query_size=max(args.S, 1), fc_mode=mode)
    dense, idx = rs.fill_query(spec, args.rows, 5, 0, args.S)
    for _ in range(args.reps):
        acc.forward(dense, idx)
    print("ok", acc.info.kernels_per_forward)


if __name__ == "__main__":
    main()
