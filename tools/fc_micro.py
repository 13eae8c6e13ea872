"""FC microbenchmark through the C-ABI: a model with no tables whose predict
stack is the layer(s) under test, so the forward graph is just the GEMM
kernel(s). Reports the graph's device time (CUDA events) per query size for
the FFMA (fp32) and tcgen05 (tf32) paths.

  python tools/fc_micro.py [--K 656] [--dims 512] [--sizes 128,323,1000]
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
    ap.add_argument("--K", type=int, default=656)
    ap.add_argument("--dims", default="512")
    ap.add_argument("--sizes", default="128,323,1000")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2001_02772_b200 as rs
    dims = [int(x) for x in args.dims.split(",")]
    spec = rs.ModelSpec("fc-micro", predict_fc=rs.LayerStack(dims),
                        embeddings=rs.EmbeddingConfig(0), dense_input_dim=args.K)
    sizes = [int(x) for x in args.sizes.split(",")]
    res = {}
    for mode, label in ((rs.FC_FP32, "fp32"), (rs.FC_TF32, "tf32")):
        acc = rs.Accelerator(spec, 1, max_query_size=max(sizes), fc_mode=mode)
        row = {}
        for S in sizes:
            d = torch.randn(S, args.K, device="cuda")
            o = torch.empty(S, acc.output_dim, device="cuda")
            ts = []
            for rep in range(9):
                t = acc.forward_ptr(S, d.data_ptr(), 0, o.data_ptr(), rs.MEM_DEVICE, timed=True)
                if rep >= 3:
                    ts.append(t.compute_ms * 1e3)
            us = statistics.median(ts)
            flops = 2.0 * S * sum(a * b for a, b in zip([args.K] + dims[:-1], dims))
            row[S] = {"us": round(us, 2), "tflops": round(flops / (us * 1e-6) / 1e12, 2)}
        res[label] = row
        acc.close()
    print(json.dumps({"K": args.K, "dims": dims, "graph_time": res}))


if __name__ == "__main__":
    main()
