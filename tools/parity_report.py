"""Parity report: for every zoo archetype and the BASELINE configs, the GPU
forward (fp32 FFMA path and tf32 tcgen05 path) against the fp64 oracle.

Prints one JSON object: max |gpu-ref|/mag (the tolerance-rule statistic),
normwise max|gpu-ref|/max|ref|, and whether SLS pooled sums are bit-exact.

  python tools/parity_report.py > profiles/parity_r2.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2001_02772_b200 as rs
    from oracle import Oracle
    cases = [(n, rs.builtin_model(n), 20000) for n in rs.zoo_names()]
    cases.append(("cfg1-RMC1", rs.ModelSpec("cfg1", dense_fc=rs.LayerStack([256, 128, 32]),
                                            predict_fc=rs.LayerStack([256, 64, 1]),
                                            embeddings=rs.EmbeddingConfig(8, 80, 32, "Sum"),
                                            dense_input_dim=256), 1_000_000))
    cases.append(("cfg5-DIEN-L100", rs.ModelSpec("cfg5", predict_fc=rs.LayerStack([200, 80, 2]),
                                                 embeddings=rs.EmbeddingConfig(20, 100, 32,
                                                                               "AttentionRNN"),
                                                 recurrent_hidden_dim=64), 100000))
    report = {}
    for name, spec, rows in cases:
        orc = Oracle(spec, rows, seed=3)
        dense, idx = rs.fill_query(spec, rows, 103, 0, 200)
        ref, mag, pref, pmag = orc.forward64(dense, idx)
        row = {}
        for mode, label in ((rs.FC_FP32, "fp32"), (rs.FC_TF32, "tf32"), (rs.FC_BF16, "bf16")):
            acc = rs.Accelerator(spec, rows, seed=3, max_query_size=200, fc_mode=mode)
            out = acc.forward(dense, idx).astype(np.float64)
            row[label] = {
                "max_err_over_mag": float(np.max(np.abs(out - ref) / mag)),
                "normwise_rel": float(np.max(np.abs(out - ref)) / np.max(np.abs(ref))),
                "tcgen05_layers": acc.info.fc_layers_tcgen05,
                # the SURVEY 8c statistic: max |d| / max(|ref|, mag 2^-10)
                "max_err_over_survey_scale": float(np.max(np.abs(out - ref) / np.maximum(
                    np.abs(ref), mag * 2.0 ** -10))),
            }
            if label == "fp32" and spec.embeddings.num_tables:
                pooled = acc.pooled(idx).astype(np.float64)
                if spec.embeddings.pooling == "Sum":
                    row["pooled_bit_exact"] = bool(np.array_equal(
                        acc.pooled(idx), orc.sls_canonical(idx)))
                row["pooled_max_err_over_mag"] = float(np.max(np.abs(pooled - pref) / pmag))
            acc.close()
        report[name] = row
        print(name, json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps({"items_per_query": 200, "oracle": "fp64 (oracle/forward.c)",
                      "models": report}, indent=1))


if __name__ == "__main__":
    main()
