"""DIEN pooled/logit error of the tensor-core GRU vs the fp64 oracle (L=20/100)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2001_02772_b200 as rs
    from oracle import Oracle
    for L in (20, 100):
        for augru in (False, True):
            spec = rs.ModelSpec(f"dien-L{L}", predict_fc=rs.LayerStack([200, 80, 2]),
                                embeddings=rs.EmbeddingConfig(20, L, 32, "AttentionRNN"),
                                recurrent_hidden_dim=64)
            acc = rs.Accelerator(spec, 50000, seed=3, max_query_size=256, fc_mode=rs.FC_TF32,
                                 rnn_cell=rs.RNN_AUGRU if augru else rs.RNN_GRU)
            orc = Oracle(spec, 50000, seed=3, augru=augru)
            dense, idx = rs.fill_query(spec, 50000, 103, 0, 200)
            out = acc.forward(dense, idx)
            pooled = acc.pooled(idx)
            ref, mag, pref, pmag = orc.forward64(dense, idx)
            d = np.abs(pooled - pref)
            e = np.abs(out - ref)
            print(f"L={L} augru={augru}: pooled max|d|/mag {np.max(d / np.maximum(pmag, 1e-30)):.2e} "
                  f"normwise {np.max(d) / np.max(np.abs(pref)):.2e}; logits normwise "
                  f"{np.max(e) / np.max(np.abs(ref)):.2e}", flush=True)
            acc.close()


if __name__ == "__main__":
    main()
