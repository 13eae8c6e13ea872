"""The CPU side of the split (rs_host_model / rs_host_forward, SURVEY §8a a9,
§8f-4): the whole forward of every zoo archetype and BASELINE config on the
host cores, against the fp64 oracle under the fp32 rule of
tests/parity_rule.py — no GPU needed. Same seeded parameters as the device
handle, so a query gives the same logits on either side of the
split within tolerance."""
import numpy as np
import pytest

import paper_2001_02772_b200 as rs
from oracle import Oracle
from parity_rule import FP32, assert_close


def cfg_models():
    return {
        "cfg1-RMC1": rs.ModelSpec("cfg1-RMC1", dense_fc=rs.LayerStack([256, 128, 32]),
                                  predict_fc=rs.LayerStack([256, 64, 1]),
                                  embeddings=rs.EmbeddingConfig(8, 80, 32, "Sum"),
                                  dense_input_dim=256),
        "cfg3-RMC2": rs.ModelSpec("cfg3-RMC2", dense_fc=rs.LayerStack([256, 128, 64]),
                                  predict_fc=rs.LayerStack([512, 128, 1]),
                                  embeddings=rs.EmbeddingConfig(32, 80, 64, "Sum"),
                                  dense_input_dim=256),
        "cfg5-DIEN": rs.ModelSpec("cfg5-DIEN", predict_fc=rs.LayerStack([200, 80, 2]),
                                  embeddings=rs.EmbeddingConfig(20, 100, 32, "AttentionRNN"),
                                  recurrent_hidden_dim=64),
        "odd-D": rs.ModelSpec("odd-D", dense_fc=rs.LayerStack([13, 24]),
                              predict_fc=rs.LayerStack([7, 3]),
                              embeddings=rs.EmbeddingConfig(3, 5, 24, "Sum"), dense_input_dim=13),
    }


@pytest.mark.parametrize("name", ["NCF", "WND", "MT-WND", "DLRM-RMC1", "DLRM-RMC2", "DLRM-RMC3",
                                  "DIN", "DIEN"])
def test_host_forward_zoo_matches_oracle(name):
    spec = rs.builtin_model(name)
    rows = 3000
    host = rs.HostModel(spec, rows, seed=3)
    orc = Oracle(spec, rows, seed=3)
    for S in (1, 9):
        dense, idx = rs.fill_query(spec, rows, 21, S, S)
        ref, mag, _, _ = orc.forward64(dense, idx)
        assert_close(host.forward(dense, idx), ref, mag, FP32, f"host {name} S={S}")
    host.close()


@pytest.mark.parametrize("name", ["cfg1-RMC1", "cfg3-RMC2", "cfg5-DIEN", "odd-D"])
def test_host_forward_configs_match_oracle(name):
    spec = cfg_models()[name]
    rows = 5000
    host = rs.HostModel(spec, rows, seed=2)
    orc = Oracle(spec, rows, seed=2)
    S = 3 if name == "cfg5-DIEN" else 20
    dense, idx = rs.fill_query(spec, rows, 4, 0, S)
    ref, mag, _, _ = orc.forward64(dense, idx)
    assert_close(host.forward(dense, idx), ref, mag, FP32, f"host {name}")
    host.close()


def test_host_forward_augru_and_threads_and_errors():
    spec = rs.builtin_model("DIEN")
    rows = 2000
    host = rs.HostModel(spec, rows, seed=5, rnn_cell=rs.RNN_AUGRU)
    orc = Oracle(spec, rows, seed=5, augru=True)
    dense, idx = rs.fill_query(spec, rows, 8, 0, 6)
    ref, mag, _, _ = orc.forward64(dense, idx)
    one = host.forward(dense, idx, threads=1)
    assert_close(one, ref, mag, FP32, "host AUGRU")
    # items dealt to threads: each item's arithmetic is the same
    assert np.array_equal(host.forward(dense, idx, threads=4), one)
    bad = idx.copy()
    bad[2, 1, 3] = rows
    with pytest.raises(rs.IndexOutOfRange):
        host.forward(dense, bad)
    host.close()
    with pytest.raises(rs.InvalidArgument):
        rs.HostModel(rs.ModelSpec("bad", dense_fc=rs.LayerStack([8, 16]),
                                  predict_fc=rs.LayerStack([4]),
                                  embeddings=rs.EmbeddingConfig(2, 3, 32, "Sum"),
                                  dense_input_dim=4), 100)


def test_serve_hybrid_cpu_only_splits_and_matches_forward():
    """rs_serve_hybrid with no replica: every query split into floor(S/B)
    requests of B items plus S mod B (proj/src/sim.cpp:184-188) on a pool of
    host worker threads; each query's logits equal the whole-query host
    forward bit for bit (per-item arithmetic), latencies positive."""
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 4000
    host = rs.HostModel(spec, rows, seed=7)
    sizes = [1, 63, 64, 65, 200, 7, 130]
    qs = [rs.fill_query(spec, rows, 3, k, S) for k, S in enumerate(sizes)]
    outs = [np.zeros((S, host.output_dim), dtype=np.float32) for S in sizes]
    b = rs.Accelerator.batch(sizes, [d.ctypes.data for d, _ in qs], [i.ctypes.data for _, i in qs],
                             [o.ctypes.data for o in outs], rs.MEM_HOST)
    lat, off = rs.serve_hybrid(host, 3, 64, 0, [], b, np.arange(len(sizes)) * 1e-3)
    assert (off == 0).all() and (lat > 0).all()
    for (d, i), o in zip(qs, outs):
        assert np.array_equal(o, host.forward(d, i))
    with pytest.raises(rs.InvalidArgument):
        rs.serve_hybrid(host, 0, 64, 0, [], b, np.zeros(len(sizes)))
    host.close()
