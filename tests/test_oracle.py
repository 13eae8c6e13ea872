"""The oracle itself, pinned before it is trusted: against the committed torch
golden fixtures (tests/golden/make_golden.py) and against the product's host-side
implementation of the shared input spec."""
import os
import sys

import numpy as np
import pytest

import paper_2001_02772_b200 as rs
from oracle import Oracle, table_value

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden as mg  # noqa: E402

GOLD = np.load(os.path.join(HERE, "golden", "forward_golden.npz"))


def spec_of(name, cfg):
    return rs.ModelSpec(
        name=name, dense_fc=rs.LayerStack(cfg["dense_fc"]) if cfg["dense_fc"] else None,
        predict_fc=rs.LayerStack(cfg["predict_fc"]), num_parallel_predict_stacks=cfg["stacks"],
        embeddings=rs.EmbeddingConfig(cfg["T"], cfg["L"], cfg["D"], cfg["pooling"]),
        dense_input_dim=cfg["dense_in"], recurrent_hidden_dim=cfg["hidden"] or None)


CASES = [(n, a) for n, c in mg.MODELS.items()
         for a in ([False, True] if c["pooling"] == "AttentionRNN" else [False])]


@pytest.mark.parametrize("name,augru", CASES)
def test_oracle_matches_torch_golden(name, augru):
    key = name + ("-augru" if augru else "")
    spec = spec_of(name, mg.MODELS[name])
    o = Oracle(spec, mg.ROWS, seed=mg.SEED, augru=augru)
    out, mag, pooled, _ = o.forward64(GOLD[key + "/dense"], GOLD[key + "/idx"])
    np.testing.assert_allclose(out, GOLD[key + "/out"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(pooled, GOLD[key + "/pooled"], rtol=1e-12, atol=1e-14)
    assert np.all(mag >= np.abs(out) * (1 - 1e-12))   # mag bounds |value|
    assert o.p_in == rs.predict_input_dim(spec)


def test_golden_outputs_are_not_degenerate():
    for n, a in CASES:
        out = GOLD[n + ("-augru" if a else "") + "/out"]
        assert np.ptp(out, axis=0).max() > 1e-4, n


def test_table_spec_pin():
    row = GOLD["spec/table0_row7"]
    got = np.array([table_value(mg.SEED, 0, 7, c, 8) for c in range(8)], dtype=np.float32)
    assert np.array_equal(row, got)


@pytest.mark.parametrize("model", ["DLRM-RMC1", "WND", "DIN", "DIEN"])
def test_product_and_oracle_inputs_agree_bitwise(model):
    spec = rs.builtin_model(model)
    o = Oracle(spec, 123457, seed=9)
    d1, i1 = rs.fill_query(spec, 123457, seed=9, query_id=77, size=5)
    d2, i2 = o.fill_query(77, 5)
    assert np.array_equal(d1, d2) and np.array_equal(i1, i2)
    assert i1.min() >= 0 and i1.max() < 123457
    if d1.size:
        assert -1 <= d1.min() and d1.max() < 1


def test_canonical_sls_is_a_reordering_of_the_exact_sum():
    spec = rs.builtin_model("DLRM-RMC1")
    o = Oracle(spec, 5000, seed=2)
    _, idx = o.fill_query(1, 4)
    canon = o.sls_canonical(idx)
    _, _, pooled, pmag = o.forward64(np.zeros((4, 256), np.float32), idx)
    err = np.abs(canon - pooled) / pmag
    assert err.max() < 80 * 2 ** -24


def test_fp32_oracle_tracks_fp64():
    spec = rs.builtin_model("DLRM-RMC3")
    o = Oracle(spec, 5000, seed=2)
    dense, idx = o.fill_query(3, 6)
    out, mag, _, _ = o.forward64(dense, idx)
    o32 = o.forward32(dense, idx)
    assert np.max(np.abs(o32 - out) / mag) < 1e-5


def test_out_of_range_index_is_an_error():
    spec = rs.builtin_model("DLRM-RMC1")
    o = Oracle(spec, 100, seed=2)
    _, idx = o.fill_query(1, 2)
    idx[1, 3, 5] = 100
    with pytest.raises(RuntimeError):
        o.forward64(np.zeros((2, 256), np.float32), idx)
