"""Operator API and accounting: the product's host mirror (model.cpp) against the
reference's own known answers (proj/tests/test_model_zoo.cpp, test_platform.cpp)
and, bit-for-bit, against the compiled reference library (oracle/_ref)."""
import ctypes as C

import numpy as np
import pytest

from paper_2001_02772_b200 import (EmbeddingConfig, LayerStack, ModelSpec, accel_input_bytes,
                                   builtin_model, predict_input_dim, sla_target, work,
                                   zoo_names)
import paper_2001_02772_b200 as rs


def test_zoo_has_the_eight_archetypes():                       # test_model_zoo.cpp:7-14
    names = zoo_names()
    assert names == ["NCF", "WND", "MT-WND", "DLRM-RMC1", "DLRM-RMC2", "DLRM-RMC3", "DIN",
                     "DIEN"]
    for n in names:
        builtin_model(n)
    with pytest.raises(rs.UnknownModel):
        builtin_model("")


def test_rmc1_and_ncf_table_parameters():                      # test_model_zoo.cpp:16-31
    m = builtin_model("DLRM-RMC1")
    assert m.dense_fc.dims == [256, 128, 32]
    assert m.predict_fc.dims == [256, 64, 1]
    assert (m.embeddings.num_tables, m.embeddings.lookups_per_table) == (10, 80)
    assert m.embeddings.pooling == "Sum"
    ncf = builtin_model("NCF")
    assert ncf.dense_fc is None
    assert ncf.predict_fc.dims == [256, 256, 128]
    assert (ncf.embeddings.num_tables, ncf.embeddings.lookups_per_table) == (4, 1)
    assert ncf.embeddings.pooling == "Concat"


def test_single_fc_layer_flops():                              # test_model_zoo.cpp:33-44
    m = ModelSpec("synthetic-fc", dense_fc=LayerStack([2]), predict_fc=LayerStack([1]),
                  embeddings=EmbeddingConfig(num_tables=0), dense_input_dim=4)
    m.validate()
    assert work(m, 1)["DenseFC"][0] == 16.0


def test_rmc1_embedding_bytes():                               # test_model_zoo.cpp:46-50
    assert work(builtin_model("DLRM-RMC1"), 1)["EmbeddingLookup"][1] == 102400.0


@pytest.mark.parametrize("name", ["NCF", "WND", "MT-WND", "DLRM-RMC1", "DLRM-RMC2",
                                  "DLRM-RMC3", "DIN", "DIEN"])
def test_work_is_linear_in_batch(name):                        # test_model_zoo.cpp:52-66
    m = builtin_model(name)
    base = work(m, 3)
    for k in (2, 4, 8):
        s = work(m, 3 * k)
        np.testing.assert_allclose(s.flops, np.array(base.flops) * k, rtol=1e-12)
        np.testing.assert_allclose(s.bytes, np.array(base.bytes) * k, rtol=1e-12)


def test_validation_rejects_malformed_specs():                 # test_model_zoo.cpp:92-103
    m = builtin_model("DIEN")
    m.recurrent_hidden_dim = None
    with pytest.raises(rs.InvalidArgument):
        m.validate()
    bad = builtin_model("NCF")
    bad.predict_fc = LayerStack([])
    with pytest.raises(rs.InvalidArgument):
        bad.validate()
    dims = builtin_model("NCF")
    dims.embeddings.embedding_dim = 4
    with pytest.raises(rs.InvalidArgument):
        dims.validate()


def test_predict_input_widths():
    # NCF 128, WND/MT-WND 1640, RMC1 119 (D9), RMC2 884, RMC3 119,
    # DIN 640, DIEN 1280.
    want = {"NCF": 128, "WND": 1640, "MT-WND": 1640, "DLRM-RMC1": 119, "DLRM-RMC2": 884,
            "DLRM-RMC3": 119, "DIN": 640, "DIEN": 1280}
    for n, w in want.items():
        assert predict_input_dim(builtin_model(n)) == w


def test_rmc1_predict_fc_flops_per_item_matches_d9():
    # PredictFC flops for RMC1 = 2*(119*256 + 256*64 + 64*1) = 93,824
    assert work(builtin_model("DLRM-RMC1"), 1)["PredictFC"][0] == 93824.0


def test_accel_input_bytes_per_item():
    want = {"NCF": 32, "WND": 4160, "DLRM-RMC1": 7424, "DLRM-RMC2": 26624,
            "DLRM-RMC3": 2624, "DIN": 32000, "DIEN": 3200}
    for n, b in want.items():
        assert accel_input_bytes(builtin_model(n), 1) == b


def test_sla_targets():                                        # autotune.cpp:73-88
    assert sla_target("DLRM-RMC1", "medium") == 0.100
    assert sla_target("DLRM-RMC2", "low") == 0.200
    assert sla_target("DIEN", "high") == pytest.approx(0.0525)
    with pytest.raises(rs.UnknownModel):
        sla_target("ResNet50", "medium")


# ---- bit-for-bit against the compiled reference ----------------------------
def _ref_or_skip(orc):
    if not orc.ref_available():
        pytest.skip("oracle/_ref/librecsim_ref.so not built (no /root/reference here)")
    return orc.ref


def _cfg3(name):
    """BASELINE cfg3 shapes as inline ModelSpecs."""
    L = 80 if name == "RMC2" else 20
    dense = [256, 128, 64] if name == "RMC2" else [2560, 512, 64]
    pred = [512, 128, 1]
    return ModelSpec(f"cfg3-{name}", dense_fc=LayerStack(dense), predict_fc=LayerStack(pred),
                     embeddings=EmbeddingConfig(32, L, 64, "Sum"), dense_input_dim=256)


def _inline_specs():
    yield ModelSpec("cfg1-RMC1", dense_fc=LayerStack([256, 128, 32]),
                    predict_fc=LayerStack([256, 64, 1]),
                    embeddings=EmbeddingConfig(8, 80, 32, "Sum"), dense_input_dim=256)
    yield _cfg3("RMC2")
    yield _cfg3("RMC3")
    yield ModelSpec("cfg5-DIEN", predict_fc=LayerStack([200, 80, 2]),
                    embeddings=EmbeddingConfig(20, 100, 32, "AttentionRNN"),
                    recurrent_hidden_dim=64)
    yield ModelSpec("sum-no-dense", predict_fc=LayerStack([3]),
                    embeddings=EmbeddingConfig(5, 7, 24, "Sum"), dense_input_dim=9)
    yield ModelSpec("empty", predict_fc=LayerStack([2]), embeddings=EmbeddingConfig(0))


@pytest.mark.parametrize("batch", [1, 7, 64, 1000])
def test_work_equals_reference_bitwise(orc, batch):
    ref = _ref_or_skip(orc)
    specs = [builtin_model(n) for n in zoo_names()] + list(_inline_specs())
    for spec in specs:
        om = orc.model_to_or(spec)
        f = (C.c_double * 7)()
        b = (C.c_double * 7)()
        g = C.c_double()
        assert ref.ref_work(C.byref(om), batch, f, b, C.byref(g)) == 0
        w = work(spec, batch)
        assert list(f) == w.flops, spec.name
        assert list(b) == w.bytes, spec.name
        assert g.value == w.gather_stream
        ib = C.c_double()
        assert ref.ref_accel_input_bytes(C.byref(om), batch, C.byref(ib)) == 0
        assert ib.value == accel_input_bytes(spec, batch)


def test_builtin_models_equal_reference(orc):
    ref = _ref_or_skip(orc)
    for n in zoo_names():
        om = orc.OrModel()
        assert ref.ref_builtin_model(n.encode(), C.byref(om)) == 0
        assert bytes(om) == bytes(orc.model_to_or(builtin_model(n))), n


def test_sla_targets_equal_reference(orc):
    ref = _ref_or_skip(orc)
    for n in zoo_names():
        for lvl in ("low", "medium", "high"):
            v = C.c_double()
            assert ref.ref_sla_target(n.encode(), lvl.encode(), C.byref(v)) == 0
            assert v.value == sla_target(n, lvl)


def test_validation_agrees_with_reference(orc):
    ref = _ref_or_skip(orc)
    cases = list(_inline_specs())
    bad = builtin_model("DIN")
    bad.embeddings.embedding_dim = 300
    cases.append(bad)
    bad2 = builtin_model("DIEN")
    bad2.recurrent_hidden_dim = None
    cases.append(bad2)
    bad3 = builtin_model("NCF")
    bad3.num_parallel_predict_stacks = 0
    cases.append(bad3)
    for spec in cases:
        r = ref.ref_validate(C.byref(orc.model_to_or(spec)))
        try:
            spec.validate()
            mine = 0
        except rs.InvalidArgument:
            mine = -1
        assert mine == r, spec.name
