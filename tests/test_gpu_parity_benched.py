"""GPU parity at the sizes and shapes the benchmark runs:

  * BASELINE configs[2] — DLRM-RMC2 / RMC3 at 32 tables x 10M rows x D=64
    (81.9 GB of tables on one B200), both FC paths (FC_AUTO = tcgen05 tf32,
    the benched path; FC_FP32 = FFMA), S in {1, 127, 128, 129, 330, 1000}
    (M-tile boundaries of the 128-row UMMA tile, the stream's mean, the max);
  * configs[1]/[3]/[4] — NCF, WND, MT-WND (4 stacks), DIN, DIEN at L=100
    (GRU and AUGRU, tensor-core and FFMA recurrences) at S=1000;
  * the e2e path: packed [dense | indices] pinned host queries through
    rs_forward_many (the call bench.py's e2e number is measured with),
    checked against the oracle and bitwise against single calls.

Shapes: /root/reference/proj/src/model_zoo.cpp:141-170 (zoo), BASELINE.json
configs, SURVEY.md D2/D3. Tolerances: tests/parity_rule.py.
"""
import numpy as np
import pytest

import paper_2001_02772_b200 as rs
from oracle import Oracle
from parity_rule import FP32, TF32, assert_attention_pooled, assert_close, assert_gru_state

pytestmark = pytest.mark.gpu

ROWS_CFG3 = 10_000_000
SIZES = (1, 127, 128, 129, 330, 1000)


def cfg3(model):
    """configs[2] shapes (bench.py workload_spec): dense stack ends at D=64 (D2)."""
    if model == "RMC2":
        return rs.ModelSpec("cfg3-DLRM-RMC2", dense_fc=rs.LayerStack([256, 128, 64]),
                            predict_fc=rs.LayerStack([512, 128, 1]),
                            embeddings=rs.EmbeddingConfig(32, 80, 64, "Sum"),
                            dense_input_dim=256)
    return rs.ModelSpec("cfg3-DLRM-RMC3", dense_fc=rs.LayerStack([2560, 512, 64]),
                        predict_fc=rs.LayerStack([512, 128, 1]),
                        embeddings=rs.EmbeddingConfig(32, 20, 64, "Sum"), dense_input_dim=256)


def cfg5_dien():
    return rs.ModelSpec("cfg5-DIEN", predict_fc=rs.LayerStack([200, 80, 2]),
                        embeddings=rs.EmbeddingConfig(20, 100, 32, "AttentionRNN"),
                        recurrent_hidden_dim=64)


def path_of(fc_mode):
    return FP32 if fc_mode == rs.FC_FP32 else TF32


def check_query(acc, orc, spec, dense, idx, fc_mode, what):
    out = acc.forward(dense, idx)
    ref, mag, pref, pmag = orc.forward64(dense, idx)
    assert_close(out, ref, mag, path_of(fc_mode), what + " logits")
    e = spec.embeddings
    pooled = acc.pooled(idx)
    if e.pooling == "Sum":
        assert np.array_equal(pooled, orc.sls_canonical(idx)), what + ": SLS not bit-exact"
    elif e.pooling == "AttentionRNN":
        assert_gru_state(pooled, pref, path_of(fc_mode), what + " GRU state")
    else:
        assert_attention_pooled(pooled, pref, pmag, e.lookups_per_table, what + " pooled")
    return out


@pytest.mark.parametrize("fc_mode", [rs.FC_AUTO, rs.FC_FP32], ids=["auto-tf32", "fp32"])
@pytest.mark.parametrize("model", ["RMC2", "RMC3"])
def test_cfg3_benched_sizes(model, fc_mode):
    """The headline configuration at every benched size, 10M-row tables."""
    spec = cfg3(model)
    acc = rs.Accelerator(spec, ROWS_CFG3, seed=1, max_query_size=1000, fc_mode=fc_mode)
    if fc_mode == rs.FC_AUTO:
        assert acc.info.fc_layers_tcgen05 > 0
    orc = Oracle(spec, ROWS_CFG3, seed=1)
    assert orc.p_in == acc.info.predict_input_dim == 656  # 64 + 64 + 528 pairs (D9)
    for k, S in enumerate(SIZES):
        dense, idx = rs.fill_query(spec, ROWS_CFG3, 77, k, S)
        check_query(acc, orc, spec, dense, idx, fc_mode, f"cfg3-{model} S={S}")
    acc.close()


@pytest.mark.parametrize("fc_mode", [rs.FC_AUTO, rs.FC_FP32], ids=["auto-tf32", "fp32"])
@pytest.mark.parametrize("name", ["NCF", "WND", "MT-WND", "DIN"])
def test_zoo_at_s1000(name, fc_mode):
    spec = rs.builtin_model(name)
    rows = 1_000_000
    acc = rs.Accelerator(spec, rows, seed=2, max_query_size=1000, fc_mode=fc_mode)
    orc = Oracle(spec, rows, seed=2)
    dense, idx = rs.fill_query(spec, rows, 31, 0, 1000)
    check_query(acc, orc, spec, dense, idx, fc_mode, f"{name} S=1000")
    acc.close()


@pytest.mark.parametrize("fc_mode", [rs.FC_AUTO, rs.FC_FP32], ids=["auto-tc-gru", "fp32-ffma-gru"])
@pytest.mark.parametrize("augru", [False, True], ids=["gru", "augru"])
def test_cfg5_dien_l100_s1000(augru, fc_mode):
    """configs[4] DIEN with 100-step sequences: the tensor-core recurrence
    (gru_tc_kernel, AUTO) and the FFMA recurrence (gru_kernel, FP32)."""
    spec = cfg5_dien()
    rows = 1_000_000
    acc = rs.Accelerator(spec, rows, seed=4, max_query_size=1000, fc_mode=fc_mode,
                         rnn_cell=rs.RNN_AUGRU if augru else rs.RNN_GRU)
    orc = Oracle(spec, rows, seed=4, augru=augru)
    for k, S in enumerate((1, 1000)):
        dense, idx = rs.fill_query(spec, rows, 13, k, S)
        check_query(acc, orc, spec, dense, idx, fc_mode, f"DIEN-L100 augru={augru} S={S}")
    acc.close()


@pytest.mark.parametrize("model", ["RMC2", "RMC3"])
def test_e2e_packed_host_queue_matches_oracle(model):
    """bench.py's e2e call: packed pinned host queries [dense | int64 indices]
    through rs_forward_many (8 lanes, two copy streams, FC_AUTO) at the cfg3
    shape — each query's logits within the tf32 rule of the oracle and
    bit-identical to the same query served alone."""
    spec = cfg3(model)
    acc = rs.Accelerator(spec, ROWS_CFG3, seed=1, max_query_size=1000, fc_mode=rs.FC_AUTO,
                         queue_depth=8)
    orc = Oracle(spec, ROWS_CFG3, seed=1)
    sizes = [330, 1, 1000, 128, 129, 57, 700, 127, 300, 2]
    qs = [rs.fill_query(spec, ROWS_CFG3, 91, k, S) for k, S in enumerate(sizes)]
    bufs, outs = [], []
    for (d, i), S in zip(qs, sizes):
        b = rs.PinnedBuffer(d.nbytes + i.nbytes)
        raw = b.view(np.uint8, (d.nbytes + i.nbytes,))
        raw[:d.nbytes] = d.reshape(-1).view(np.uint8)
        raw[d.nbytes:] = i.reshape(-1).view(np.uint8)
        bufs.append(b)
        outs.append(rs.PinnedBuffer(S * acc.output_dim * 4))
    batch = acc.batch(sizes, [b.ptr for b in bufs],
                      [b.ptr + d.nbytes for b, (d, _) in zip(bufs, qs)],
                      [o.ptr for o in outs], rs.MEM_HOST)
    svc = acc.forward_many(None, timed=True, prepared=batch)
    assert len(svc) == len(sizes) and (svc >= 0).all()
    for k, ((d, i), S) in enumerate(zip(qs, sizes)):
        got = outs[k].view(np.float32, (S, acc.output_dim)).copy()
        ref, mag, _, _ = orc.forward64(d, i)
        assert_close(got, ref, mag, TF32, f"e2e {model} query {k} S={S}")
        assert np.array_equal(got, acc.forward(d, i)), k
    acc.close()


@pytest.mark.parametrize("name", ["MT-WND", "WND", "NCF", "DLRM-RMC1", "DLRM-RMC2", "DLRM-RMC3",
                                  "DIN", "DIEN", "cfg3-RMC2", "cfg3-RMC3"])
def test_bf16_fc_variant(name):
    """RS_FC_BF16 (labelled lower-precision variant): tcgen05 kind::f16 with
    bf16 weights and activations, fp32 accumulate — within the stated bf16
    rule of the fp64 oracle at S in {1, 129, 1000}; the embedding stage is the
    fp32 one (SLS bit-exact)."""
    from parity_rule import BF16
    if name.startswith("cfg3"):
        spec, rows = cfg3(name[-4:]), 2_000_000
    else:
        spec, rows = rs.builtin_model(name), 200_000
    acc = rs.Accelerator(spec, rows, seed=3, max_query_size=1000, fc_mode=rs.FC_BF16)
    assert acc.info.fc_layers_tcgen05 > 0
    orc = Oracle(spec, rows, seed=3)
    for k, S in enumerate((1, 129, 1000)):
        dense, idx = rs.fill_query(spec, rows, 51, k, S)
        out = acc.forward(dense, idx)
        ref, mag, _, _ = orc.forward64(dense, idx)
        assert_close(out, ref, mag, BF16, f"bf16 {name} S={S}")
        if spec.embeddings.pooling == "Sum":
            assert np.array_equal(acc.pooled(idx), orc.sls_canonical(idx))
    acc.close()


@pytest.mark.parametrize("fc_mode", [rs.FC_AUTO, rs.FC_BF16], ids=["auto-tf32", "bf16"])
@pytest.mark.parametrize("name", ["MT-WND", "WND"])
def test_cta_pair_wide_graph(name, fc_mode):
    """RS_OPT_CTA_PAIRS: the wide graph (fc_tc2_kernel, tcgen05.mma.cta_group::2
    on 256-row CTA pairs) serves the queries whose 128-row tile count is even
    and at least the handle's threshold (256 items for batched stacks, 640
    with a single stack); odd tile counts stay on the one-CTA graph. Both
    handles (option on / default off) against the oracle at sizes on each
    side of the rule."""
    from parity_rule import BF16
    spec = rs.builtin_model(name)
    rows = 1_000_000
    path = BF16 if fc_mode == rs.FC_BF16 else TF32
    acc = rs.Accelerator(spec, rows, seed=4, max_query_size=1000, fc_mode=fc_mode)
    acc.set_option(rs.OPT_CTA_PAIRS, 1)
    base = rs.Accelerator(spec, rows, seed=4, max_query_size=1000, fc_mode=fc_mode)
    orc = Oracle(spec, rows, seed=4)
    for k, S in enumerate((255, 256, 300, 384, 640, 700, 1000)):
        dense, idx = rs.fill_query(spec, rows, 55, k, S)
        out = acc.forward(dense, idx)
        ref, mag, _, _ = orc.forward64(dense, idx)
        assert_close(out, ref, mag, path, f"{name} S={S} wide-graph handle")
        assert_close(base.forward(dense, idx), ref, mag, path, f"{name} S={S} one-CTA handle")
    acc.close()
    base.close()


def test_coresident_interaction_is_bit_identical(monkeypatch):
    """The 2-warp interaction CTAs the handle picks for strongly gather-bound
    models (cfg3 RMC2) compute every output in the 256-thread kernel's order:
    logits bit for bit against a handle forced to 256 threads
    (RS_INTER_THREADS)."""
    spec = cfg3("RMC2")
    rows = 100_000
    acc = rs.Accelerator(spec, rows, seed=8, max_query_size=1000, fc_mode=rs.FC_AUTO)
    monkeypatch.setenv("RS_INTER_THREADS", "256")
    ref = rs.Accelerator(spec, rows, seed=8, max_query_size=1000, fc_mode=rs.FC_AUTO)
    monkeypatch.delenv("RS_INTER_THREADS")
    qs = [rs.fill_query(spec, rows, 12, k, S) for k, S in enumerate((1, 129, 330, 1000))]
    for dense, idx in qs:
        a, b = acc.forward(dense, idx), ref.forward(dense, idx)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    acc.close()
    ref.close()
