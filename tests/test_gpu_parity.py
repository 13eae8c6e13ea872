"""GPU parity: the sm_100a path, called through the C-ABI, against the CPU oracle
on the same seeded inputs.

Tolerance rule: tests/parity_rule.py (SURVEY.md §8c's elementwise rule
|d| <= 1e-5*max(|ref|, Σ|terms|*2^-10) for the fp32 path; 2^-10*Σ|terms| and
normwise 5e-3 for the tf32 tcgen05 path; SLS pooled sums bit-identical; the
bounded GRU state on its unit scale).
"""
import numpy as np
import pytest

import paper_2001_02772_b200 as rs
from oracle import Oracle
from parity_rule import FP32, TF32, assert_attention_pooled, assert_close, assert_gru_state

pytestmark = pytest.mark.gpu

# measured-slower alternatives exist only in an experiments build (make EXPERIMENTS=1)
needs_experiments = pytest.mark.skipif(not rs.experiments_built(),
                                       reason="library built without EXPERIMENTS=1")

# path labels kept as the tolerance argument of check_forward
FP32_TOL = FP32
TF32_TOL = TF32


def rel_err(got, ref, mag):
    """max |gpu - ref| / mag (reported statistic)."""
    d = np.abs(got.astype(np.float64) - ref)
    return float(np.max(d / np.maximum(mag, 1e-30)))


def check_fp32(got, ref, mag, what=""):
    return assert_close(got, ref, mag, FP32, what)


def check_forward(spec, rows, S, fc_mode=rs.FC_FP32, augru=False, seed=3, qid=0, tol=FP32_TOL,
                  max_q=256):
    acc = rs.Accelerator(spec, rows, seed=seed, max_query_size=max_q, fc_mode=fc_mode,
                         rnn_cell=rs.RNN_AUGRU if augru else rs.RNN_GRU)
    orc = Oracle(spec, rows, seed=seed, augru=augru)
    dense, idx = rs.fill_query(spec, rows, seed=seed + 100, query_id=qid, size=S)
    out = acc.forward(dense, idx)
    ref, mag, pref, pmag = orc.forward64(dense, idx)
    assert_close(out, ref, mag, tol, f"{spec.name} logits S={S}")
    if spec.embeddings.num_tables > 0:
        pooled = acc.pooled(idx)
        if spec.embeddings.pooling == "Sum":
            assert np.array_equal(pooled, orc.sls_canonical(idx)), "SLS not bit-exact"
        elif spec.embeddings.pooling == "AttentionRNN":
            # the tf32/auto handle pools DIEN with the tensor-core recurrence
            tc_rnn = fc_mode != rs.FC_FP32
            assert_gru_state(pooled, pref, TF32 if tc_rnn else FP32, f"{spec.name} GRU state")
        else:
            assert_attention_pooled(pooled, pref, pmag, spec.embeddings.lookups_per_table,
                                    f"{spec.name} pooled")
    acc.close()
    return rel_err(out, ref, mag)


@pytest.mark.parametrize("name", ["NCF", "WND", "MT-WND", "DLRM-RMC1", "DLRM-RMC2",
                                  "DLRM-RMC3", "DIN", "DIEN"])
def test_zoo_fp32(name):
    check_forward(rs.builtin_model(name), rows=20000, S=9)


def test_dien_augru():
    check_forward(rs.builtin_model("DIEN"), rows=5000, S=7, augru=True)


@pytest.mark.parametrize("D", [8, 16, 32, 64, 128, 256, 24, 12])
def test_sls_bit_exact_every_vector_width(D):
    spec = rs.ModelSpec(f"sls-D{D}", dense_fc=None, predict_fc=rs.LayerStack([4]),
                        embeddings=rs.EmbeddingConfig(3, 37, D, "Sum"), dense_input_dim=0)
    check_forward(spec, rows=3001, S=11)


def test_cfg1_rmc1_single_query_batch64():
    """BASELINE configs[0]: DLRM-RMC1, 8 tables x 1M rows x dim 32, 80 lookups,
    one query of 64 items, fp32."""
    spec = rs.ModelSpec("cfg1-RMC1", dense_fc=rs.LayerStack([256, 128, 32]),
                        predict_fc=rs.LayerStack([256, 64, 1]),
                        embeddings=rs.EmbeddingConfig(8, 80, 32, "Sum"), dense_input_dim=256)
    check_forward(spec, rows=1_000_000, S=64, max_q=64)


@pytest.mark.parametrize("name", ["MT-WND", "WND", "DLRM-RMC3", "DLRM-RMC1", "DLRM-RMC2", "NCF",
                                  "DIN", "DIEN"])
def test_tf32_tcgen05_path(name):
    spec = rs.builtin_model(name)
    acc = rs.Accelerator(spec, 2000, seed=1, max_query_size=300, fc_mode=rs.FC_TF32)
    assert acc.info.fc_layers_tcgen05 > 0
    acc.close()
    for S in (1, 130, 300):
        check_forward(spec, rows=2000, S=S, fc_mode=rs.FC_TF32, tol=TF32_TOL, max_q=300)


def test_edges_sizes_and_errors():
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 1000
    acc = rs.Accelerator(spec, rows, seed=5, max_query_size=50)
    orc = Oracle(spec, rows, seed=5)
    for S in (1, 50):
        dense, idx = rs.fill_query(spec, rows, 1, S, S)
        ref, mag, _, _ = orc.forward64(dense, idx)
        check_fp32(acc.forward(dense, idx), ref, mag)
    dense, idx = rs.fill_query(spec, rows, 1, 0, 51)
    with pytest.raises(rs.CapacityError):
        acc.forward(dense, idx)
    dense, idx = rs.fill_query(spec, rows, 1, 0, 4)
    idx[2, 7, 11] = rows            # out of range
    with pytest.raises(rs.IndexOutOfRange):
        acc.forward(dense, idx)
    idx[2, 7, 11] = -1
    with pytest.raises(rs.IndexOutOfRange):
        acc.forward(dense, idx)
    idx[2, 7, 11] = 0               # the handle recovers
    ref, mag, _, _ = orc.forward64(dense, idx)
    check_fp32(acc.forward(dense, idx), ref, mag)
    acc.close()


def test_device_resident_inputs_and_streams_are_identical():
    torch = pytest.importorskip("torch")
    spec = rs.builtin_model("DLRM-RMC2")
    rows = 4000
    acc = rs.Accelerator(spec, rows, seed=2, max_query_size=128)
    dense, idx = rs.fill_query(spec, rows, 4, 0, 100)
    host = acc.forward(dense, idx)
    again = acc.forward(dense, idx)
    assert np.array_equal(host, again)                     # run-to-run bitwise
    d_dense = torch.from_numpy(dense).cuda()
    d_idx = torch.from_numpy(idx).cuda()
    d_out = torch.empty((100, acc.output_dim), device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for st in (s1, s2):
        o = torch.empty_like(d_out)
        acc.forward_ptr(100, d_dense.data_ptr(), d_idx.data_ptr(), o.data_ptr(),
                        rs.MEM_DEVICE, stream=st.cuda_stream)
        outs.append(o)
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), host)
    acc.close()


def test_service_time_is_measured_and_memoised():
    spec = rs.builtin_model("DLRM-RMC1")
    acc = rs.Accelerator(spec, 10000, seed=2, max_query_size=512)
    t1 = acc.service_time(300)
    assert 0 < t1 < 0.1
    assert acc.service_time(300) == t1
    assert acc.service_time(1) > 0
    acc.close()


def test_cfg3_rmc2_ten_million_rows():
    """BASELINE configs[2]: 32 tables x 10M rows x dim 64 (81.9 GB on one B200);
    parity on a query of 16 items (oracle regenerates the touched rows)."""
    spec = rs.ModelSpec("cfg3-RMC2", dense_fc=rs.LayerStack([256, 128, 64]),
                        predict_fc=rs.LayerStack([512, 128, 1]),
                        embeddings=rs.EmbeddingConfig(32, 80, 64, "Sum"), dense_input_dim=256)
    check_forward(spec, rows=10_000_000, S=16, max_q=64)


def test_forward_many_matches_single_calls_and_auto_graphs():
    """rs_forward_many (pipelined host queue and device path) returns the same
    logits as one-at-a-time rs_forward; AUTO mode runs the tcgen05 graph at
    every size (no FFMA graph captured), within the tf32 tolerance."""
    torch = pytest.importorskip("torch")
    spec = rs.builtin_model("DLRM-RMC3")
    rows = 3000
    acc = rs.Accelerator(spec, rows, seed=8, max_query_size=400, fc_mode=rs.FC_AUTO)
    assert acc.info.fc_layers_tcgen05 > 0
    assert acc.info.kernels_per_forward_small == 0
    orc = Oracle(spec, rows, seed=8)
    sizes = [5, 200, 1, 399, 127, 128]
    qs = [rs.fill_query(spec, rows, 3, i, S) for i, S in enumerate(sizes)]
    singles = [acc.forward(d, i) for d, i in qs]
    for (d, i), out, S in zip(qs, singles, sizes):
        ref, mag, _, _ = orc.forward64(d, i)
        assert_close(out, ref, mag, TF32, f"S={S}")
    # host path through the two-slot queue
    hd = [rs.PinnedBuffer(max(d.nbytes, 16)) for d, _ in qs]
    hi = [rs.PinnedBuffer(i.nbytes) for _, i in qs]
    ho = [rs.PinnedBuffer(S * acc.output_dim * 4) for S in sizes]
    for k, (d, i) in enumerate(qs):
        hd[k].view(np.float32, d.shape)[...] = d
        hi[k].view(np.int64, i.shape)[...] = i
    svc = acc.forward_many(sizes, [b.ptr for b in hd], [b.ptr for b in hi], [b.ptr for b in ho],
                           rs.MEM_HOST)
    # FIFO delivery gaps: non-negative (a query finishing under its
    # predecessor on another lane is delivered with it), positive in total
    assert len(svc) == len(sizes) and (svc >= 0).all() and svc.sum() > 0
    for k, S in enumerate(sizes):
        assert np.array_equal(ho[k].view(np.float32, (S, acc.output_dim)), singles[k])
    # device path
    dd = [torch.from_numpy(d).cuda() for d, _ in qs]
    di = [torch.from_numpy(i).cuda() for _, i in qs]
    do = [torch.empty((S, acc.output_dim), device="cuda") for S in sizes]
    acc.forward_many(sizes, [t.data_ptr() for t in dd], [t.data_ptr() for t in di],
                     [t.data_ptr() for t in do], rs.MEM_DEVICE)
    for k in range(len(sizes)):
        assert np.array_equal(do[k].cpu().numpy(), singles[k])
    # a bad index in an asynchronous call is reported by rs_sync, then cleared
    d, i = qs[0]
    bad = i.copy()
    bad[0, 0, 0] = rows + 5
    di_bad = torch.from_numpy(bad).cuda()
    acc.forward_ptr(5, dd[0].data_ptr(), di_bad.data_ptr(), do[0].data_ptr(), rs.MEM_DEVICE)
    with pytest.raises(rs.IndexOutOfRange):
        acc.sync()
    acc.sync()
    acc.close()


@pytest.mark.parametrize("augru", [False, True])
@pytest.mark.parametrize("L", [20, 100])
def test_dien_tensor_core_recurrence(augru, L):
    """The tcgen05 GRU/AUGRU (tf32 gate matmuls, fp32 cell math) against the
    fp64 oracle, zoo DIEN (L=20) and BASELINE configs[4] sequence length 100."""
    spec = rs.ModelSpec(f"dien-L{L}", predict_fc=rs.LayerStack([200, 80, 2]),
                        embeddings=rs.EmbeddingConfig(20, L, 32, "AttentionRNN"),
                        recurrent_hidden_dim=64)
    for S in (5, 200):
        check_forward(spec, rows=50000, S=S, fc_mode=rs.FC_TF32, augru=augru, tol=TF32_TOL,
                      max_q=256)


@pytest.mark.parametrize("desc_memop", ["0", pytest.param("1", marks=needs_experiments)])
def test_forward_many_long_batch_host_runs_ahead(desc_memop, monkeypatch):
    """2000 small queries over 2 lanes: the host enqueues far ahead of the GPU,
    so every query must carry its own descriptor (item count, pointers) by
    value — the event-guarded pinned ring (wraps every 256 queries per lane),
    or stream memory writes."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("RS_DESC_MEMOP", desc_memop)
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 5000
    acc = rs.Accelerator(spec, rows, seed=4, max_query_size=64, fc_mode=rs.FC_FP32,
                         queue_depth=2)
    rng = np.random.default_rng(0)
    sizes = [int(s) for s in rng.integers(1, 65, size=2000)]
    pool = [rs.fill_query(spec, rows, 9, q, 64) for q in range(16)]
    dd = [torch.from_numpy(d).cuda() for d, _ in pool]
    di = [torch.from_numpy(i).cuda() for _, i in pool]
    outs = torch.zeros((len(sizes), 64, acc.output_dim), device="cuda")
    acc.forward_many(sizes, [dd[k % 16].data_ptr() for k in range(len(sizes))],
                     [di[k % 16].data_ptr() for k in range(len(sizes))],
                     [outs[k].data_ptr() for k in range(len(sizes))], rs.MEM_DEVICE)
    got = outs.cpu().numpy()
    singles = {}
    for k, S in enumerate(sizes):
        key = (k % 16, S)
        if key not in singles:
            d, i = pool[k % 16]
            singles[key] = acc.forward(np.ascontiguousarray(d[:S]), np.ascontiguousarray(i[:S]))
        assert np.array_equal(got[k, :S], singles[key]), k
        assert not got[k, S:].any(), k  # nothing written past the query's own rows
    acc.close()


@pytest.mark.parametrize("variant", ["0", pytest.param("1", marks=needs_experiments), "2",
                                     pytest.param("3", marks=needs_experiments),
                                     pytest.param("4", marks=needs_experiments)])
@pytest.mark.parametrize("D,L", [(32, 80), (64, 80), (64, 20), (128, 33), (256, 7)])
def test_sls_kernel_variants_bit_exact(variant, D, L, monkeypatch):
    """Every SLS kernel variant (RS_SLS_VARIANT) reproduces the oracle's
    canonical fp32 order bit for bit."""
    monkeypatch.setenv("RS_SLS_VARIANT", variant)
    spec = rs.ModelSpec(f"sls-v{variant}-D{D}", dense_fc=None, predict_fc=rs.LayerStack([4]),
                        embeddings=rs.EmbeddingConfig(5, L, D, "Sum"), dense_input_dim=0)
    rows = 20011
    acc = rs.Accelerator(spec, rows, seed=2, max_query_size=300)
    orc = Oracle(spec, rows, seed=2)
    for S in (1, 37, 300):
        _, idx = rs.fill_query(spec, rows, 6, S, S)
        assert np.array_equal(acc.pooled(idx), orc.sls_canonical(idx)), (variant, D, L, S)
    acc.close()


@pytest.mark.parametrize("name", ["DLRM-RMC2", "DIN", "WND"])
def test_int32_index_variant_is_bit_identical(name):
    """RS_INDEX_I32 (labelled input-format variant): int32
    indices over the link, widened on the device — the same logits and pooled
    rows as the int64 query, host and device paths, and bad indices still
    reported."""
    torch = pytest.importorskip("torch")
    spec = rs.builtin_model(name)
    rows = 7000
    acc = rs.Accelerator(spec, rows, seed=5, max_query_size=300, fc_mode=rs.FC_AUTO)
    for S in (3, 150, 300):
        dense, idx = rs.fill_query(spec, rows, 8, S, S)
        ref = acc.forward(dense, idx)
        assert np.array_equal(acc.forward(dense, idx.astype(np.int32)), ref)
        assert np.array_equal(acc.pooled(idx.astype(np.int32)), acc.pooled(idx))
        d_dense = torch.from_numpy(dense).cuda()
        d_idx32 = torch.from_numpy(idx.astype(np.int32)).cuda()
        out = torch.empty((S, acc.output_dim), device="cuda")
        acc.forward_ptr(S, d_dense.data_ptr(), d_idx32.data_ptr(), out.data_ptr(), rs.MEM_DEVICE,
                        index_type=rs.INDEX_I32)
        acc.sync()
        assert np.array_equal(out.cpu().numpy(), ref)
        b = acc.batch([S, S], [d_dense.data_ptr()] * 2, [d_idx32.data_ptr()] * 2,
                      [out.data_ptr()] * 2, rs.MEM_DEVICE, index_type=rs.INDEX_I32)
        acc.forward_many(None, prepared=b)
        assert np.array_equal(out.cpu().numpy(), ref)
    dense, idx = rs.fill_query(spec, rows, 8, 1, 4)
    bad = idx.astype(np.int32)
    bad[1, 0, 0] = -1
    with pytest.raises(rs.IndexOutOfRange):
        acc.forward(dense, bad)
    acc.close()


@pytest.mark.parametrize("fc_mode", [rs.FC_FP32, rs.FC_TF32])
@pytest.mark.parametrize("location", [rs.MEM_HOST, rs.MEM_DEVICE])
def test_merged_queries_match_single_calls(fc_mode, location):
    """RS_OPT_MERGE_QUERIES (labelled scheduler extension):
    consecutive queries staged back to back and served by one launch return
    exactly the rows each query gets alone (per-row arithmetic does not depend
    on the row's position in the launch; one FC path per handle here)."""
    torch = pytest.importorskip("torch")
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 4000
    acc = rs.Accelerator(spec, rows, seed=6, max_query_size=400, fc_mode=fc_mode,
                         queue_depth=2)
    acc.set_option(rs.OPT_MERGE_QUERIES, 3)
    sizes = [5, 40, 100, 7, 300, 2, 399, 1]
    qs = [rs.fill_query(spec, rows, 2, k, S) for k, S in enumerate(sizes)]
    singles = [acc.forward(d, i) for d, i in qs]
    if location == rs.MEM_HOST:
        bd = [rs.PinnedBuffer(max(d.nbytes, 16)) for d, _ in qs]
        bi = [rs.PinnedBuffer(i.nbytes) for _, i in qs]
        bo = [rs.PinnedBuffer(S * acc.output_dim * 4) for S in sizes]
        for k, (d, i) in enumerate(qs):
            bd[k].view(np.float32, d.shape)[...] = d
            bi[k].view(np.int64, i.shape)[...] = i
        svc = acc.forward_many(sizes, [b.ptr for b in bd], [b.ptr for b in bi],
                               [b.ptr for b in bo], rs.MEM_HOST)
        got = [bo[k].view(np.float32, (S, acc.output_dim)).copy() for k, S in enumerate(sizes)]
    else:
        dd = [torch.from_numpy(d).cuda() for d, _ in qs]
        di = [torch.from_numpy(i).cuda() for _, i in qs]
        do = [torch.empty((S, acc.output_dim), device="cuda") for S in sizes]
        svc = acc.forward_many(sizes, [t.data_ptr() for t in dd], [t.data_ptr() for t in di],
                               [t.data_ptr() for t in do], rs.MEM_DEVICE)
        got = [t.cpu().numpy() for t in do]
    assert (svc >= 0).all() and svc.sum() > 0
    for k in range(len(sizes)):
        assert np.array_equal(got[k], singles[k]), k
    with pytest.raises(rs.InvalidArgument):
        acc.set_option(rs.OPT_MERGE_QUERIES, 0)
    acc.close()


def test_realtime_serve_matches_single_calls_and_queues():
    """rs_serve (real-time executor, K-server pool): released on the clock,
    routed to the least-loaded replica (two handles on one GPU here), every
    output equals its single-call result; sparse arrivals see ~service-time
    latency, a burst at t=0 sees queueing."""
    torch = pytest.importorskip("torch")
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 3000
    reps = [rs.Accelerator(spec, rows, seed=7, max_query_size=256, queue_depth=2)
            for _ in range(2)]
    sizes = [int(s) for s in np.random.default_rng(1).integers(1, 257, size=40)]
    qs = [rs.fill_query(spec, rows, 4, k, S) for k, S in enumerate(sizes)]
    singles = [reps[0].forward(d, i) for d, i in qs]
    dd = [torch.from_numpy(d).cuda() for d, _ in qs]
    di = [torch.from_numpy(i).cuda() for _, i in qs]
    do = [torch.zeros((S, reps[0].output_dim), device="cuda") for S in sizes]
    b = reps[0].batch(sizes, [t.data_ptr() for t in dd], [t.data_ptr() for t in di],
                      [t.data_ptr() for t in do], rs.MEM_DEVICE)
    sparse = rs.serve(reps, b, np.arange(len(sizes)) * 2e-3)  # one query every 2 ms
    for k in range(len(sizes)):
        assert np.array_equal(do[k].cpu().numpy(), singles[k]), k
    assert (sparse > 0).all() and np.median(sparse) < 2.0
    burst = rs.serve(reps, b, np.zeros(len(sizes)))
    assert burst.max() > np.median(sparse)  # the last of a burst waits behind the rest
    with pytest.raises(rs.InvalidArgument):
        rs.serve(reps, b, np.arange(len(sizes))[::-1] * 1e-3)  # decreasing arrivals
    for r in reps:
        r.close()


def test_packed_host_query_one_transfer():
    """A host query whose indices follow its dense features in one pinned
    buffer is moved with one transfer — same results as separate buffers."""
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 3000
    acc = rs.Accelerator(spec, rows, seed=9, max_query_size=200, fc_mode=rs.FC_AUTO)
    for S in (1, 50, 200):
        dense, idx = rs.fill_query(spec, rows, 3, S, S)
        ref = acc.forward(dense, idx)
        buf = rs.PinnedBuffer(dense.nbytes + idx.nbytes)
        raw = buf.view(np.uint8, (dense.nbytes + idx.nbytes,))
        raw[:dense.nbytes] = dense.reshape(-1).view(np.uint8)
        raw[dense.nbytes:] = idx.reshape(-1).view(np.uint8)
        out = rs.PinnedBuffer(S * acc.output_dim * 4)
        acc.forward_ptr(S, buf.ptr, buf.ptr + dense.nbytes, out.ptr, rs.MEM_HOST, timed=True)
        assert np.array_equal(out.view(np.float32, (S, acc.output_dim)), ref), S
    acc.close()


def test_sls_bandwidth_floor():
    """Performance guard for the dominant kernel: one 1000-item SLS launch at
    the cfg3 row shape (32 tables x 80 lookups x 256-byte rows) moves at least
    5 TB/s of algorithmic bytes (measured 6.3 TB/s)."""
    torch = pytest.importorskip("torch")
    T, L, D, rows, S = 32, 80, 64, 1_000_000, 1000
    spec = rs.ModelSpec("sls-perf", dense_fc=None, predict_fc=rs.LayerStack([4]),
                        embeddings=rs.EmbeddingConfig(T, L, D, "Sum"), dense_input_dim=0)
    acc = rs.Accelerator(spec, rows, seed=1, max_query_size=S)
    _, idx = rs.fill_query(spec, rows, 7, 0, S)
    d_idx = torch.from_numpy(idx).cuda()
    out = torch.empty((S, T * D), device="cuda")
    times = []
    for rep in range(6):
        t = acc.pooled_ptr(S, d_idx.data_ptr(), out.data_ptr(), rs.MEM_DEVICE, timed=True)
        if rep >= 1:
            times.append(t.compute_ms)
    gbs = S * (T * L * (D * 4 + 8) + T * D * 4) / (min(times) * 1e-3) / 1e9
    assert gbs >= 5000, f"SLS {gbs:.0f} GB/s"
    acc.close()


@pytest.mark.parametrize("name", ["WND", "DLRM-RMC1"])
def test_bf16_dense_variant_matches_rounded_fp32(name):
    """RS_DENSE_BF16 (labelled input-format flag): bfloat16 dense
    features over the link, widened on the device — identical to the fp32
    query whose dense features are the same bf16 values; combinable with int32
    indices; packed single-transfer path included."""
    spec = rs.builtin_model(name)
    rows = 4000
    acc = rs.Accelerator(spec, rows, seed=5, max_query_size=200, fc_mode=rs.FC_AUTO)
    for S in (2, 150):
        dense, idx = rs.fill_query(spec, rows, 8, S, S)
        bits = (dense.view(np.uint32) >> 16).astype(np.uint16)  # truncate to bf16
        rounded = (bits.astype(np.uint32) << 16).view(np.float32)
        ref = acc.forward(rounded, idx)
        assert np.array_equal(acc.forward(bits, idx), ref)
        assert np.array_equal(acc.forward(bits, idx.astype(np.int32)), ref)
        buf = rs.PinnedBuffer(bits.nbytes + idx.nbytes)
        raw = buf.view(np.uint8, (bits.nbytes + idx.nbytes,))
        raw[:bits.nbytes] = bits.reshape(-1).view(np.uint8)
        raw[bits.nbytes:] = idx.reshape(-1).view(np.uint8)
        out = rs.PinnedBuffer(S * acc.output_dim * 4)
        acc.forward_ptr(S, buf.ptr, buf.ptr + bits.nbytes, out.ptr, rs.MEM_HOST, timed=True,
                        index_type=rs.DENSE_BF16)
        assert np.array_equal(out.view(np.float32, (S, acc.output_dim)), ref)
    acc.close()


@needs_experiments
@pytest.mark.parametrize("name", ["DLRM-RMC1", "DIN", "NCF"])
def test_fc_chain_kernel_parity(name, monkeypatch):
    """The whole-stack tcgen05 kernel (RS_FC_CHAIN=1, off by default — measured
    slower): activations kept in shared memory between layers, streamed
    layer-0 input (DIN's 640-wide), fused narrow output; tf32 tolerance."""
    monkeypatch.setenv("RS_FC_CHAIN", "1")
    spec = rs.builtin_model(name)
    for S in (1, 130, 300):
        check_forward(spec, rows=3000, S=S, fc_mode=rs.FC_TF32, tol=TF32_TOL, max_q=300)


def test_queue_edge_cases():
    """16 lanes; merged groups of int32 queries (host and device); a bad index
    inside rs_forward_many and inside rs_serve is reported after the call and
    the handle keeps serving."""
    torch = pytest.importorskip("torch")
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 3000
    acc = rs.Accelerator(spec, rows, seed=3, max_query_size=300, fc_mode=rs.FC_FP32,
                         queue_depth=16)
    sizes = [7, 33, 120, 5, 64, 200, 1, 90] * 3
    qs = [rs.fill_query(spec, rows, 1, k, S) for k, S in enumerate(sizes)]
    singles = [acc.forward(d, i) for d, i in qs]
    for merge in (1, 3):
        acc.set_option(rs.OPT_MERGE_QUERIES, merge)
        for loc in (rs.MEM_HOST, rs.MEM_DEVICE):
            if loc == rs.MEM_HOST:
                bd = [rs.PinnedBuffer(max(d.nbytes, 16)) for d, _ in qs]
                bi = [rs.PinnedBuffer(i.nbytes // 2) for _, i in qs]
                for k, (d, i) in enumerate(qs):
                    bd[k].view(np.float32, d.shape)[...] = d
                    bi[k].view(np.int32, i.shape)[...] = i.astype(np.int32)
                outs = [rs.PinnedBuffer(S * acc.output_dim * 4) for S in sizes]
                b = acc.batch(sizes, [x.ptr for x in bd], [x.ptr for x in bi],
                              [o.ptr for o in outs], loc, index_type=rs.INDEX_I32)
                acc.forward_many(None, prepared=b)
                got = [outs[k].view(np.float32, (S, acc.output_dim)) for k, S in
                       enumerate(sizes)]
            else:
                dd = [torch.from_numpy(d).cuda() for d, _ in qs]
                di = [torch.from_numpy(i.astype(np.int32)).cuda() for _, i in qs]
                do = [torch.empty((S, acc.output_dim), device="cuda") for S in sizes]
                b = acc.batch(sizes, [t.data_ptr() for t in dd], [t.data_ptr() for t in di],
                              [t.data_ptr() for t in do], loc, index_type=rs.INDEX_I32)
                acc.forward_many(None, prepared=b)
                got = [t.cpu().numpy() for t in do]
            for k in range(len(sizes)):
                assert np.array_equal(got[k], singles[k]), (merge, loc, k)
    acc.set_option(rs.OPT_MERGE_QUERIES, 1)
    # a bad index in the queue and in the real-time executor
    d, i = qs[2]
    bad = i.copy()
    bad[3, 0, 0] = rows
    dd, dbad = torch.from_numpy(d).cuda(), torch.from_numpy(bad).cuda()
    out = torch.empty((sizes[2], acc.output_dim), device="cuda")
    b = acc.batch([sizes[2]], [dd.data_ptr()], [dbad.data_ptr()], [out.data_ptr()],
                  rs.MEM_DEVICE)
    with pytest.raises(rs.IndexOutOfRange):
        acc.forward_many(None, prepared=b)
    with pytest.raises(rs.IndexOutOfRange):
        rs.serve([acc], b, np.zeros(1))
    assert np.array_equal(acc.forward(d, i), singles[2])
    acc.close()


@needs_experiments
@pytest.mark.parametrize("splits", ["2", "4"])
def test_split_k_parity(splits, monkeypatch):
    """Split-K tcgen05 layers (RS_SPLITK=n, off by default — measured slower):
    the last split to arrive sums the partials in split order, so results are
    deterministic run to run; tf32 tolerance vs the oracle; RMC3's 2560-wide
    bottom layer and MT-WND's 1640-wide stacked layer."""
    monkeypatch.setenv("RS_SPLITK", splits)
    for name in ("DLRM-RMC3", "MT-WND"):
        spec = rs.builtin_model(name)
        for S in (1, 200):
            check_forward(spec, rows=2000, S=S, fc_mode=rs.FC_TF32, tol=TF32_TOL, max_q=300)
    acc = rs.Accelerator(rs.builtin_model("DLRM-RMC3"), 2000, seed=2, max_query_size=300,
                         fc_mode=rs.FC_TF32)
    d, i = rs.fill_query(rs.builtin_model("DLRM-RMC3"), 2000, 4, 0, 257)
    assert np.array_equal(acc.forward(d, i), acc.forward(d, i))
    acc.close()


@pytest.mark.parametrize("name", ["DLRM-RMC1", "DLRM-RMC2"])
def test_l2_hot_block_is_bit_identical(name):
    """l2_persist_mb (SURVEY §8d Zipf/L2-persistence variant): rows [0, R) of
    every table are served from the persisting hot block. Pooled sums stay
    bit-identical to the oracle's canonical order and the logits to the
    accelerator without the block, for Zipf and uniform indices, including
    rows on both sides of the hot boundary."""
    spec = rs.builtin_model(name)
    rows = 50_000
    plain = rs.Accelerator(spec, rows, seed=4, max_query_size=300, fc_mode=rs.FC_AUTO)
    hot = rs.Accelerator(spec, rows, seed=4, max_query_size=300, fc_mode=rs.FC_AUTO,
                         l2_persist_mb=2)
    R = hot.info.hot_rows
    assert 0 < R < rows
    orc = Oracle(spec, rows, seed=4)
    for S, alpha in ((1, 1.05), (130, 1.05), (300, 0.0)):
        dense, idx = rs.fill_query(spec, rows, 9, S, S, zipf_alpha=alpha)
        idx[0, 0, :2] = [R - 1, R]  # both sides of the boundary
        assert np.array_equal(hot.pooled(idx), orc.sls_canonical(idx))
        assert np.array_equal(hot.forward(dense, idx), plain.forward(dense, idx))
        # int32 indices (widened on the device) and the pipelined queue
        assert np.array_equal(hot.forward(dense, idx.astype(np.int32)), plain.forward(dense, idx))
    torch = pytest.importorskip("torch")
    sizes = [7, 300, 64]
    qs = [rs.fill_query(spec, rows, 5, k, S, zipf_alpha=1.05) for k, S in enumerate(sizes)]
    dd = [torch.from_numpy(d).cuda() for d, _ in qs]
    di = [torch.from_numpy(i).cuda() for _, i in qs]
    outs = [torch.empty((S, hot.output_dim), device="cuda") for S in sizes]
    b = hot.batch(sizes, [t.data_ptr() for t in dd], [t.data_ptr() for t in di],
                  [o.data_ptr() for o in outs], rs.MEM_DEVICE)
    hot.forward_many(None, prepared=b)
    for (d, i), o in zip(qs, outs):
        assert np.array_equal(o.cpu().numpy(), plain.forward(d, i))
    # bad index still reported on the hot path
    d, i = rs.fill_query(spec, rows, 5, 9, 4, zipf_alpha=1.05)
    i[2, 1, 3] = rows
    with pytest.raises(rs.IndexOutOfRange):
        hot.forward(d, i)
    hot.close()
    plain.close()


def test_embed_kernel_timing():
    """rs_timing.embed_ms: the embedding kernel alone (event nodes captured
    around it in the pool graph) — positive, inside the graph's own time, and
    0 for a full forward."""
    torch = pytest.importorskip("torch")
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 10_000
    acc = rs.Accelerator(spec, rows, seed=2, max_query_size=256, fc_mode=rs.FC_AUTO)
    d, i = rs.fill_query(spec, rows, 4, 0, 200)
    td, ti = torch.from_numpy(d).cuda(), torch.from_numpy(i).cuda()
    pooled = torch.empty((200, acc.pooled_dim), device="cuda")
    out = torch.empty((200, acc.output_dim), device="cuda")
    for _ in range(3):
        t = acc.pooled_ptr(200, ti.data_ptr(), pooled.data_ptr(), rs.MEM_DEVICE, timed=True)
    assert 0 < t.embed_ms <= t.compute_ms
    f = acc.forward_ptr(200, td.data_ptr(), ti.data_ptr(), out.data_ptr(), rs.MEM_DEVICE,
                        timed=True)
    assert f.embed_ms == 0.0 and f.compute_ms > 0
    acc.close()


def test_service_breakdown_is_a_measured_service_time():
    """rs_service_breakdown: the whole recsim::ServiceTime measured — total,
    transfer (H2D + D2H) and per-category compute summing to total - transfer,
    with the embedding categories carrying the SLS-bound model's time."""
    spec = rs.builtin_model("DLRM-RMC2")
    acc = rs.Accelerator(spec, 200_000, seed=2, max_query_size=512, fc_mode=rs.FC_AUTO)
    b = acc.service_breakdown(300)
    pc = b["per_category"]
    assert 0 < b["transfer"] < b["total"] < 0.1
    assert abs(sum(pc.values()) - (b["total"] - b["transfer"])) <= 1e-9 + 1e-6 * b["total"]
    assert all(v >= 0 for v in pc.values())
    assert pc["EmbeddingLookup"] > pc["DenseFC"] and pc["PredictFC"] > 0
    assert pc["Attention"] == 0 and pc["Recurrent"] == 0
    acc.close()


def test_serve_hybrid_cpu_and_gpu():
    """rs_serve_hybrid: DeepRecSched in real time — queries above T go whole to
    the B200 replica (the tf32 rule of the oracle, bit-identical to rs_forward),
    the rest run as B-item requests on host worker threads (bit-identical to
    the host forward); the offload flags follow the strict S > T rule."""
    spec = rs.builtin_model("DLRM-RMC1")
    rows = 5000
    acc = rs.Accelerator(spec, rows, seed=6, max_query_size=400, fc_mode=rs.FC_AUTO)
    host = rs.HostModel(spec, rows, seed=6)
    orc = Oracle(spec, rows, seed=6)
    sizes = [5, 300, 64, 65, 200, 1, 399, 120]
    T, B = 100, 32
    qs = [rs.fill_query(spec, rows, 2, k, S) for k, S in enumerate(sizes)]
    hb = []
    for d, i in qs:
        b = rs.PinnedBuffer(d.nbytes + i.nbytes)
        raw = b.view(np.uint8, (d.nbytes + i.nbytes,))
        raw[:d.nbytes] = d.reshape(-1).view(np.uint8)
        raw[d.nbytes:] = i.reshape(-1).view(np.uint8)
        hb.append((b, d.nbytes))
    outs = [rs.PinnedBuffer(S * acc.output_dim * 4) for S in sizes]
    batch = acc.batch(sizes, [b.ptr for b, _ in hb], [b.ptr + n for b, n in hb],
                      [o.ptr for o in outs], rs.MEM_HOST)
    lat, off = rs.serve_hybrid(host, 4, B, T, [acc], batch, np.arange(len(sizes)) * 5e-4)
    assert list(off) == [int(S > T) for S in sizes]
    assert (lat > 0).all()
    for k, ((d, i), S) in enumerate(zip(qs, sizes)):
        got = outs[k].view(np.float32, (S, acc.output_dim)).copy()
        ref, mag, _, _ = orc.forward64(d, i)
        if off[k]:
            assert_close(got, ref, mag, TF32, f"hybrid gpu query {k}")
            assert np.array_equal(got, acc.forward(d, i))
        else:
            assert_close(got, ref, mag, FP32, f"hybrid cpu query {k}")
            assert np.array_equal(got, host.forward(d, i))
    host.close()
    acc.close()
