"""The CPU side of the split. Host-core SparseLengthsSum:
bit-identical to the oracle's canonical order (oracle/forward.c
or_sls_canonical) on CPU, and to the B200 kernel's pooled output on the GPU.
Host FC: the fp32 tolerance rule of DESIGN.md §4 against an fp64 product."""
import numpy as np
import pytest

import paper_2001_02772_b200 as rs
from oracle import Oracle, table_value


def sum_spec(T, L, D):
    return rs.ModelSpec(name=f"sum-T{T}-L{L}-D{D}", dense_fc=None,
                        predict_fc=rs.LayerStack([4, 1]), num_parallel_predict_stacks=1,
                        embeddings=rs.EmbeddingConfig(T, L, D, "Sum"), dense_input_dim=0,
                        recurrent_hidden_dim=None)


def tables_of(seed, T, rows, D):
    """The oracle's table spec materialised on the host."""
    tab = np.empty((T, rows, D), dtype=np.float32)
    for t in range(T):
        for r in range(rows):
            for c in range(D):
                tab[t, r, c] = table_value(seed, t, r, c, D)
    return tab


@pytest.mark.parametrize("D", [8, 16, 32, 64, 128, 256, 24])
@pytest.mark.parametrize("L", [1, 37, 80])
def test_host_sls_matches_canonical_oracle(D, L):
    T, rows, seed, S = 3, 61, 5, 4
    spec = sum_spec(T, L, D)
    o = Oracle(spec, rows, seed=seed)
    _, idx = o.fill_query(query_id=3, size=S)
    tab = tables_of(seed, T, rows, D)
    for threads in (1, 5):
        got = rs.host_sls(tab, idx, threads=threads)
        assert np.array_equal(got.view(np.uint32), o.sls_canonical(idx).view(np.uint32))


def test_host_sls_edges():
    tab = np.ones((2, 10, 8), dtype=np.float32)
    assert rs.host_sls(tab, np.zeros((0, 2, 3), dtype=np.int64)).shape == (0, 16)
    assert np.array_equal(rs.host_sls(tab, np.zeros((2, 2, 0), dtype=np.int64)),
                          np.zeros((2, 16), dtype=np.float32))     # empty bags pool to 0
    idx = np.full((3, 2, 4), 9, dtype=np.int64)
    assert np.array_equal(rs.host_sls(tab, idx, threads=64), np.full((3, 16), 4.0, np.float32))
    idx[2, 1, 3] = 10                                                # one past the end
    with pytest.raises(rs.IndexOutOfRange, match="item 2, table 1, lookup 3"):
        rs.host_sls(tab, idx)
    idx[2, 1, 3] = -1
    with pytest.raises(rs.IndexOutOfRange):
        rs.host_sls(tab, idx)
    with pytest.raises(rs.InvalidArgument):
        rs.host_sls(tab, np.zeros((1, 3, 2), dtype=np.int64))     # table count mismatch


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["DLRM-RMC1", "DLRM-RMC3", "NCF"])
def test_host_sls_matches_b200_pooled(name):
    """A query split between host cores and the B200 pools identically."""
    spec = rs.builtin_model(name)
    e = spec.embeddings
    rows, seed = 3000, 4
    acc = rs.Accelerator(spec, rows, seed=seed, device=0, max_query_size=32)
    try:
        _, idx = rs.fill_query(spec, rows, seed=seed, query_id=1, size=17)
        dev = acc.pooled(idx)
        tab = tables_of(seed, e.num_tables, rows, e.embedding_dim)
        assert np.array_equal(rs.host_sls(tab, idx).view(np.uint32), dev.view(np.uint32))
    finally:
        acc.close()


# ---- host FC (the GEMM half of §8f-4) --------------------------------------
@pytest.mark.parametrize("M,K,N", [(1, 13, 512), (7, 64, 1), (33, 256, 128), (5, 0, 8),
                                   (130, 1024, 67)])
@pytest.mark.parametrize("relu", [True, False])
def test_host_fc_matches_fp64(M, K, N, relu):
    """DESIGN.md §4 fp32 tolerance rule: |y - ref| / mag <= 1e-5, with mag the
    absolute-value forward (|b| + |x| @ |W|^T)."""
    rng = np.random.default_rng(M * 1000 + K + N)
    x = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    w = (rng.uniform(-1, 1, (N, K)) / np.sqrt(max(K, 1))).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    ref = x.astype(np.float64) @ w.T.astype(np.float64) + b
    mag = np.abs(x.astype(np.float64)) @ np.abs(w.T.astype(np.float64)) + np.abs(b) + 1e-30
    if relu:
        ref = np.maximum(ref, 0)
    for threads in (1, 3):
        y = rs.host_fc(x, w, b, relu=relu, threads=threads)
        assert y.shape == (M, N) and y.dtype == np.float32
        assert np.max(np.abs(y - ref) / mag, initial=0) <= 1e-5
        if relu:
            assert np.all(y >= 0)


def test_host_fc_edges():
    x = np.ones((3, 4), np.float32)
    w = np.ones((2, 4), np.float32)
    assert np.array_equal(rs.host_fc(x, w, None, relu=False), np.full((3, 2), 4, np.float32))
    assert rs.host_fc(np.zeros((0, 4), np.float32), w).shape == (0, 2)
    with pytest.raises(rs.InvalidArgument):
        rs.host_fc(x, np.ones((2, 5), np.float32))
    with pytest.raises(rs.InvalidArgument):
        rs.host_fc(x, w, np.ones(3, np.float32))


def test_host_fc_takes_device_layout_padded_weights():
    """the device keeps weights [out][round4(in)] zero-padded; an
    in % 4 != 0 layer (RMC1's 13-input bottom layer) passes them as is with
    ldw = round4(in) and gives the same y as the unpadded weight."""
    rng = np.random.default_rng(5)
    M, K, N = 9, 13, 24
    x = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    w = rng.uniform(-0.3, 0.3, (N, K)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    padded = np.zeros((N, 16), np.float32)
    padded[:, :K] = w
    padded[:, K:] = 7.0  # the pad columns must never be read
    y = rs.host_fc(x, padded, b, relu=True, in_dim=K)
    assert np.array_equal(y, rs.host_fc(x, w, b, relu=True))
    with pytest.raises(rs.InvalidArgument):
        rs.host_fc(x, np.ones((N, 12), np.float32), b, in_dim=K)  # ldw < in
