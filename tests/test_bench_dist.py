"""bench.py's multi-GPU plumbing on CPU (gloo, world_size 2): independent replica
streams per rank, slowest-rank timing, whole-job aggregation — the same
functions bench.py calls under torchrun/NCCL. There is no data-path collective
(SURVEY §8e): replicas serve independent query streams."""
import os
import socket

import pytest

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        qps = 1000.0 + 100.0 * rank          # rank 0 is the slowest replica
        t = 2.0 - 0.5 * rank                 # rank 0 takes longest
        agg = bench.aggregate(qps, t, queries=500 + rank, world=world)
        q.put((rank, agg, bench.rank_seed(rank)))
    finally:
        dist.destroy_process_group()


def test_two_rank_aggregation_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict((r, (a, s)) for r, a, s in (q.get() for _ in range(2)))
    for r in (0, 1):
        agg, _ = res[r]
        assert agg["time_s"] == pytest.approx(2.0)            # max over ranks
        assert agg["value"] == pytest.approx(2 * 1000.0)      # N x min rank QPS
        assert agg["saturated_qps"] == pytest.approx(1001 / 2.0)
    assert res[0][1] != res[1][1]                             # independent streams
    assert res[0][1] == 42 and res[1][1] == 42 + 10007         # autotune.cpp:23 seeds


def test_single_process_aggregation_is_identity():
    agg = bench.aggregate(123.0, 0.5, queries=10, world=1)
    assert agg == {"time_s": 0.5, "value": 123.0, "saturated_qps": 20.0}


@pytest.mark.parametrize("workload", ["cfg3-rmc2", "cfg3-rmc3", "cfg1-rmc1", "cfg5-dien",
                                      "cfg5-din", "mt-wnd", "ncf"])
def test_reference_arm_config_equals_ours(workload):
    """The driver compares the two arms' `config` objects: the reference arm
    builds its workload from the compiled reference's zoo (no product import),
    ours from the product's mirror — same shapes, sizes, SLA, hence the same
    config dict."""
    import argparse
    import math
    import numpy as np
    import bench
    import paper_2001_02772_b200 as rs
    from oracle import cpu_arm
    if not cpu_arm.available():
        pytest.skip("oracle/_ref not built")
    args = argparse.Namespace(workload=workload, queries_per_step=256, steps=20, index_bits=64,
                              dense_bits=32, size_median=300.0, max_query=1000, fc="auto",
                              merge=1, zipf=0.0, l2_persist_mb=0, size_fixed=0, rnn="gru",
                              sla=0.0)
    spec, rows, zoo = bench.workload_spec(rs, workload)
    _, sizes = rs.gen_trace(bench.rank_seed(0), 1000.0,
                            rs.SizeDistribution.log_normal(math.log(300.0), 0.5), 512)
    e = spec.embeddings
    ours = bench.make_config(args, spec.name, (e.num_tables, e.lookups_per_table,
                                               e.embedding_dim, spec.dense_input_dim),
                             rows, np.minimum(sizes, 1000), 1,
                             bench.sla_for(args, zoo, rs.sla_target))
    m, rows2, zoo2 = bench.workload_or_model(workload)
    sizes2 = cpu_arm.gen_trace_sizes(bench.rank_seed(0), math.log(300.0), 0.5, 512, 1000)
    theirs = bench.make_config(args, m.name.decode(), (m.T, m.L, m.D, m.dense_in), rows2,
                               np.minimum(sizes2, 1000), 1,
                               bench.sla_for(args, zoo2, cpu_arm.sla_target))
    assert ours == theirs


def test_cta_pairs_only_for_uniform_queues():
    """RS_OPT_CTA_PAIRS is measured faster for uniform-size queues and slower
    in mixed streams: bench turns it on for --size-fixed only
    unless told otherwise, and the config records the choice."""
    import argparse
    ns = lambda **k: argparse.Namespace(**{"cta_pairs": "auto", "size_fixed": 0, **k})
    assert bench.cta_pairs_on(ns()) is False
    assert bench.cta_pairs_on(ns(size_fixed=1024)) is True
    assert bench.cta_pairs_on(ns(size_fixed=1024, cta_pairs="off")) is False
    assert bench.cta_pairs_on(ns(cta_pairs="on")) is True
    # namespaces without the flag (e.g. the reference arm's) read as auto
    assert bench.cta_pairs_on(argparse.Namespace(size_fixed=0)) is False
