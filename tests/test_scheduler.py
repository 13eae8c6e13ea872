"""Scheduler interface: split/offload decisions, query streams and the
QPS-under-SLA search. Decision and stream parity are checked against the
compiled, unmodified reference (oracle/_ref) — SURVEY §8c "decision oracle"."""
import ctypes as C
import math
from collections import defaultdict

import numpy as np
import pytest

import paper_2001_02772_b200 as rs
from paper_2001_02772_b200 import SizeDistribution, builtin_model, gen_trace, route


def test_split_known_answers():                                # test_sim.cpp:54-65
    assert route(10, 4, None) == ("cpu", [4, 4, 2])
    assert route(8, 4, None) == ("cpu", [4, 4])
    assert route(3, 4, None) == ("cpu", [3])
    # SURVEY §8a a7 probe, B=64 T=324
    assert route(1, 64, 324) == ("cpu", [1])
    assert route(65, 64, 324) == ("cpu", [64, 1])
    assert route(324, 64, 324) == ("cpu", [64] * 5 + [4])
    assert route(325, 64, 324) == ("accel", [325])
    assert route(1000, 64, 324) == ("accel", [1000])


def test_strict_greater_offload_boundary():                    # test_sim.cpp:125-156
    assert route(25, 16, 25)[0] == "cpu"
    assert route(25, 16, 24)[0] == "accel"
    assert route(25, 16, None)[0] == "cpu"


def test_route_validation():
    with pytest.raises(rs.ConfigError):
        route(10, 0, None)
    with pytest.raises(rs.InvalidArgument):
        route(0, 4, None)


def test_fixed_distribution_and_determinism():                 # test_loadgen.cpp:9-31
    a, s = gen_trace(1, 1000, SizeDistribution.fixed(25), 10)
    assert (s == 25).all() and len(a) == 10 and np.all(np.diff(a) > 0)
    d = SizeDistribution.production_heavy_tail()
    a1, s1 = gen_trace(7, 500, d, 5000)
    a2, s2 = gen_trace(7, 500, d, 5000)
    assert np.array_equal(a1, a2) and np.array_equal(s1, s2)
    a3, _ = gen_trace(8, 500, d, 5000)
    assert not np.array_equal(a1, a3)


def test_sizes_clamped_and_invalid_rejected():                 # test_loadgen.cpp:49-62,117-123
    for d in (SizeDistribution.production_heavy_tail(), SizeDistribution.normal(5, 50),
              SizeDistribution.log_normal(math.log(800), 1.0)):
        _, s = gen_trace(3, 1000, d, 200000)
        assert s.min() >= 1 and s.max() <= d.max_size
    with pytest.raises(rs.InvalidDistribution):
        gen_trace(1, 100, SizeDistribution.log_normal(float("nan"), 1), 10)
    with pytest.raises(rs.InvalidDistribution):
        gen_trace(1, -5, SizeDistribution.fixed(1), 10)


def test_production_stream_statistics():
    # SURVEY §8a a13 probe: mean 412.9, p50 347, 7.2% clamped at 1000 (n=1e5)
    _, s = gen_trace(42, 1000, SizeDistribution.production_heavy_tail(), 100000)
    assert abs(s.mean() - 412.9) < 3
    assert abs(np.median(s) - 347) <= 2
    assert abs((s == 1000).mean() - 0.072) < 0.003


def _ref(orc):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    return orc.ref


DISTS = [SizeDistribution.production_heavy_tail(), SizeDistribution.log_normal(math.log(300), 0.5),
         SizeDistribution.log_normal(math.log(30), 0.5), SizeDistribution.normal(50, 20),
         SizeDistribution.fixed(17)]


@pytest.mark.parametrize("dist", DISTS, ids=lambda d: d.kind)
def test_gen_trace_bit_identical_to_reference(orc, dist):
    ref = _ref(orc)
    n = 20000
    for seed in (42, 42 + 10007, 0x9e3779b9 + 42):
        a, s = gen_trace(seed, 733.0, dist, n)
        ra = np.empty(n)
        rsz = np.empty(n, dtype=np.int64)
        rc = ref.ref_gen_trace(seed, 733.0, dist.KINDS[dist.kind], dist.p0, dist.p1, dist.p2,
                               dist.p3, dist.max_size, n, ra.ctypes.data_as(C.POINTER(C.c_double)),
                               rsz.ctypes.data_as(C.POINTER(C.c_int64)))
        assert rc == 0
        assert np.array_equal(a, ra)      # bit-identical doubles
        assert np.array_equal(s, rsz)


def _ref_decisions(orc, ref, spec, dist, seed, lam, n, batch, thr):
    cap = n * 1100
    k = np.empty(cap, dtype=np.int32)
    q = np.empty(cap, dtype=np.int64)
    it = np.empty(cap, dtype=np.int64)
    cnt = C.c_int64()
    p95 = C.c_double()
    rc = ref.ref_simulate_decisions(
        C.byref(orc.model_to_or(spec)), b"skylake", seed, lam, dist.KINDS[dist.kind], dist.p0,
        dist.p1, dist.p2, dist.p3, dist.max_size, n, batch, thr,
        k.ctypes.data_as(C.POINTER(C.c_int32)), q.ctypes.data_as(C.POINTER(C.c_int64)),
        it.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(cnt), C.byref(p95))
    assert rc == 0 and cnt.value <= cap
    per_query = defaultdict(list)
    for j in range(cnt.value):
        per_query[int(q[j])].append(("accel" if k[j] == 3 else "cpu", int(it[j])))
    return per_query


@pytest.mark.parametrize("model,batch,thr", [("DLRM-RMC1", 64, 324), ("DLRM-RMC1", 1024, 448),
                                             ("WND", 64, 320), ("NCF", 128, 0),
                                             ("DIEN", 8, 1), ("DLRM-RMC3", 25, 0),
                                             ("DIN", 128, 352)])
def test_decisions_identical_to_reference_simulate(orc, model, batch, thr):
    """Every query: same offload decision and same request-size sequence as the
    reference simulate()'s Dispatch/AccelStart events (sim.cpp:173-191)."""
    ref = _ref(orc)
    spec = builtin_model(model)
    dist = SizeDistribution.production_heavy_tail()
    n, seed, lam = 3000, 42, 300.0
    per_query = _ref_decisions(orc, ref, spec, dist, seed, lam, n, batch, thr)
    _, sizes = gen_trace(seed, lam, dist, n)
    offloaded = 0
    for i, S in enumerate(sizes):
        kind, reqs = route(int(S), batch, thr or None)
        got = per_query[i]
        if kind == "accel":
            offloaded += 1
            assert got == [("accel", int(S))], i
        else:
            assert got == [("cpu", r) for r in reqs], i
    if thr and thr > 1:
        assert 0 < offloaded < n


# ---- QPS under SLA over measured service times -------------------------------
def test_qps_deterministic_service_bound():                    # test_sim.cpp:171-190 analogue
    s = 1e-3
    svc = np.full(8000, s)
    ok = rs.qps_under_sla(svc, sla=20 * s)
    assert 0.5 / s < ok.qps < 1.2 / s and ok.p95 <= 20 * s
    bad = rs.qps_under_sla(svc, sla=s / 100)
    assert bad.qps == 0 and bad.at_lambda == 0


def test_qps_mm1_like_tail_and_servers():
    # M/D/1: p95 grows with load; two servers sustain about twice the rate.
    s = 2e-3
    svc = np.full(20000, s)
    one = rs.qps_under_sla(svc, sla=10 * s, servers=1)
    two = rs.qps_under_sla(svc, sla=10 * s, servers=2)
    assert 1.7 < two.qps / one.qps < 2.3
    assert one.evaluations >= 3


def test_qps_rejects_bad_config():
    with pytest.raises(rs.ConfigError):
        rs.qps_under_sla([1e-3] * 10, 1.0, servers=0)
    with pytest.raises(rs.InvalidArgument):
        rs.qps_under_sla([1e-3] * 10, -1.0)
