"""ORACLE — TEST INFRASTRUCTURE ONLY: the CPU side of DeepRecSched, run for real
on this host's cores, as bench.py's reference arm and cpu_baseline.

What is timed: the oracle's fp32 forward (oracle/forward.c `or_forward32`, the
same operator order as the accelerator path) on REQUESTS of b items — the unit
the reference's scheduler hands a CPU core (proj/src/sim.cpp:184-188: a query
of S items becomes floor(S/B) requests of B items plus one of S mod B). Every
request size is timed with one core busy and with all C cores busy at once
(`or_time_requests`), over tables materialised at the benchmark's full row
count (DRAM-resident gathers, as on the accelerator).

How QPS@p95 is obtained: those measured times replace the reference's modeled
`cpu_service_time` (proj/src/platform.cpp:71-97) through a link-time wrap
(oracle/ref_cpu_adapter.cpp -> oracle/_ref/librecsim_ref_cpu.so), and the
UNMODIFIED reference then runs DeepRecSched CPU-only: `tune()` phase 1
(proj/src/autotune.cpp:90-152) climbs the batch-size ladder, each rung scored
by `max_qps_under_sla` (proj/src/sim.cpp:246-290: the C-core FIFO simulation
with the split rule, exact p95, geometric lambda bisection to 1%) on
`gen_trace` streams of n queries. The same methodology as the GPU arm: measured
service times replayed by the reference's open-loop rule.

Nothing here imports the product package (paper_2001_02772_b200).
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from . import OrModel, lib, _HERE

P = C.POINTER

ref_cpu = None
_p = os.path.join(_HERE, "_ref", "librecsim_ref_cpu.so")
if os.path.exists(_p):
    ref_cpu = C.CDLL(_p)
    ref_cpu.ref_cpu_set_table.argtypes = [C.c_int, P(C.c_int64), P(C.c_double), P(C.c_double),
                                          C.c_int64]
    ref_cpu.ref_tune.argtypes = [
        P(OrModel), C.c_char_p, C.c_char_p, C.c_double, C.c_uint64, C.c_int, C.c_double,
        C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int,
        P(C.c_int64), P(C.c_int64), P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_int64)]
    ref_cpu.ref_max_qps_accel.argtypes = [
        P(OrModel), C.c_char_p, C.c_char_p, C.c_double, C.c_uint64, C.c_int, C.c_double,
        C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
        P(C.c_double), P(C.c_double), P(C.c_double)]
    ref_cpu.ref_builtin_model.argtypes = [C.c_char_p, P(OrModel)]
    ref_cpu.ref_sla_target.argtypes = [C.c_char_p, C.c_char_p, P(C.c_double)]
    ref_cpu.ref_gen_trace.argtypes = [C.c_uint64, C.c_double, C.c_int, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_int64, C.c_int64,
                                      P(C.c_double), P(C.c_int64)]

if lib is not None:
    lib.or_time_requests.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_uint64,
                                     P(C.c_double)]

LOGNORMAL = 2  # recsim::SizeDistribution::Kind::LogNormal (loadgen.hpp:23-45)

# request sizes timed: a power-of-two ladder plus the largest query (the
# reference's tune() ladder is 1..1024, proj/src/autotune.cpp:101)
REQUEST_SIZES = (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1000)


def available() -> bool:
    return lib is not None and ref_cpu is not None


def builtin_model(name: str) -> OrModel:
    """The reference's own zoo shape (proj/src/model_zoo.cpp:141-170)."""
    m = OrModel()
    if ref_cpu.ref_builtin_model(name.encode(), C.byref(m)):
        raise ValueError(f"unknown model {name}")
    return m


def sla_target(name: str, level: str = "medium") -> float:
    v = C.c_double()
    if ref_cpu.ref_sla_target(name.encode(), level.encode(), C.byref(v)):
        raise ValueError(f"no SLA for {name}")
    return v.value


def gen_trace_sizes(seed: int, mu: float, sigma: float, n: int, max_size: int = 1000):
    arr = np.empty(n, dtype=np.float64)
    sz = np.empty(n, dtype=np.int64)
    rc = ref_cpu.ref_gen_trace(seed, 1000.0, LOGNORMAL, mu, sigma, 0.0, 0.0, max_size, n,
                               arr.ctypes.data_as(P(C.c_double)), sz.ctypes.data_as(P(C.c_int64)))
    if rc:
        raise RuntimeError(f"ref_gen_trace rc={rc}")
    return sz


class CpuDeepRecSched:
    """Materialised oracle model + measured request-time table + the
    reference's CPU-only DeepRecSched on it."""

    def __init__(self, model: OrModel, rows: int, threads: int = 0, seed: int = 1):
        if not available():
            raise ImportError("oracle/liboracle.so or oracle/_ref/librecsim_ref_cpu.so missing")
        self.model = model
        self.rows = rows
        self.threads = threads or (os.cpu_count() or 1)
        t0 = time.time()
        self.h = lib.or_create(C.byref(model), rows, seed, 0, 1)
        if not self.h:
            raise MemoryError("or_create (materialised tables) failed")
        self.fill_s = time.time() - t0
        self.samples = {b: ([], []) for b in REQUEST_SIZES}
        self._round = 0

    def close(self):
        if getattr(self, "h", None):
            lib.or_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _time(self, b: int, threads: int, per_thread: int) -> np.ndarray:
        t = np.zeros(threads * per_thread)
        self._round += 1
        rc = lib.or_time_requests(self.h, b, threads, per_thread, 1000 + self._round,
                                  t.ctypes.data_as(P(C.c_double)))
        if rc:
            raise RuntimeError(f"or_time_requests rc={rc}")
        return t

    def sample(self, budget_s: float) -> float:
        """One bounded sample: every request size once on one core and once on
        all cores; returns the wall seconds spent."""
        t0 = time.time()
        per_size = budget_s / len(REQUEST_SIZES)
        for b in REQUEST_SIZES:
            one = self._time(b, 1, 1)
            per_thread = max(1, min(4, int(per_size / 2 / max(one[0], 1e-6))))
            allc = self._time(b, self.threads, per_thread)
            self.samples[b][0].extend(one.tolist())
            self.samples[b][1].extend(allc.tolist())
        return time.time() - t0

    def table(self):
        bs = np.array(REQUEST_SIZES, dtype=np.int64)
        t1 = np.array([np.median(self.samples[b][0]) for b in REQUEST_SIZES])
        tc = np.array([np.median(self.samples[b][1]) for b in REQUEST_SIZES])
        return bs, t1, tc

    def install(self, lib_=None):
        """Put the measured table into `lib_` (default: librecsim_ref_cpu.so;
        any reference build that links oracle/ref_cpu_adapter.cpp)."""
        bs, t1, tc = self.table()
        lib_ = lib_ or ref_cpu
        lib_.ref_cpu_set_table.argtypes = ref_cpu.ref_cpu_set_table.argtypes
        rc = lib_.ref_cpu_set_table(len(bs), bs.ctypes.data_as(P(C.c_int64)),
                                       t1.ctypes.data_as(P(C.c_double)),
                                       tc.ctypes.data_as(P(C.c_double)), self.threads)
        if rc:
            raise RuntimeError("ref_cpu_set_table failed")

    def tune(self, sla: float, mu: float, sigma: float, n: int = 50_000, seed: int = 42,
             max_size: int = 1000, kind: int = 2) -> dict:
        """Reference tune() CPU-only on the measured table: (B, QPS@p95).
        kind/mu/sigma: the SizeDistribution (LogNormal(mu, sigma), or kind 0 =
        Fixed(mu))."""
        self.install()
        b, t, steps = C.c_int64(), C.c_int64(), C.c_int64()
        q, p, f = C.c_double(), C.c_double(), C.c_double()
        rc = ref_cpu.ref_tune(C.byref(self.model), b"measured", b"", sla, seed, kind, mu,
                              sigma, 0.0, 0.0, max_size, n, 1, C.byref(b), C.byref(t),
                              C.byref(q), C.byref(p), C.byref(f), C.byref(steps))
        if rc == -5:  # recsim::InfeasibleSLA: no batch size meets the SLA on these cores
            return {"batch": None, "qps": 0.0, "p95_s": None, "search_steps": None,
                    "infeasible": "reference tune(): no CPU batch size meets the SLA "
                                  "(InfeasibleSLA, autotune.cpp)"}
        if rc:
            raise RuntimeError(f"ref_tune rc={rc}")
        return {"batch": b.value, "qps": q.value, "p95_s": p.value, "search_steps": steps.value}

    def max_qps(self, sla: float, mu: float, sigma: float, batch: int, n: int = 50_000,
                seed: int = 42, max_size: int = 1000) -> dict:
        """Reference max_qps_under_sla, CPU-only, fixed batch size."""
        self.install()
        q, p, f = C.c_double(), C.c_double(), C.c_double()
        rc = ref_cpu.ref_max_qps_accel(C.byref(self.model), b"measured", b"default", sla, seed,
                                       LOGNORMAL, mu, sigma, 0.0, 0.0, max_size, n, batch, 0,
                                       C.byref(q), C.byref(p), C.byref(f))
        if rc:
            raise RuntimeError(f"ref_max_qps_accel rc={rc}")
        return {"batch": batch, "qps": q.value, "p95_s": p.value}


def make_model(name: str, predict_fc, T: int, L: int, D: int, pooling: int, dense_in: int = 0,
               dense_fc=None, stacks: int = 1, hidden: int = 0) -> OrModel:
    """An inline ModelSpec (model_zoo.hpp:20-65) as the oracle's C struct;
    pooling 0 Sum, 1 Concat, 2 AttentionFC, 3 AttentionRNN."""
    m = OrModel()
    m.name = name.encode()[:31]
    if dense_fc:
        m.has_dense_fc = 1
        m.dense_fc.n = len(dense_fc)
        for i, v in enumerate(dense_fc):
            m.dense_fc.dims[i] = v
    m.predict_fc.n = len(predict_fc)
    for i, v in enumerate(predict_fc):
        m.predict_fc.dims[i] = v
    m.stacks, m.T, m.L, m.D, m.pooling = stacks, T, L, D, pooling
    m.dense_in, m.hidden = dense_in, hidden
    return m
