"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of
  * liboracle.so  — the C restatement of the forward pass (oracle/forward.c),
  * _ref/librecsim_ref.so — the unmodified reference library compiled from
    /root/reference/proj/src plus oracle/ref_shim.cpp (decision/accounting
    oracle; optional: absent when the reference was never built here).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as part of the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
P = C.POINTER


class OrStack(C.Structure):
    _fields_ = [("n", C.c_int32), ("dims", C.c_int64 * 8)]


class OrModel(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("has_dense_fc", C.c_int32), ("dense_fc", OrStack),
                ("predict_fc", OrStack), ("stacks", C.c_int64), ("T", C.c_int64),
                ("L", C.c_int64), ("D", C.c_int64), ("pooling", C.c_int32),
                ("dense_in", C.c_int64), ("hidden", C.c_int64)]


def model_to_or(spec) -> OrModel:
    """From paper_2001_02772_b200.ModelSpec (same field order as rs_model_desc)."""
    m = OrModel()
    m.name = spec.name.encode()[:31]
    if spec.dense_fc is not None:
        m.has_dense_fc = 1
        m.dense_fc.n = len(spec.dense_fc.dims)
        for i, v in enumerate(spec.dense_fc.dims):
            m.dense_fc.dims[i] = v
    m.predict_fc.n = len(spec.predict_fc.dims)
    for i, v in enumerate(spec.predict_fc.dims):
        m.predict_fc.dims[i] = v
    m.stacks = spec.num_parallel_predict_stacks
    e = spec.embeddings
    m.T, m.L, m.D = e.num_tables, e.lookups_per_table, e.embedding_dim
    m.pooling = {"Sum": 0, "Concat": 1, "AttentionFC": 2, "AttentionRNN": 3}[e.pooling]
    m.dense_in = spec.dense_input_dim
    m.hidden = spec.recurrent_hidden_dim or 0
    return m


def _load(path):
    return C.CDLL(path) if os.path.exists(path) else None


lib = _load(os.path.join(_HERE, "liboracle.so"))
ref = _load(os.path.join(_HERE, "_ref", "librecsim_ref.so"))

if lib is not None:
    lib.or_create.restype = C.c_void_p
    lib.or_create.argtypes = [P(OrModel), C.c_int64, C.c_uint64, C.c_int, C.c_int]
    lib.or_destroy.argtypes = [C.c_void_p]
    for f in ("or_predict_input_dim", "or_output_dim", "or_pooled_dim"):
        getattr(lib, f).restype = C.c_int64
        getattr(lib, f).argtypes = [C.c_void_p]
    lib.or_forward64.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p]
    lib.or_forward64_mt.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    lib.or_forward32.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.or_sls_canonical.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    lib.or_table_value.restype = C.c_float
    lib.or_table_value.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
    lib.or_fill_query.argtypes = [P(OrModel), C.c_int64, C.c_uint64, C.c_uint64, C.c_int64,
                                  C.c_void_p, C.c_void_p]
    lib.or_bench_queries.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_uint64,
                                     P(C.c_double)]


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


class Oracle:
    """fp64 forward (with error-scale magnitudes) and the canonical fp32 SLS."""

    def __init__(self, spec, rows: int, seed: int = 1, augru: bool = False,
                 materialize: bool = False):
        if lib is None:
            raise ImportError("oracle/liboracle.so is not built (make -C oracle)")
        self.spec = spec
        self._m = model_to_or(spec)
        self.rows = rows
        self.seed = seed
        self.h = lib.or_create(C.byref(self._m), rows, seed, int(augru), int(materialize))
        if not self.h:
            raise MemoryError("or_create failed")
        self.p_in = lib.or_predict_input_dim(self.h)
        self.out_dim = lib.or_output_dim(self.h)
        self.pooled_dim = lib.or_pooled_dim(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib.or_destroy(self.h)
            self.h = None

    def forward64(self, dense, idx, threads: int = 0):
        """fp64 forward; items are spread over `threads` host threads
        (0 = every core; results do not depend on the thread count)."""
        S = idx.shape[0] if idx.size else dense.shape[0]
        dense = np.ascontiguousarray(dense, dtype=np.float32)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros((S, self.out_dim))
        mag = np.zeros((S, self.out_dim))
        pooled = np.zeros((S, max(self.pooled_dim, 1)))
        pmag = np.zeros((S, max(self.pooled_dim, 1)))
        rc = lib.or_forward64_mt(self.h, S, _ptr(dense), _ptr(idx), out.ctypes.data,
                                 mag.ctypes.data, pooled.ctypes.data, pmag.ctypes.data,
                                 threads or (os.cpu_count() or 1))
        if rc:
            raise RuntimeError(f"or_forward64 rc={rc}")
        return out, mag, pooled[:, :self.pooled_dim], pmag[:, :self.pooled_dim]

    def forward32(self, dense, idx):
        S = idx.shape[0] if idx.size else dense.shape[0]
        dense = np.ascontiguousarray(dense, dtype=np.float32)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros((S, self.out_dim), dtype=np.float32)
        rc = lib.or_forward32(self.h, S, _ptr(dense), _ptr(idx), out.ctypes.data)
        if rc:
            raise RuntimeError(f"or_forward32 rc={rc}")
        return out

    def sls_canonical(self, idx):
        S = idx.shape[0]
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros((S, self.spec.embeddings.num_tables * self.spec.embeddings.embedding_dim),
                       dtype=np.float32)
        rc = lib.or_sls_canonical(self.h, S, idx.ctypes.data, out.ctypes.data)
        if rc:
            raise RuntimeError(f"or_sls_canonical rc={rc}")
        return out

    def fill_query(self, query_id: int, size: int):
        e = self.spec.embeddings
        dense = np.zeros((size, self.spec.dense_input_dim), dtype=np.float32)
        idx = np.zeros((size, e.num_tables, e.lookups_per_table), dtype=np.int64)
        lib.or_fill_query(C.byref(self._m), self.rows, self.seed, query_id, size, _ptr(dense),
                          _ptr(idx))
        return dense, idx

    def bench_queries(self, sizes, threads: int, seed: int = 7) -> float:
        sizes = np.ascontiguousarray(sizes, dtype=np.int64)
        sec = C.c_double()
        rc = lib.or_bench_queries(self.h, len(sizes), sizes.ctypes.data, threads, seed,
                                  C.byref(sec))
        if rc:
            raise RuntimeError(f"or_bench_queries rc={rc}")
        return sec.value


def table_value(seed, t, r, c, D):
    return lib.or_table_value(seed, t, r, c, D)


# ---- the compiled reference (decision / accounting oracle) -----------------
if ref is not None:
    ref.ref_builtin_model.argtypes = [C.c_char_p, P(OrModel)]
    ref.ref_validate.argtypes = [P(OrModel)]
    ref.ref_work.argtypes = [P(OrModel), C.c_int64, P(C.c_double), P(C.c_double),
                             P(C.c_double)]
    ref.ref_accel_input_bytes.argtypes = [P(OrModel), C.c_int64, P(C.c_double)]
    ref.ref_accel_service_time_default.argtypes = [P(OrModel), C.c_int64, P(C.c_double),
                                                   P(C.c_double)]
    ref.ref_sla_target.argtypes = [C.c_char_p, C.c_char_p, P(C.c_double)]
    ref.ref_gen_trace.argtypes = [C.c_uint64, C.c_double, C.c_int, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_int64, C.c_int64,
                                  P(C.c_double), P(C.c_int64)]
    ref.ref_simulate_decisions.argtypes = [
        P(OrModel), C.c_char_p, C.c_uint64, C.c_double, C.c_int, C.c_double, C.c_double,
        C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int64, C.c_int64, P(C.c_int32),
        P(C.c_int64), P(C.c_int64), C.c_int64, P(C.c_int64), P(C.c_double)]
    ref.ref_max_qps.argtypes = [P(OrModel), C.c_char_p, C.c_double, C.c_uint64, C.c_int,
                                C.c_double, C.c_double, C.c_double, C.c_double, C.c_int64,
                                C.c_int64, C.c_int64, C.c_int64, P(C.c_double),
                                P(C.c_double)]


def ref_available() -> bool:
    return ref is not None


# The same reference with accel_service_time wrapped to the B200 path
# (oracle/ref_b200_adapter.cpp). It links the product library,
# so it is loaded only on request (load_ref_b200), never by the CPU arms.
_ACCEL_ARGTYPES = [
    P(OrModel), C.c_char_p, C.c_char_p, C.c_double, C.c_uint64, C.c_int, C.c_double,
    C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
    P(C.c_double), P(C.c_double), P(C.c_double)]
_TUNE_ARGTYPES = [
    P(OrModel), C.c_char_p, C.c_char_p, C.c_double, C.c_uint64, C.c_int, C.c_double,
    C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int,
    P(C.c_int64), P(C.c_int64), P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_int64)]


def _bind_accel(lib_):
    lib_.ref_max_qps_accel.argtypes = _ACCEL_ARGTYPES
    lib_.ref_tune.argtypes = _TUNE_ARGTYPES
    lib_.ref_accel_service_time_named.argtypes = [P(OrModel), C.c_char_p, C.c_int64,
                                                  P(C.c_double), P(C.c_double), P(C.c_double)]


def ref_accel_service_time(lib_, spec, accel: str, S: int):
    """The reference accel_service_time on a named accelerator: (rc, total,
    transfer, per_category[7]); rc = the shim's exception code (0 ok, -1
    std::invalid_argument, -2 UnknownModel, -3 ConfigError, -99 other)."""
    t, x = C.c_double(), C.c_double()
    pc = (C.c_double * 7)()
    rc = lib_.ref_accel_service_time_named(C.byref(model_to_or(spec)), accel.encode(), S,
                                           C.byref(t), C.byref(x), pc)
    return rc, t.value, x.value, list(pc)


if ref is not None:
    _bind_accel(ref)
_ref_b200 = None


def load_ref_b200():
    """oracle/_ref/librecsim_ref_b200.so (reference + B200 adapter), or None."""
    global _ref_b200
    if _ref_b200 is None:
        _ref_b200 = _load(os.path.join(_HERE, "_ref", "librecsim_ref_b200.so"))
        if _ref_b200 is not None:
            _bind_accel(_ref_b200)
    return _ref_b200


def ref_max_qps(lib_, spec, accel: str, cpu: str, sla: float, dist, n: int, batch: int,
                threshold: int, seed: int = 42):
    """Reference max_qps_under_sla with a named accelerator ("default" | "b200")."""
    q, p, f = C.c_double(), C.c_double(), C.c_double()
    rc = lib_.ref_max_qps_accel(C.byref(model_to_or(spec)), cpu.encode(), accel.encode(), sla,
                                seed, dist.KINDS[dist.kind], dist.p0, dist.p1, dist.p2,
                                dist.p3, dist.max_size, n, batch, threshold, C.byref(q),
                                C.byref(p), C.byref(f))
    if rc:
        raise RuntimeError(f"ref_max_qps_accel rc={rc}")
    return q.value, p.value, f.value


def ref_tune(lib_, spec, accel: str, cpu: str, sla: float, dist, n: int, seeds: int = 1,
             seed: int = 42):
    """Reference DeepRecSched tune() (autotune.cpp:90-217); accel "" = CPU only."""
    b, t, steps = C.c_int64(), C.c_int64(), C.c_int64()
    q, p, f = C.c_double(), C.c_double(), C.c_double()
    rc = lib_.ref_tune(C.byref(model_to_or(spec)), cpu.encode(), accel.encode(), sla, seed,
                       dist.KINDS[dist.kind], dist.p0, dist.p1, dist.p2, dist.p3,
                       dist.max_size, n, seeds, C.byref(b), C.byref(t), C.byref(q),
                       C.byref(p), C.byref(f), C.byref(steps))
    if rc:
        raise RuntimeError(f"ref_tune rc={rc}")
    return {"batch": b.value, "threshold": t.value, "qps": q.value, "p95": p.value,
            "accel_work_fraction": f.value, "search_steps": steps.value}
