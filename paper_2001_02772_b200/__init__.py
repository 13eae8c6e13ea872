"""paper_2001_02772_b200 — B200-native accelerator path for DeepRecSched.

Python mirror of the reference's operator and scheduler interface
(``recsim::ModelSpec``, ``work``, ``accel_input_bytes``, ``gen_trace``, the
offload/split rule of ``simulate``) over the C-ABI in ``include/rs_accel.h``.
Every compute call goes through ``librecsys_b200.so`` (sm_100a kernels); there
is no CPU fallback: if the library is missing, importing this package raises.

Reference citations are ``path:line`` under ``/root/reference/proj``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

# rs_forward_many's lanes, copy stream and graph branches need more than the
# default 8 hardware work queues or unrelated lanes serialise;
# effective when this package is imported before the CUDA context is created.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

_HERE = os.path.dirname(os.path.abspath(__file__))
# RS_LIB_VARIANT=exp loads the experiments build (make EXPERIMENTS=1 OUT=
# ../librecsys_b200_exp.so): the measured-slower alternatives, for tools only.
LIB_PATH = os.path.join(_HERE, "librecsys_b200_exp.so" if os.environ.get("RS_LIB_VARIANT") == "exp"
                        else "librecsys_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the accelerator path)")
_lib = C.CDLL(LIB_PATH)

# ---- error mapping (mirrors the reference's exception types) ---------------
RS_OK = 0


class RecsimError(RuntimeError):
    code = -99


class InvalidArgument(ValueError):           # std::invalid_argument
    code = -1


class UnknownModel(RecsimError):            # model_zoo.hpp:15-18
    code = -2


class ConfigError(RecsimError):             # sim.hpp:15-17
    code = -3


class InvalidDistribution(RecsimError):     # loadgen.hpp:12-14
    code = -4


class CudaError(RecsimError):
    code = -5


class OutOfMemory(RecsimError):
    code = -6


class IndexOutOfRange(RecsimError):
    code = -7


class NoDevice(RecsimError):
    code = -8


class CapacityError(RecsimError):
    code = -9


class EmptyResult(RecsimError):             # sim.hpp:19-21
    code = -10


_ERRORS = {c.code: c for c in (InvalidArgument, UnknownModel, ConfigError, InvalidDistribution,
                               CudaError, OutOfMemory, IndexOutOfRange, NoDevice,
                               CapacityError, EmptyResult)}


def _check(rc: int) -> None:
    if rc != RS_OK:
        msg = _lib.rs_last_error().decode()
        raise _ERRORS.get(rc, RecsimError)(msg)


# ---- C structs (include/rs_accel.h) ----------------------------------------
MAX_LAYERS = 8
NUM_OP_CATEGORIES = 7
POOLING = {"Sum": 0, "Concat": 1, "AttentionFC": 2, "AttentionRNN": 3}
POOLING_NAMES = {v: k for k, v in POOLING.items()}
OP_CATEGORIES = ["DenseFC", "PredictFC", "EmbeddingLookup", "Pooling", "Attention",
                 "Recurrent", "Interaction"]
FC_FP32, FC_TF32, FC_AUTO, FC_BF16 = 0, 1, 2, 3  # FC_BF16: labelled bf16 tcgen05 variant
RNN_GRU, RNN_AUGRU = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1
INDEX_I64, INDEX_I32 = 0, 1  # rs_query.index_type (I32: labelled input variant)
DENSE_BF16 = 2               # rs_query.index_type flag: bf16 dense (labelled variant)
OPT_MERGE_QUERIES = 1        # rs_accel_set_option (labelled scheduler extension)
OPT_STAGE_TIMING = 2         # rs_accel_set_option: per-stage event timing of rs_forward
OPT_CTA_PAIRS = 3            # rs_accel_set_option: CTA-pair FC tiles for uniform-size queues


class CLayerStack(C.Structure):
    _fields_ = [("n", C.c_int32), ("dims", C.c_int64 * MAX_LAYERS)]


class CModelDesc(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("has_dense_fc", C.c_int32),
                ("dense_fc", CLayerStack), ("predict_fc", CLayerStack),
                ("num_parallel_predict_stacks", C.c_int64), ("num_tables", C.c_int64),
                ("lookups_per_table", C.c_int64), ("embedding_dim", C.c_int64),
                ("pooling", C.c_int32), ("dense_input_dim", C.c_int64),
                ("recurrent_hidden_dim", C.c_int64)]


class CWork(C.Structure):
    _fields_ = [("flops", C.c_double * NUM_OP_CATEGORIES),
                ("bytes", C.c_double * NUM_OP_CATEGORIES), ("gather_stream", C.c_double)]


class CSizeDist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("p0", C.c_double), ("p1", C.c_double),
                ("p2", C.c_double), ("p3", C.c_double), ("max_size", C.c_int64)]


class CQpsResult(C.Structure):
    _fields_ = [("qps", C.c_double), ("at_lambda", C.c_double), ("p95", C.c_double),
                ("p50", C.c_double), ("evaluations", C.c_int32)]


class CInitDesc(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("rows_per_table", C.c_int64),
                ("max_query_size", C.c_int64), ("fc_mode", C.c_int32),
                ("rnn_cell", C.c_int32), ("l2_persist_mb", C.c_int32),
                ("queue_depth", C.c_int32)]


class CQuery(C.Structure):
    _fields_ = [("size", C.c_int64), ("dense", C.c_void_p), ("indices", C.c_void_p),
                ("location", C.c_int32), ("index_type", C.c_int32)]


class CTiming(C.Structure):
    _fields_ = [("h2d_ms", C.c_double), ("compute_ms", C.c_double), ("d2h_ms", C.c_double),
                ("total_ms", C.c_double), ("embed_ms", C.c_double), ("fc_ms", C.c_double)]


class CAccelInfo(C.Structure):
    _fields_ = [("device", C.c_int32), ("sm_count", C.c_int32),
                ("kernels_per_forward", C.c_int32), ("kernels_per_forward_small", C.c_int32),
                ("fc_layers_tcgen05", C.c_int32),
                ("predict_input_dim", C.c_int64), ("output_dim", C.c_int64),
                ("pooled_dim", C.c_int64), ("table_bytes", C.c_int64),
                ("weight_bytes", C.c_int64), ("l2_bytes", C.c_int64),
                ("hot_rows", C.c_int64)]


def _sig(name, restype, *argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


P = C.POINTER
_sig("rs_last_error", C.c_char_p)
_sig("rs_abi_version", C.c_int)
_sig("rs_model_builtin", C.c_int, C.c_char_p, P(CModelDesc))
_sig("rs_zoo_names", C.c_int, P(C.c_char_p), C.c_int, P(C.c_int))
_sig("rs_model_validate", C.c_int, P(CModelDesc))
_sig("rs_work", C.c_int, P(CModelDesc), C.c_int64, P(CWork))
_sig("rs_predict_input_dim", C.c_int, P(CModelDesc), P(C.c_int64))
_sig("rs_accel_input_bytes", C.c_int, P(CModelDesc), C.c_int64, P(C.c_double))
_sig("rs_sla_target", C.c_int, C.c_char_p, C.c_char_p, P(C.c_double))
_sig("rs_route", C.c_int, C.c_int64, C.c_int64, C.c_int64, P(C.c_int32), P(C.c_int64),
     C.c_int64, P(C.c_int64))
_sig("rs_dist_production", C.c_int, P(CSizeDist))
_sig("rs_gen_trace", C.c_int, C.c_uint64, C.c_double, P(CSizeDist), C.c_int64,
     P(C.c_double), P(C.c_int64))
_sig("rs_qps_under_sla", C.c_int, P(C.c_double), P(C.c_double), C.c_int64, C.c_int32,
     C.c_double, C.c_double, C.c_uint64, C.c_double, P(CQpsResult))
_sig("rs_accel_create", C.c_int, P(CModelDesc), P(CInitDesc), C.c_int, P(C.c_void_p))
_sig("rs_accel_destroy", C.c_int, C.c_void_p)
_sig("rs_accel_info_get", C.c_int, C.c_void_p, P(CAccelInfo))
_sig("rs_forward", C.c_int, C.c_void_p, P(CQuery), C.c_void_p, C.c_void_p, P(CTiming))
_sig("rs_pooled", C.c_int, C.c_void_p, P(CQuery), C.c_void_p, C.c_void_p, P(CTiming))
_sig("rs_forward_many", C.c_int, C.c_void_p, C.c_int64, P(CQuery), P(C.c_void_p), C.c_void_p,
     P(C.c_double), P(C.c_double))
_sig("rs_forward_many_ev", C.c_int, C.c_void_p, C.c_int64, P(CQuery), P(C.c_void_p), C.c_void_p,
     P(C.c_double), P(C.c_double), C.c_void_p)
_sig("rs_sync", C.c_int, C.c_void_p, C.c_void_p)
_sig("rs_accel_set_option", C.c_int, C.c_void_p, C.c_int32, C.c_int64)
_sig("rs_serve", C.c_int, P(C.c_void_p), C.c_int32, C.c_int64, P(CQuery), P(C.c_double),
     P(C.c_void_p), P(C.c_double))
_sig("rs_service_time", C.c_int, C.c_void_p, C.c_int64, P(C.c_double))
_sig("rs_service_breakdown", C.c_int, C.c_void_p, C.c_int64, P(C.c_double), P(C.c_double),
     P(C.c_double))
_sig("rs_host_sls", C.c_int, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
     C.c_int64, C.c_void_p, C.c_void_p, C.c_int32)
_sig("rs_host_fc", C.c_int, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
     C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32)
_sig("rs_fill_query", C.c_int, P(CModelDesc), C.c_int64, C.c_uint64, C.c_uint64, C.c_int64,
     C.c_void_p, C.c_void_p)
_sig("rs_fill_query_zipf", C.c_int, P(CModelDesc), C.c_int64, C.c_uint64, C.c_uint64, C.c_int64,
     C.c_double, C.c_void_p, C.c_void_p)
_sig("rs_alloc_pinned", C.c_int, C.c_size_t, P(C.c_void_p))
_sig("rs_alloc_pinned_flags", C.c_int, C.c_size_t, C.c_uint32, P(C.c_void_p))
_sig("rs_free_pinned", C.c_int, C.c_void_p)
_sig("rs_device_count", C.c_int, P(C.c_int))
_sig("rs_host_model_create", C.c_int, P(CModelDesc), P(CInitDesc), C.c_int32, P(C.c_void_p))
_sig("rs_host_model_destroy", C.c_int, C.c_void_p)
_sig("rs_host_forward", C.c_int, C.c_void_p, P(CQuery), C.c_void_p, C.c_int32)
_sig("rs_serve_hybrid", C.c_int, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, P(C.c_void_p),
     C.c_int32, C.c_int64, P(CQuery), P(C.c_double), P(C.c_void_p), P(C.c_double),
     P(C.c_int32))
_sig("rs_build_flags", C.c_int)

EXPORTED_SYMBOLS = [
    "rs_abi_version", "rs_last_error", "rs_model_builtin", "rs_zoo_names", "rs_model_validate",
    "rs_work", "rs_predict_input_dim", "rs_accel_input_bytes", "rs_sla_target", "rs_route",
    "rs_dist_production", "rs_gen_trace", "rs_qps_under_sla", "rs_accel_create",
    "rs_accel_destroy", "rs_accel_info_get", "rs_forward", "rs_forward_many", "rs_forward_many_ev", "rs_sync",
    "rs_pooled", "rs_service_time", "rs_service_breakdown", "rs_host_sls", "rs_host_fc",
    "rs_fill_query", "rs_fill_query_zipf", "rs_alloc_pinned", "rs_alloc_pinned_flags", "rs_free_pinned",
    "rs_device_count", "rs_accel_set_option", "rs_serve", "rs_build_flags",
    "rs_host_model_create", "rs_host_model_destroy", "rs_host_forward", "rs_serve_hybrid"]


# ---- operator API (model_zoo.hpp mirror) ------------------------------------
@dataclass
class LayerStack:
    """recsim::LayerStack (model_zoo.hpp:39-44)."""
    dims: List[int]

    def output_dim(self) -> int:
        return self.dims[-1]


@dataclass
class EmbeddingConfig:
    """recsim::EmbeddingConfig (model_zoo.hpp:46-52)."""
    num_tables: int = 0
    lookups_per_table: int = 1
    embedding_dim: int = 32
    pooling: str = "Sum"


@dataclass
class ModelSpec:
    """recsim::ModelSpec (model_zoo.hpp:54-65)."""
    name: str = ""
    dense_fc: Optional[LayerStack] = None
    predict_fc: LayerStack = field(default_factory=lambda: LayerStack([1]))
    num_parallel_predict_stacks: int = 1
    embeddings: EmbeddingConfig = field(default_factory=EmbeddingConfig)
    dense_input_dim: int = 0
    recurrent_hidden_dim: Optional[int] = None

    def to_c(self) -> CModelDesc:
        d = CModelDesc()
        d.name = self.name.encode()[:31]
        if self.dense_fc is not None:
            if len(self.dense_fc.dims) > MAX_LAYERS:
                raise InvalidArgument("dense_fc: too many layers")
            d.has_dense_fc = 1
            d.dense_fc.n = len(self.dense_fc.dims)
            for i, v in enumerate(self.dense_fc.dims):
                d.dense_fc.dims[i] = int(v)
        if len(self.predict_fc.dims) > MAX_LAYERS:
            raise InvalidArgument("predict_fc: too many layers")
        d.predict_fc.n = len(self.predict_fc.dims)
        for i, v in enumerate(self.predict_fc.dims):
            d.predict_fc.dims[i] = int(v)
        d.num_parallel_predict_stacks = self.num_parallel_predict_stacks
        e = self.embeddings
        d.num_tables, d.lookups_per_table, d.embedding_dim = (
            e.num_tables, e.lookups_per_table, e.embedding_dim)
        if e.pooling not in POOLING:
            raise InvalidArgument("unknown pooling: " + str(e.pooling))
        d.pooling = POOLING[e.pooling]
        d.dense_input_dim = self.dense_input_dim
        d.recurrent_hidden_dim = self.recurrent_hidden_dim or 0
        return d

    @staticmethod
    def from_c(d: CModelDesc) -> "ModelSpec":
        return ModelSpec(
            name=d.name.decode(),
            dense_fc=LayerStack([d.dense_fc.dims[i] for i in range(d.dense_fc.n)])
            if d.has_dense_fc else None,
            predict_fc=LayerStack([d.predict_fc.dims[i] for i in range(d.predict_fc.n)]),
            num_parallel_predict_stacks=d.num_parallel_predict_stacks,
            embeddings=EmbeddingConfig(d.num_tables, d.lookups_per_table, d.embedding_dim,
                                       POOLING_NAMES[d.pooling]),
            dense_input_dim=d.dense_input_dim,
            recurrent_hidden_dim=d.recurrent_hidden_dim or None)

    def validate(self) -> None:
        """ModelSpec::validate (model_zoo.cpp:41-59)."""
        _check(_lib.rs_model_validate(C.byref(self.to_c())))


def builtin_model(name: str) -> ModelSpec:
    """builtin_model (model_zoo.cpp:141-170)."""
    d = CModelDesc()
    _check(_lib.rs_model_builtin(name.encode(), C.byref(d)))
    return ModelSpec.from_c(d)


def zoo_names() -> List[str]:
    """zoo_names (model_zoo.cpp:172-175)."""
    n = C.c_int()
    arr = (C.c_char_p * 16)()
    _check(_lib.rs_zoo_names(arr, 16, C.byref(n)))
    return [arr[i].decode() for i in range(n.value)]


@dataclass
class WorkBreakdown:
    """recsim::WorkBreakdown (model_zoo.hpp:72-84): per-category flops/bytes."""
    flops: List[float]
    bytes: List[float]
    gather_stream: float

    def __getitem__(self, cat: str):
        i = OP_CATEGORIES.index(cat)
        return self.flops[i], self.bytes[i]

    def total_flops(self) -> float:
        return sum(self.flops)

    def total_bytes(self) -> float:
        return sum(self.bytes)


def work(model: ModelSpec, batch: int) -> WorkBreakdown:
    """work(m, batch) (model_zoo.cpp:177-245)."""
    w = CWork()
    _check(_lib.rs_work(C.byref(model.to_c()), batch, C.byref(w)))
    return WorkBreakdown(list(w.flops), list(w.bytes), w.gather_stream)


def predict_input_dim(model: ModelSpec) -> int:
    """predict_input_dim (model_zoo.cpp:113-137)."""
    v = C.c_int64()
    _check(_lib.rs_predict_input_dim(C.byref(model.to_c()), C.byref(v)))
    return v.value


def accel_input_bytes(model: ModelSpec, query_size: int) -> float:
    """accel_input_bytes (platform.cpp:105-111)."""
    v = C.c_double()
    _check(_lib.rs_accel_input_bytes(C.byref(model.to_c()), query_size, C.byref(v)))
    return v.value


def sla_target(model_name: str, level: str) -> float:
    """sla_target (autotune.cpp:73-88), seconds."""
    v = C.c_double()
    _check(_lib.rs_sla_target(model_name.encode(), level.encode(), C.byref(v)))
    return v.value


# ---- scheduler interface ----------------------------------------------------
def route(query_size: int, batch_size: int, threshold: Optional[int]):
    """The arrival decision of simulate() (sim.cpp:178-188).

    Returns ("accel", [query_size]) or ("cpu", [request sizes in FIFO order]).
    """
    off = C.c_int32()
    cap = query_size // max(batch_size, 1) + 2
    reqs = (C.c_int64 * cap)()
    n = C.c_int64()
    _check(_lib.rs_route(query_size, batch_size, threshold or 0, C.byref(off), reqs, cap,
                         C.byref(n)))
    if off.value:
        return "accel", [query_size]
    return "cpu", [reqs[i] for i in range(n.value)]


@dataclass
class SizeDistribution:
    """recsim::SizeDistribution (loadgen.hpp:23-45)."""
    kind: str = "Fixed"
    p0: float = 25.0
    p1: float = 0.0
    p2: float = 0.0
    p3: float = 0.0
    max_size: int = 1000

    KINDS = {"Fixed": 0, "Normal": 1, "LogNormal": 2, "ProductionHeavyTail": 3}

    @staticmethod
    def production_heavy_tail() -> "SizeDistribution":
        c = CSizeDist()
        _check(_lib.rs_dist_production(C.byref(c)))
        return SizeDistribution("ProductionHeavyTail", c.p0, c.p1, c.p2, c.p3, c.max_size)

    @staticmethod
    def fixed(size: int) -> "SizeDistribution":
        return SizeDistribution("Fixed", float(size))

    @staticmethod
    def log_normal(mu: float, sigma: float) -> "SizeDistribution":
        return SizeDistribution("LogNormal", mu, sigma)

    @staticmethod
    def normal(mu: float, sigma: float) -> "SizeDistribution":
        return SizeDistribution("Normal", mu, sigma)

    def to_c(self) -> CSizeDist:
        return CSizeDist(self.KINDS[self.kind], self.p0, self.p1, self.p2, self.p3,
                         self.max_size)


def gen_trace(seed: int, lam: float, dist: SizeDistribution, n: int):
    """gen_trace (loadgen.cpp:106-125): (arrival_times f64[n], sizes i64[n])."""
    arr = np.empty(n, dtype=np.float64)
    sz = np.empty(n, dtype=np.int64)
    _check(_lib.rs_gen_trace(seed, lam, C.byref(dist.to_c()), n,
                             arr.ctypes.data_as(P(C.c_double)),
                             sz.ctypes.data_as(P(C.c_int64))))
    return arr, sz


@dataclass
class QpsResult:
    qps: float
    at_lambda: float
    p95: float
    p50: float
    evaluations: int


def qps_under_sla(service_s: Sequence[float], sla: float, servers: int = 1,
                  warmup_fraction: float = 0.1, base_seed: int = 42,
                  lambda_hi: float = 0.0, extra_s: Optional[Sequence[float]] = None
                  ) -> QpsResult:
    """max_qps_under_sla (sim.cpp:246-290) over measured per-query service times;
    extra_s adds each query's in-pipeline residence beyond its service gap."""
    s = np.ascontiguousarray(service_s, dtype=np.float64)
    x = None if extra_s is None else np.ascontiguousarray(extra_s, dtype=np.float64)
    if x is not None and len(x) != len(s):
        raise InvalidArgument("extra_s length differs from service_s")
    r = CQpsResult()
    _check(_lib.rs_qps_under_sla(s.ctypes.data_as(P(C.c_double)),
                                 x.ctypes.data_as(P(C.c_double)) if x is not None else None,
                                 len(s), servers, sla, warmup_fraction, base_seed, lambda_hi,
                                 C.byref(r)))
    return QpsResult(r.qps, r.at_lambda, r.p95, r.p50, r.evaluations)


def experiments_built() -> bool:
    """True if the library was built with the measured-slower alternatives
    (make EXPERIMENTS=1; rs_build_flags)."""
    return bool(_lib.rs_build_flags() & 1)


def device_count() -> int:
    n = C.c_int()
    _check(_lib.rs_device_count(C.byref(n)))
    return n.value


def fill_query(model: ModelSpec, rows: int, seed: int, query_id: int, size: int,
               zipf_alpha: float = 0.0):
    """Synthetic inputs of DESIGN.md §3: (dense f32[S,dense_in], idx i64[S,T,L]).
    zipf_alpha > 0: indices from the bounded power law of rs_fill_query_zipf
    (low indices hot), same dense features."""
    e = model.embeddings
    dense = np.empty((size, model.dense_input_dim), dtype=np.float32)
    idx = np.empty((size, e.num_tables, e.lookups_per_table), dtype=np.int64)
    if zipf_alpha > 0:
        _check(_lib.rs_fill_query_zipf(C.byref(model.to_c()), rows, seed, query_id, size,
                                       float(zipf_alpha), dense.ctypes.data, idx.ctypes.data))
    else:
        _check(_lib.rs_fill_query(C.byref(model.to_c()), rows, seed, query_id, size,
                                  dense.ctypes.data, idx.ctypes.data))
    return dense, idx


def host_sls(tables: np.ndarray, idx: np.ndarray, threads: int = 0) -> np.ndarray:
    """SparseLengthsSum on the host cores (the CPU side of the split, SURVEY
    §8f-4): tables f32[T, rows, D], idx i64[S, T, L] -> pooled f32[S, T*D],
    bit-identical to Accelerator.pooled's Sum path. threads <= 0: all."""
    tables = np.ascontiguousarray(tables, dtype=np.float32)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    T, rows, D = tables.shape
    S, Ti, L = idx.shape
    if Ti != T:
        raise InvalidArgument(f"indices name {Ti} tables, tables hold {T}")
    out = np.empty((S, T * D), dtype=np.float32)
    _check(_lib.rs_host_sls(tables.ctypes.data, rows, T, L, D, S, idx.ctypes.data,
                            out.ctypes.data, int(threads)))
    return out


def host_fc(x: np.ndarray, weight: np.ndarray, bias: Optional[np.ndarray] = None,
            relu: bool = True, threads: int = 0, in_dim: Optional[int] = None) -> np.ndarray:
    """Fully connected layer on the host cores: x f32[M, in],
    weight f32[out, ldw] with ldw >= in (the device layout pads rows to
    round4(in); pass in_dim when the weight rows are padded), bias f32[out] or
    None -> f32[M, out]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    weight = np.ascontiguousarray(weight, dtype=np.float32)
    M, K = x.shape
    N, ldw = weight.shape
    if in_dim is not None and in_dim != K:
        raise InvalidArgument(f"in_dim {in_dim} but x has {K} features")
    if ldw < K or (in_dim is None and ldw != K):
        raise InvalidArgument(f"weight is [{N}, {ldw}], x has {K} features")
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    if b is not None and b.shape != (N,):
        raise InvalidArgument(f"bias shape {b.shape}, expected ({N},)")
    y = np.empty((M, N), dtype=np.float32)
    _check(_lib.rs_host_fc(x.ctypes.data, M, K, weight.ctypes.data, ldw,
                           None if b is None else b.ctypes.data, N, int(relu),
                           y.ctypes.data, int(threads)))
    return y


# ---- the accelerator -------------------------------------------------------
@dataclass
class Timing:
    h2d_ms: float
    compute_ms: float
    d2h_ms: float
    total_ms: float
    embed_ms: float = 0.0
    fc_ms: float = 0.0


class Accelerator:
    """One model replica on one B200 (rs_accel_create). Replaces the modeled
    accelerator of accel_service_time (platform.cpp:113-136) with execution."""

    def __init__(self, model: ModelSpec, rows_per_table: int, seed: int = 1,
                 device: int = 0, max_query_size: int = 1000, fc_mode: int = FC_FP32,
                 rnn_cell: int = RNN_GRU, queue_depth: int = 4, l2_persist_mb: int = 0):
        self.model = model
        self.rows = rows_per_table
        self.seed = seed
        self._desc = model.to_c()
        init = CInitDesc(seed, rows_per_table, max_query_size, fc_mode, rnn_cell, l2_persist_mb,
                         queue_depth)
        h = C.c_void_p()
        _check(_lib.rs_accel_create(C.byref(self._desc), C.byref(init), device, C.byref(h)))
        self._h = h
        info = CAccelInfo()
        _check(_lib.rs_accel_info_get(self._h, C.byref(info)))
        self.info = info
        self.output_dim = info.output_dim
        self.pooled_dim = info.pooled_dim

    def close(self) -> None:
        if getattr(self, "_h", None):
            _check(_lib.rs_accel_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _query(self, size, dense_ptr, idx_ptr, location, index_type=INDEX_I64) -> CQuery:
        return CQuery(size, dense_ptr, idx_ptr, location, index_type)

    def forward_ptr(self, size: int, dense_ptr: int, idx_ptr: int, out_ptr: int,
                    location: int, stream: int = 0, timed: bool = False,
                    index_type: int = 0):
        """Raw-pointer call (host pinned or device memory), the C-ABI as is.
        index_type INDEX_I32: `idx_ptr` holds int32 (labelled input variant)."""
        q = self._query(size, dense_ptr, idx_ptr, location, index_type)
        t = CTiming()
        _check(_lib.rs_forward(self._h, C.byref(q), out_ptr, stream or None,
                               C.byref(t) if timed else None))
        return Timing(t.h2d_ms, t.compute_ms, t.d2h_ms, t.total_ms, t.embed_ms, t.fc_ms) if timed else None

    def pooled_ptr(self, size: int, idx_ptr: int, out_ptr: int, location: int,
                   stream: int = 0, timed: bool = False, dense_ptr: int = 0,
                   index_type: int = 0):
        q = self._query(size, dense_ptr, idx_ptr, location, index_type)
        t = CTiming()
        _check(_lib.rs_pooled(self._h, C.byref(q), out_ptr, stream or None,
                              C.byref(t) if timed else None))
        return Timing(t.h2d_ms, t.compute_ms, t.d2h_ms, t.total_ms, t.embed_ms, t.fc_ms) if timed else None

    @staticmethod
    def batch(sizes, dense_ptrs, idx_ptrs, out_ptrs, location: int, index_type: int = 0):
        """Pre-built argument arrays for forward_many (keeps Python work out of
        timed regions)."""
        n = len(sizes)
        qs = (CQuery * n)()
        for i in range(n):
            qs[i] = CQuery(int(sizes[i]), dense_ptrs[i] or None, idx_ptrs[i] or None, location,
                           index_type)
        outs = (C.c_void_p * n)(*[C.c_void_p(p) for p in out_ptrs])
        return n, qs, outs

    def forward_many(self, sizes, dense_ptrs=None, idx_ptrs=None, out_ptrs=None,
                     location: int = MEM_DEVICE, stream: int = 0, timed: bool = True,
                     residence: bool = False, prepared=None, done_event: int = 0):
        """rs_forward_many: n whole queries, FIFO-dispatched over the handle's
        lanes. Returns per-query service times in ms when timed (else None);
        with residence=True returns (service_ms, residence_ms)."""
        n, qs, outs = prepared or self.batch(sizes, dense_ptrs, idx_ptrs, out_ptrs, location)
        svc = np.zeros(n, dtype=np.float64) if timed else None
        lat = np.zeros(n, dtype=np.float64) if (timed and residence) else None
        _check(_lib.rs_forward_many_ev(self._h, n, qs, outs, stream or None,
                                       svc.ctypes.data_as(P(C.c_double)) if timed else None,
                                       lat.ctypes.data_as(P(C.c_double)) if lat is not None
                                       else None, done_event or None))
        return (svc, lat) if residence else svc

    def set_option(self, option: int, value: int) -> None:
        """rs_accel_set_option, e.g. (OPT_MERGE_QUERIES, 2): up to 2 consecutive
        queries per launch in forward_many (labelled)."""
        _check(_lib.rs_accel_set_option(self._h, option, value))

    def sync(self, stream: int = 0) -> None:
        """rs_sync: wait for `stream`, raise any sticky error (e.g. bad index)."""
        _check(_lib.rs_sync(self._h, stream or None))

    def forward(self, dense: np.ndarray, idx: np.ndarray) -> np.ndarray:
        """Host numpy in, host numpy out (synchronous): logits [S, stacks*out].
        int32 `idx` selects the labelled INDEX_I32 input variant."""
        S = int(idx.shape[0]) if idx.size else int(dense.shape[0])
        bf16 = dense.dtype == np.uint16  # raw bfloat16 bit patterns: labelled variant
        dense = np.ascontiguousarray(dense, dtype=np.uint16 if bf16 else np.float32)
        i32 = idx.dtype == np.int32
        idx = np.ascontiguousarray(idx, dtype=np.int32 if i32 else np.int64)
        out = np.empty((S, self.output_dim), dtype=np.float32)
        self.forward_ptr(S, dense.ctypes.data, idx.ctypes.data, out.ctypes.data, MEM_HOST,
                         timed=True, index_type=(INDEX_I32 if i32 else INDEX_I64) |
                         (DENSE_BF16 if bf16 else 0))
        return out

    def pooled(self, idx: np.ndarray, dense: Optional[np.ndarray] = None) -> np.ndarray:
        S = int(idx.shape[0])
        i32 = idx.dtype == np.int32
        idx = np.ascontiguousarray(idx, dtype=np.int32 if i32 else np.int64)
        out = np.empty((S, self.pooled_dim), dtype=np.float32)
        self.pooled_ptr(S, idx.ctypes.data, out.ctypes.data, MEM_HOST, timed=True,
                        index_type=INDEX_I32 if i32 else INDEX_I64)
        return out

    def service_breakdown(self, query_size: int) -> dict:
        """rs_service_breakdown: the measured recsim::ServiceTime (seconds):
        total, transfer and the per-category split of the compute time."""
        tot, tr = C.c_double(), C.c_double()
        pc = (C.c_double * NUM_OP_CATEGORIES)()
        _check(_lib.rs_service_breakdown(self._h, query_size, C.byref(tot), C.byref(tr), pc))
        return {"total": tot.value, "transfer": tr.value,
                "per_category": dict(zip(OP_CATEGORIES, list(pc)))}

    def service_time(self, query_size: int) -> float:
        """Measured whole-query seconds, memoised per size (sim.cpp:81-88)."""
        v = C.c_double()
        _check(_lib.rs_service_time(self._h, query_size, C.byref(v)))
        return v.value


def serve(replicas: Sequence["Accelerator"], prepared, arrival_s) -> np.ndarray:
    """rs_serve: release query i at arrival_s[i] (seconds from the call),
    least-outstanding-items replica, real execution; returns per-query
    latency (ms) = completion - arrival. `prepared` = Accelerator.batch(...)."""
    n, qs, outs = prepared
    arr = np.ascontiguousarray(arrival_s, dtype=np.float64)
    if arr.shape[0] != n:
        raise InvalidArgument("arrival_s must have one entry per query")
    hs = (C.c_void_p * len(replicas))(*[r._h for r in replicas])
    lat = np.zeros(n, dtype=np.float64)
    _check(_lib.rs_serve(hs, len(replicas), n, qs, arr.ctypes.data_as(P(C.c_double)), outs,
                         lat.ctypes.data_as(P(C.c_double))))
    return lat


class HostModel:
    """The same model on the host cores (rs_host_model): the CPU side of
    DeepRecSched's split, executed (proj/src/sim.cpp:114-124, 184-188)."""

    def __init__(self, model: ModelSpec, rows_per_table: int, seed: int = 1,
                 rnn_cell: int = RNN_GRU, threads: int = 0):
        self.model = model
        self._desc = model.to_c()
        init = CInitDesc(seed, rows_per_table, 1, FC_FP32, rnn_cell, 0, 0)
        h = C.c_void_p()
        _check(_lib.rs_host_model_create(C.byref(self._desc), C.byref(init), int(threads),
                                         C.byref(h)))
        self._h = h
        self.output_dim = model.num_parallel_predict_stacks * model.predict_fc.dims[-1]

    def close(self) -> None:
        if getattr(self, "_h", None):
            _check(_lib.rs_host_model_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, dense: np.ndarray, idx: np.ndarray, threads: int = 1) -> np.ndarray:
        """One request on the host cores: logits f32[S, stacks*out]."""
        S = int(idx.shape[0]) if idx.size else int(dense.shape[0])
        dense = np.ascontiguousarray(dense, dtype=np.float32)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty((S, self.output_dim), dtype=np.float32)
        q = CQuery(S, dense.ctypes.data or None, idx.ctypes.data or None, MEM_HOST, 0)
        _check(_lib.rs_host_forward(self._h, C.byref(q), out.ctypes.data, int(threads)))
        return out


def serve_hybrid(cpu: HostModel, cores: int, batch: int, threshold: int,
                 replicas: Sequence["Accelerator"], prepared, arrival_s):
    """rs_serve_hybrid: real-time DeepRecSched over `cores` host threads and
    the replicas; returns (latency_ms, offloaded) per query."""
    n, qs, outs = prepared
    arr = np.ascontiguousarray(arrival_s, dtype=np.float64)
    if arr.shape[0] != n:
        raise InvalidArgument("arrival_s must have one entry per query")
    hs = (C.c_void_p * max(1, len(replicas)))(*[r._h for r in replicas])
    lat = np.zeros(n, dtype=np.float64)
    off = np.zeros(n, dtype=np.int32)
    _check(_lib.rs_serve_hybrid(cpu._h, int(cores), int(batch), int(threshold), hs,
                                len(replicas), n, qs, arr.ctypes.data_as(P(C.c_double)), outs,
                                lat.ctypes.data_as(P(C.c_double)),
                                off.ctypes.data_as(P(C.c_int32))))
    return lat, off


class PinnedBuffer:
    """Page-locked host buffer from rs_alloc_pinned, viewable as numpy."""

    def __init__(self, nbytes: int, write_combined: bool = False):
        p = C.c_void_p()
        _check(_lib.rs_alloc_pinned_flags(nbytes, 1 if write_combined else 0, C.byref(p)))
        self.ptr = p.value
        self.nbytes = nbytes

    def view(self, dtype, shape):
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        assert n <= self.nbytes
        buf = (C.c_char * n).from_address(self.ptr)
        return np.frombuffer(buf, dtype=dtype).reshape(shape)

    def __del__(self):
        if getattr(self, "ptr", None):
            _lib.rs_free_pinned(C.c_void_p(self.ptr))
            self.ptr = None
