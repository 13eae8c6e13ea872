"""bench.py — QPS at a p95 SLA for the offloaded recommendation forward pass on
B200 replicas, plus the SLS kernel's HBM roofline and the CPU baseline.

Workload (BASELINE.json configs[2], the SLS-bound DLRM config the 1/2/4/8-GPU
sweep is defined on; its metric names "SLS HBM GB/s vs peak"):
  DLRM-RMC2 at cfg3 shape: 32 tables x 10M rows x dim 64 fp32 (81.9 GB per
  GPU), 80 lookups/table, bottom MLP 256-128-64, top MLP 656-512-128-1;
  query sizes LogNormal(ln 300, 0.5) clamped to [1, 1000],
  Poisson arrivals; SLA = sla_target("DLRM-RMC2", "medium") = 400 ms.

A step = one window of Q consecutive queries of the rank's stream, each served
whole through the C-ABI (rs_forward), back to back on one CUDA stream.
  value  = QPS at p95 <= SLA: per-query device service times from CUDA events
           inside the timed region, replayed open-loop with Poisson arrivals
           (FIFO server, exact p95, geometric lambda bisection to 1% — the rule
           of proj/src/sim.cpp:246-290); whole job = N x min over ranks.
  e2e    = the same metric with host (pinned) inputs: H2D of dense+indices and
           D2H of the logits inside every query's service time.
Multi-GPU: one process per GPU, independent replicas (each rank its own
query stream, seed 42 + 10007*rank); no collective on the data path
 — only the timing barrier and max-over-ranks reduction.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the pipelined queue runs 8 lane streams + a copy stream + graph branches;
# with the default 8 hardware work queues unrelated lanes serialise behind
# each other (tools/timeline.py). Must be set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "QPS at p95 tail-latency SLA per model at 1/2/4/8 B200; SLS HBM GB/s vs peak"
NOMINAL_HBM_GBS = 8000.0


# Workloads as neutral shape descriptions, so that the CPU reference arm can
# build them without importing the product package (it uses the compiled
# reference's own zoo through oracle/cpu_arm.py). zoo=… without shapes means
# the reference's builtin_model (proj/src/model_zoo.cpp:141-170).
WORKLOADS = {
    "cfg3-rmc2": dict(name="cfg3-DLRM-RMC2", zoo="DLRM-RMC2", rows=10_000_000,
                      dense_fc=[256, 128, 64], predict_fc=[512, 128, 1], T=32, L=80, D=64,
                      pooling="Sum", dense_in=256),
    "cfg3-rmc3": dict(name="cfg3-DLRM-RMC3", zoo="DLRM-RMC3", rows=10_000_000,
                      dense_fc=[2560, 512, 64], predict_fc=[512, 128, 1], T=32, L=20, D=64,
                      pooling="Sum", dense_in=256),
    "cfg1-rmc1": dict(name="cfg1-DLRM-RMC1", zoo="DLRM-RMC1", rows=1_000_000,
                      dense_fc=[256, 128, 32], predict_fc=[256, 64, 1], T=8, L=80, D=32,
                      pooling="Sum", dense_in=256),
    # BASELINE configs[4]: DIEN GRU seq len 100
    "cfg5-dien": dict(name="cfg5-DIEN", zoo="DIEN", rows=1_000_000, predict_fc=[200, 80, 2],
                      T=20, L=100, D=32, pooling="AttentionRNN", hidden=64),
    "cfg5-din": dict(zoo="DIN", rows=1_000_000),
    "ncf": dict(zoo="NCF", rows=1_000_000), "wnd": dict(zoo="WND", rows=1_000_000),
    "mt-wnd": dict(zoo="MT-WND", rows=1_000_000), "din": dict(zoo="DIN", rows=1_000_000),
    "dien": dict(zoo="DIEN", rows=1_000_000), "rmc1": dict(zoo="DLRM-RMC1", rows=1_000_000),
    "rmc2": dict(zoo="DLRM-RMC2", rows=1_000_000), "rmc3": dict(zoo="DLRM-RMC3", rows=1_000_000),
}
# workloads whose dominant kernel is the predict stack (tensor-pipe roofline)
TENSOR_BOUND = ("mt-wnd", "wnd")


def workload_spec(rs, name):
    """(product ModelSpec, rows per table, zoo name for sla_target)."""
    w = WORKLOADS[name]
    if "T" not in w:
        return rs.builtin_model(w["zoo"]), w["rows"], w["zoo"]
    return rs.ModelSpec(w["name"], dense_fc=rs.LayerStack(w["dense_fc"]) if w.get("dense_fc") else None,
                        predict_fc=rs.LayerStack(w["predict_fc"]),
                        embeddings=rs.EmbeddingConfig(w["T"], w["L"], w["D"], w["pooling"]),
                        dense_input_dim=w.get("dense_in", 0),
                        recurrent_hidden_dim=w.get("hidden")), w["rows"], w["zoo"]


def cta_pairs_on(args):
    """RS_OPT_CTA_PAIRS: measured faster for uniform-size queues only."""
    c = getattr(args, "cta_pairs", "auto")
    return c == "on" or (c == "auto" and bool(getattr(args, "size_fixed", 0)))


def workload_or_model(name):
    """The same workload as the oracle's C model struct (no product import)."""
    from oracle import cpu_arm
    w = WORKLOADS[name]
    if "T" not in w:
        return cpu_arm.builtin_model(w["zoo"]), w["rows"], w["zoo"]
    pool = {"Sum": 0, "Concat": 1, "AttentionFC": 2, "AttentionRNN": 3}[w["pooling"]]
    return cpu_arm.make_model(w["name"], w["predict_fc"], w["T"], w["L"], w["D"], pool,
                              dense_in=w.get("dense_in", 0), dense_fc=w.get("dense_fc"),
                              hidden=w.get("hidden", 0)), w["rows"], w["zoo"]


def sla_for(args, zoo_name, sla_target):
    """configs[4] states a 100 ms p95 SLA for DIN/DIEN; elsewhere
    the reference's medium target (proj/src/autotune.cpp:73-88)."""
    if args.sla > 0:
        return args.sla
    return 0.100 if args.workload.startswith("cfg5") else sla_target(zoo_name, "medium")


def size_dist(args):
    """(p0, p1, kind) of the query-size distribution for the reference's
    tune(): LogNormal(ln m, 0.5), or Fixed(N) with --size-fixed."""
    if args.size_fixed:
        return float(args.size_fixed), 0.0, 0
    return math.log(args.size_median), 0.5, 2


def window(k, Q):
    base = (k % 2) * Q
    return range(base, base + Q)


def make_config(args, name, shape, rows, sizes, world, sla):
    """The JSON line's `config`: a function of the workload and the flags only,
    identical in both arms (the driver compares them)."""
    T, L, D, dense_in = shape
    Q, K = args.queries_per_step, args.steps
    i32, bf16 = args.index_bits == 32, args.dense_bits == 16
    items_step = float(np.mean([sum(int(sizes[q]) for q in window(k, Q)) for k in range(K)]))
    h2d_step = items_step * (dense_in * (2 if bf16 else 4) + T * L * (4 if i32 else 8))
    return {
        "workload": args.workload, "model": name, "rows_per_table": rows,
        "tables": T, "lookups": L, "dim": D, "queries_per_step": Q,
        "items_per_step": items_step, "sla_s": sla,
        "size_distribution": (f"Fixed({args.size_fixed}) (configs[3] batch sweep)"
                              if args.size_fixed else
                              f"LogNormal(ln {args.size_median:g}, 0.5) clamped to "
                              f"[1, {args.max_query}] (SURVEY 8d (i))"),
        "fc_path": args.fc, "cta_pairs": cta_pairs_on(args), "parallelism": f"replicas{world}",
        "input_format": ("LABELLED variant (SURVEY 8f-2), not the reference byte model: " +
                         " + ".join((["int32 indices"] if i32 else []) +
                                    (["bf16 dense"] if bf16 else []))
                         if (i32 or bf16) else
                         "reference byte model (int64 indices + fp32 dense)"),
        "query_merging": (f"up to {args.merge} consecutive queries per launch: LABELLED "
                          "scheduler extension (SURVEY 8f-3)" if args.merge > 1 else
                          "off (one query per launch, as the reference's accelerator server)"),
        "l2": "inputs >> L2 (tables %.1f GB, ~%.0f MB of indices per step)" % (
            T * rows * D * 4 / 1e9, h2d_step / 1e6),
        "index_distribution": (
            f"LABELLED variant (SURVEY 8d): bounded power law alpha={args.zipf:g} "
            "over [0, rows), low ids hot" if args.zipf > 0 else "uniform"),
        "l2_persist_mb": args.l2_persist_mb,
        **({"rnn_cell": args.rnn} if args.rnn != "gru" else {}),
    }


def sls_bytes_per_item(spec):
    e = spec.embeddings
    return e.num_tables * e.lookups_per_table * (e.embedding_dim * 4 + 8) + \
        e.num_tables * e.embedding_dim * 4


# ---- distributed plumbing (also exercised by tests/test_bench_dist.py) ------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def rank_seed(rank: int) -> int:
    """The reference's multi-seed scheme (proj/src/autotune.cpp:23)."""
    return 42 + 10007 * rank


def reduce_max(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_min(value: float, device=None) -> float:
    return -reduce_max(-value, device)


def reduce_sum(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(device=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        if device is not None:
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


def aggregate(per_rank_qps: float, per_rank_time: float, queries: int, world: int, device=None):
    """Whole-job numbers: slowest rank's time, N x the worst rank's SLA QPS."""
    t = reduce_max(per_rank_time, device)
    q_min = reduce_min(per_rank_qps, device)
    total_q = reduce_sum(float(queries), device)
    return {"time_s": t, "value": world * q_min, "saturated_qps": total_q / t if t > 0 else 0.0}


# ---- clocks ------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks/throttle sampler. Started before the warm-up (the tool
    needs ~0.5 s to produce its first sample); summary() keeps the samples
    whose host arrival time falls inside the timed window."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self._t = None
        self.window = (0.0, float("inf"))

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["stdbuf", "-oL", "nvidia-smi", "-i", str(self.dev),
                 f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self._t:
                self._t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = self.window
        # 20 ms sampling: allow one period of slack on each side of the window
        inside = [ln for ts, ln in self.lines if t0 - 0.03 <= ts <= t1 + 0.03]
        for ln in inside:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_tensor_peak(fc):
    """Tensor roofline denominator: tcgen05 kind::tf32 issues at half the bf16
    rate, so 0.5 x the measured dense bf16 burst (MEASURED_PEAKS.json); fp32
    FFMA path: the datasheet 75 TF/s fp32 (B200_PROFILING.md)."""
    if fc == "fp32":
        return 75.0, "fp32 FFMA datasheet ~75 TF/s (nothing measured for fp32)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            bf = json.load(f).get("bf16_tflops")
        if bf and fc == "bf16":
            return bf, f"measured dense bf16 {bf:.0f} TF/s (MEASURED_PEAKS.json)"
        if bf:
            return 0.5 * bf, f"0.5 x measured bf16 {bf:.0f} TF/s (MEASURED_PEAKS.json): tf32 rate"
    if fc == "bf16":
        return 2250.0, "fallback: bf16 dense 2.25 PF/s (B200_PROFILING.md)"
    return 1100.0, "fallback: tf32 dense 1.1 PF/s (B200_PROFILING.md)"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6548.2), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---- CPU baseline ------------------------------------------------------------
def cpu_deeprecsched(args, workload, sla, rounds, budget_s, threads=0, rank=0):
    """The CPU side of DeepRecSched run for real (oracle/cpu_arm.py): the
    oracle's fp32 forward (kind "port") timed on REQUESTS of b items on this
    host's cores (1 and all cores busy), tables materialised at the workload's
    full row count; the measured times replace the reference's modeled
    cpu_service_time and the UNMODIFIED reference tune() (CPU only: batch
    ladder, split rule floor(S/B) x B + S mod B over C cores, exact p95,
    lambda bisection; proj/src/autotune.cpp:90-152, proj/src/sim.cpp:114-124,
    184-188, 246-290) gives QPS@p95 <= SLA. Returns (result dict, per-round
    wall seconds)."""
    from oracle import cpu_arm
    m, rows, _ = workload_or_model(workload)
    arm = cpu_arm.CpuDeepRecSched(m, rows, threads=threads)
    walls = [arm.sample(budget_s) for _ in range(rounds)]
    t0 = time.time()
    res = arm.tune(sla, *size_dist(args)[:2], kind=size_dist(args)[2], n=50_000, seed=rank_seed(rank),
                   max_size=args.max_query)
    res["tune_s"] = time.time() - t0
    res["fill_s"] = arm.fill_s
    bs, t1, tc = arm.table()
    res["table"] = {"request_items": bs.tolist(), "s_1core": t1.tolist(),
                    f"s_{arm.threads}cores": tc.tolist()}
    res["threads"] = arm.threads
    res["rows"] = rows
    arm.close()
    return res, walls


def cpu_sample_text(res, rounds):
    if res.get("infeasible"):
        return (f"{rounds} timing rounds of the oracle fp32 forward on requests of "
                f"{res['table']['request_items']} items on {res['threads']} cores "
                f"({res['rows']:,} rows/table): {res['infeasible']} -> 0 QPS at this SLA")
    return (f"{rounds} timing rounds: oracle fp32 forward (oracle/forward.c) on requests of "
            f"{res['table']['request_items']} items, each timed with 1 and with all "
            f"{res['threads']} cores busy, tables materialised at {res['rows']:,} rows/table "
            f"(fill {res['fill_s']:.0f} s); QPS@p95 from the UNMODIFIED reference tune() "
            f"(CPU only) with cpu_service_time replaced by those times "
            f"(oracle/ref_cpu_adapter.cpp): chosen batch B={res['batch']}, "
            f"p95 {res['p95_s'] * 1e3:.1f} ms, n=50,000 queries per evaluation")


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path on this host (oracle port of
    the forward, the reference's own scheduler), same metric and config as the
    B200 arm. Rank 0 only under torchrun. Imports nothing from the product."""
    if rank != 0:
        return
    from oracle import cpu_arm
    m, rows, zoo_name = workload_or_model(args.workload)
    sla = sla_for(args, zoo_name, cpu_arm.sla_target)
    if args.size_fixed:
        sizes = np.full(2 * args.queries_per_step, args.size_fixed, dtype=np.int64)
    else:
        sizes = cpu_arm.gen_trace_sizes(rank_seed(0), math.log(args.size_median), 0.5,
                                        2 * args.queries_per_step, args.max_query)
    sizes = np.minimum(sizes, args.max_query)
    name = m.name.decode()
    cfg = make_config(args, name, (m.T, m.L, m.D, m.dense_in), rows, sizes, world, sla)
    # every round is a bounded sample; warm-up rounds are discarded
    budget = max(1.0, 60.0 / (args.steps + args.warmup))
    try:
        arm = cpu_arm.CpuDeepRecSched(m, rows)
    except MemoryError as e:
        # the arm materialises the workload's full tables in host RAM (82 GB
        # at configs[2]); a host without that memory gets a stated line, not
        # a crash
        gb = m.T * rows * m.D * 4 / 1e9
        print(json.dumps({"metric": METRIC, "impl": "reference", "config": cfg,
                          "unavailable": f"host RAM: the CPU arm materialises {gb:.1f} GB of "
                                         f"tables ({e})"}), flush=True)
        return
    for _ in range(args.warmup):
        arm.sample(budget)
    arm.samples = {b: ([], []) for b in cpu_arm.REQUEST_SIZES}
    walls = [arm.sample(budget) for _ in range(args.steps)]
    res = arm.tune(sla, *size_dist(args)[:2], kind=size_dist(args)[2], n=50_000, seed=rank_seed(0),
                   max_size=args.max_query)
    bs, t1, tc = arm.table()
    res.update(fill_s=arm.fill_s, threads=arm.threads, rows=rows,
               table={"request_items": bs.tolist(), "s_1core": t1.tolist(),
                      f"s_{arm.threads}cores": tc.tolist()})
    arm.close()
    v = res["qps"]
    cb = {"value": v, "unit": "queries/s", "cores": res["threads"], "kind": "port",
          "sample": cpu_sample_text(res, args.steps)}
    line = {"metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(walls)) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "impl": "reference", "config": cfg,
            "method": "CPU-only DeepRecSched on this host: reference tune() over measured "
                      "per-request times (oracle/cpu_arm.py)",
            "cpu_deeprecsched": {"batch": res["batch"],
                                 "p95_ms": res["p95_s"] * 1e3 if res["p95_s"] else None,
                                 "tune_search_steps": res["search_steps"],
                                 "request_time_table": res["table"]},
            "cpu_baseline": cb, "gpu_launches": 0,
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- the B200 arm --------------------------------------------------------------
def run_ours(args, rank, world, local):
    import torch
    import paper_2001_02772_b200 as rs

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)

    spec, rows, zoo_name = workload_spec(rs, args.workload)
    sla = sla_for(args, zoo_name, rs.sla_target)
    Q, K, W = args.queries_per_step, args.steps, args.warmup
    seed = rank_seed(rank)
    if args.size_fixed:
        sizes = np.full(2 * Q, args.size_fixed, dtype=np.int64)
    else:
        _, sizes = rs.gen_trace(seed, 1000.0, rs.SizeDistribution.log_normal(
            math.log(args.size_median), 0.5), 2 * Q)
    sizes = np.minimum(sizes, args.max_query)
    acc = rs.Accelerator(spec, rows, seed=1, device=local, max_query_size=args.max_query,
                         fc_mode={"fp32": rs.FC_FP32, "tf32": rs.FC_TF32, "auto": rs.FC_AUTO,
                                  "bf16": rs.FC_BF16}[args.fc],
                         queue_depth=args.depth, l2_persist_mb=args.l2_persist_mb,
                         rnn_cell=rs.RNN_AUGRU if args.rnn == "augru" else rs.RNN_GRU)
    if args.merge > 1:
        acc.set_option(rs.OPT_MERGE_QUERIES, args.merge)
    if cta_pairs_on(args):
        acc.set_option(rs.OPT_CTA_PAIRS, 1)
    e = spec.embeddings
    # pool of 2Q distinct queries: pinned host copies (e2e) and device copies (value)
    P = 2 * Q
    d_dense, d_idx, h_dense, h_idx = [], [], [], []
    i32 = args.index_bits == 32
    bf16 = args.dense_bits == 16
    ity = (rs.INDEX_I32 if i32 else rs.INDEX_I64) | (rs.DENSE_BF16 if bf16 else 0)
    for q in range(P):
        dn, ix = rs.fill_query(spec, rows, seed, q, int(sizes[q]), zipf_alpha=args.zipf)
        if i32:
            ix = ix.astype(np.int32)
        if bf16:
            dn = (dn.view(np.uint32) >> 16).astype(np.uint16)
        if args.pack and dn.nbytes:
            # one pinned buffer per query, [dense | indices]: the library moves
            # a packed query with one transfer (same bytes)
            hb = rs.PinnedBuffer(dn.nbytes + ix.nbytes)
            hb.view(np.uint8, (dn.nbytes + ix.nbytes,))[...] = np.concatenate(
                [dn.reshape(-1).view(np.uint8), ix.reshape(-1).view(np.uint8)])
            h_dense.append((hb, hb.ptr))
            h_idx.append((hb, hb.ptr + dn.nbytes))
        else:
            hb_d = rs.PinnedBuffer(max(dn.nbytes, 16))
            hb_i = rs.PinnedBuffer(max(ix.nbytes, 16))
            hb_d.view(dn.dtype, dn.shape)[...] = dn
            hb_i.view(ix.dtype, ix.shape)[...] = ix
            h_dense.append((hb_d, hb_d.ptr))
            h_idx.append((hb_i, hb_i.ptr))
        d_dense.append(torch.from_numpy(dn).to(device))
        d_idx.append(torch.from_numpy(ix).to(device))
    out_dev = torch.empty((args.max_query, acc.output_dim), device=device)
    out_host = rs.PinnedBuffer(args.max_query * acc.output_dim * 4)
    stream = torch.cuda.current_stream(device)
    sp = stream.cuda_stream

    def prepare(n_steps, host):
        """rs_forward_many arguments for n_steps windows (built before timing)."""
        qs = [q for k in range(n_steps) for q in window(k, Q)]
        if host:
            dp = [h_dense[q][1] for q in qs]
            ip = [h_idx[q][1] for q in qs]
            op = [out_host.ptr] * len(qs)
            loc = rs.MEM_HOST
        else:
            dp = [d_dense[q].data_ptr() for q in qs]
            ip = [d_idx[q].data_ptr() for q in qs]
            op = [out_dev.data_ptr()] * len(qs)
            loc = rs.MEM_DEVICE
        return acc.batch([int(sizes[q]) for q in qs], dp, ip, op, loc, index_type=ity)

    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    end.record(stream)               # creates the event the library stamps at completion
    torch.cuda.synchronize(device)

    def timed(host):
        with ClockSampler(local) as clk:         # started before warm-up (tool start-up)
            acc.forward_many(None, stream=sp, prepared=prepare(W, host))  # warm-up, untimed
            batch = prepare(K, host)
            torch.cuda.synchronize(device)
            barrier(device)
            torch.cuda.synchronize(device)
            t0 = time.time()
            start.record(stream)
            # per-query CUDA-event times; `end` is recorded by the library on
            # this stream when the last query completed, before it reads the
            # per-query timestamps back (rs_forward_many_ev)
            svc_ms, res_ms = acc.forward_many(None, stream=sp, timed=True, residence=True,
                                              prepared=batch, done_event=end.cuda_event)
            torch.cuda.synchronize(device)
            clk.mark(t0, time.time())
        barrier(device)
        torch.cuda.synchronize(device)
        total_s = start.elapsed_time(end) * 1e-3
        # time a query spends inside the pipelined accelerator beyond its
        # service gap is added to its latency in the SLA replay
        extra = np.maximum(res_ms - svc_ms, 0.0) * 1e-3
        return total_s, svc_ms * 1e-3, extra, clk.summary()

    def sla_qps(svc, extra, lambda_hi=0.0):
        # the reference evaluates traces of n = 50,000 queries
        # (proj/include/recsim/sim.hpp:79): the measured per-query service
        # times are cycled to that length, so an overloaded rate cannot hide
        # behind a short trace
        n = 50_000
        return rs.qps_under_sla(np.resize(svc, n), sla, servers=1, warmup_fraction=0.1,
                                base_seed=seed, extra_s=np.resize(extra, n), lambda_hi=lambda_hi)

    def stable_point(svc, extra):
        """p50/p95 at a stable load: 0.9x the measured service capacity."""
        lam = 0.9 / float(np.mean(svc))
        r = sla_qps(svc, extra, lambda_hi=lam)
        return {"load": 0.9, "lambda": lam, "p50_ms": r.p50 * 1e3, "p95_ms": r.p95 * 1e3,
                "evaluated_at_lambda": r.at_lambda}

    # ---- value: device-resident inputs
    t_dev, svc_dev, extra_dev, clocks = timed(host=False)
    r_dev = sla_qps(svc_dev, extra_dev)
    agg = aggregate(r_dev.qps, t_dev, len(svc_dev), world, device)
    st_dev = stable_point(svc_dev, extra_dev)
    # ---- e2e: host pinned inputs, H2D/D2H inside every query
    t_host, svc_host, extra_host, clocks_e2e = timed(host=True)
    r_host = sla_qps(svc_host, extra_host)
    agg_e2e = aggregate(r_host.qps, t_host, len(svc_host), world, device)
    st_host = stable_point(svc_host, extra_host)

    # ---- per-stage kernel timing (RS_OPT_STAGE_TIMING): event-record nodes
    # captured right around the embedding stage and the predict stack in a
    # timed copy of the forward graph, on the kernels' own stream
    peak_hbm, peak_src = measured_peaks()
    acc.set_option(rs.OPT_STAGE_TIMING, 1)
    emb_ms, fc_ms, fwd_ms, items_roof = 0.0, 0.0, 0.0, 0
    out_roof = torch.empty((args.max_query, acc.output_dim), device=device)
    for q in window(0, Q):
        S = int(sizes[q])
        t = acc.forward_ptr(S, d_dense[q].data_ptr(), d_idx[q].data_ptr(), out_roof.data_ptr(),
                            rs.MEM_DEVICE, stream=sp, timed=True, index_type=ity)
        emb_ms += t.embed_ms
        fc_ms += t.fc_ms
        fwd_ms += t.compute_ms
        items_roof += S
    acc.set_option(rs.OPT_STAGE_TIMING, 0)
    n_roof = len(window(0, Q))
    sls_bytes = items_roof * sls_bytes_per_item(spec)
    pred_flops = rs.work(spec, items_roof)["PredictFC"][0]
    # the SLS kernel alone (pool graph, no concurrent dense branch)
    pooled_dev = torch.empty((args.max_query, acc.pooled_dim), device=device)
    sls_ms = 0.0
    for q in window(0, Q):
        t = acc.pooled_ptr(int(sizes[q]), d_idx[q].data_ptr(), pooled_dev.data_ptr(),
                           rs.MEM_DEVICE, stream=sp, timed=True, index_type=ity)
        sls_ms += t.embed_ms
    achieved = sls_bytes / (sls_ms * 1e-3) / 1e9
    # the same kernel back to back: embedding stage only over the queue's
    # lanes (one query's tail overlaps the next one's ramp), CUDA-event
    # delivery times of rs_forward_many over two windows
    os.environ["RS_MANY_POOL_ONLY"] = "1"
    qs2 = [q for k in range(2) for q in window(k, Q)]
    b2 = acc.batch([int(sizes[q]) for q in qs2], [d_dense[q].data_ptr() for q in qs2],
                   [d_idx[q].data_ptr() for q in qs2], [pooled_dev.data_ptr()] * len(qs2),
                   rs.MEM_DEVICE, index_type=ity)
    acc.forward_many(None, stream=sp, prepared=b2)
    svc2 = acc.forward_many(None, stream=sp, prepared=b2)
    os.environ["RS_MANY_POOL_ONLY"] = "0"
    b2b = sum(int(sizes[q]) for q in qs2) * sls_bytes_per_item(spec) / (svc2.sum() * 1e-3) / 1e9

    cfg = make_config(args, spec.name, (e.num_tables, e.lookups_per_table, e.embedding_dim,
                                        spec.dense_input_dim), rows, sizes, world, sla)
    h2d_step = cfg["items_per_step"] * (spec.dense_input_dim * (2 if bf16 else 4) +
                                        e.num_tables * e.lookups_per_table * (4 if i32 else 8))
    d2h_step = float(np.mean([sum(int(sizes[q]) * acc.output_dim * 4 + 4 for q in window(k, Q))
                              for k in range(K)]))
    # kernel nodes of the graph each timed query launched (pick_graph in
    # csrc/host/accel.cu: one graph per FC path; FC_AUTO/TF32 = the tcgen05 graph)
    launches = int(acc.info.kernels_per_forward * K * Q)
    # DRAM traffic per launch from the committed ncu --set full capture
    # (profiles/sls_traffic.json: dram read+write bytes / items of that launch),
    # scaled to this run's mean items per roofline launch like `achieved`
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "sls_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f).get(args.workload)
        if tj:
            traffic = tj["dram_bytes_per_item"] * items_roof / n_roof
            traffic_src = tj.get("source")
    step_s = t_dev / K
    hbm_roof = {
        "bound": "hbm",
        "kernel": {"Sum": "sls_pipe_kernel", "Concat": "gather_concat_kernel",
                   "AttentionFC": "din_pool_kernel",
                   "AttentionRNN": ("gru_kernel" if args.fc == "fp32" else "gru_tc_kernel") +
                   " (latency-bound recurrence; bytes shown)"}[e.pooling],
        "achieved": achieved, "peak": peak_hbm, "unit": "GB/s",
        "timing": "CUDA events recorded by graph nodes right before and after the kernel, "
                  "on its stream (rs_timing.embed_ms of the embedding-stage graph)",
        "frac": achieved / peak_hbm, "peak_source": peak_src,
        "frac_of_nominal_8tbs": achieved / NOMINAL_HBM_GBS,
        "traffic": traffic, "traffic_source": traffic_src,
        "algorithmic_bytes_per_launch": sls_bytes / n_roof,
        "algorithmic_bytes_per_item": sls_bytes_per_item(spec),
        # the kernel's share of the pipelined step: the embedding stage alone
        # through the same queue (back to back) per query / the whole
        # forward's per-query step; an isolated launch (ramp + tail exposed)
        # is longer than the pipelined per-query step
        "kernel_share_of_step": float(svc2.mean() * 1e-3) / max(step_s / Q, 1e-12),
        "isolated_launch_over_step": (sls_ms * 1e-3 / n_roof) / max(step_s / Q, 1e-12),
        "back_to_back": {"achieved": b2b, "frac": b2b / peak_hbm,
                         "method": "embedding stage only, rs_forward_many over the lanes "
                                   "(RS_MANY_POOL_ONLY), algorithmic bytes / summed delivery "
                                   "gaps; the measured peak is a read+write copy, a gather "
                                   "is read-mostly"}}
    peak_tf, tf_src = measured_tensor_peak(args.fc)
    fc_tflops = pred_flops / max(fc_ms * 1e-3, 1e-12) / 1e12
    tensor_roof = {
        "bound": "tensor", "kernel": "fc_tc_kernel (predict stack: " +
        f"{len(spec.predict_fc.dims)} layers x {spec.num_parallel_predict_stacks} stacks)"
        if args.fc != "fp32" else "fc_ffma_kernel (predict stack, FFMA)",
        "achieved": fc_tflops, "peak": peak_tf, "unit": "TFLOP/s", "frac": fc_tflops / peak_tf,
        "peak_source": tf_src, "traffic": None,
        "timing": "CUDA events recorded by graph nodes right before and after the predict "
                  "stack in the forward graph, on its stream (rs_timing.fc_ms)",
        "algorithmic_flops_per_launch": pred_flops / n_roof,
        "algorithmic_flops_per_item": rs.work(spec, 1)["PredictFC"][0],
        "kernel_share_of_step": (fc_ms * 1e-3 / n_roof) / max(step_s / Q, 1e-12)}
    want_tensor = args.roofline == "tensor" or (args.roofline == "auto" and
                                                args.workload in TENSOR_BOUND)
    roof = dict(tensor_roof if want_tensor else hbm_roof)
    roof["other"] = hbm_roof if want_tensor else tensor_roof
    if rank == 0:
        line = {
            "metric": METRIC, "value": agg["value"], "unit": "queries/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": agg["time_s"] * 1e3 / K,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"fp32": "fp32", "bf16": "fp32 SLS / bf16 FC (labelled variant)"}.get(
                args.fc, "fp32 SLS / tf32 FC"),
            "data": f"synthetic (seeded random-init tables/weights, LogNormal(ln{args.size_median:g},0.5) sizes)",
            "config": cfg,
            "method": "open-loop Poisson replay (n=50,000, sim.hpp:79) of the per-query CUDA-event "
                      "service times measured in the timed region (FIFO delivery per GPU, "
                      "in-pipeline residence added to latency, exact p95, lambda bisection to "
                      "1%, sim.cpp:246-290); whole job = N x min over ranks",
            "sla": {"p95_ms": r_dev.p95 * 1e3, "p50_ms": r_dev.p50 * 1e3,
                    "at_lambda": r_dev.at_lambda, "saturated_qps": agg["saturated_qps"],
                    "mean_service_ms": float(svc_dev.mean() * 1e3),
                    "service_capacity_qps": world / float(svc_dev.mean()),
                    "stable_load": st_dev, "queue_depth": args.depth,
                    "p95_extra_residence_ms": float(np.percentile(extra_dev, 95) * 1e3)},
            "e2e": {"value": agg_e2e["value"], "unit": "queries/s",
                    "h2d_bytes_per_step": h2d_step, "d2h_bytes_per_step": d2h_step,
                    "p95_ms": r_host.p95 * 1e3, "saturated_qps": agg_e2e["saturated_qps"],
                    "stable_load": st_host,
                    "h2d_gbs": h2d_step * K / max(t_host, 1e-9) / 1e9},
            "stages": {"items": items_roof, "forward_ms": fwd_ms, "embedding_stage_ms": emb_ms,
                       "predict_stack_ms": fc_ms,
                       "method": "RS_OPT_STAGE_TIMING forward graph, one query at a time"},
            "roofline": roof,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu:
            res, walls = cpu_deeprecsched(args, args.workload, sla, rounds=3, budget_s=4.0)
            line["cpu_baseline"] = {"value": res["qps"], "unit": "queries/s",
                                    "cores": res["threads"], "kind": "port",
                                    "sample": cpu_sample_text(res, 3)}
        print(json.dumps(line), flush=True)
    acc.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---- real-time serving over K GPUs (--serve) -------------------------------------
def run_serve(args):
    """One Poisson stream over every visible GPU, served in REAL time by the
    K-replica executor (rs_serve: the reference's single FIFO accelerator,
    proj/src/sim.cpp:95-97, 126-136, as a least-outstanding-items pool with one
    dispatcher thread per replica). QPS@p95 <= SLA is found with the
    reference's search (evaluate, geometric bisection to 1%, feasible iff the
    exact p95 of post-warm-up queries meets the SLA; sim.cpp:246-290) where each
    evaluation EXECUTES n queries instead of simulating them. Host pinned
    inputs (packed [dense | int64 indices], the reference byte model): every
    query's H2D and D2H is inside its latency. One process, replica r on GPU r."""
    import paper_2001_02772_b200 as rs
    spec, rows, zoo_name = workload_spec(rs, args.workload)
    sla = sla_for(args, zoo_name, rs.sla_target)
    K = args.gpus
    if rs.device_count() < K:
        raise SystemExit(f"--serve --gpus {K}: only {rs.device_count()} devices visible")
    fc = {"fp32": rs.FC_FP32, "tf32": rs.FC_TF32, "auto": rs.FC_AUTO, "bf16": rs.FC_BF16}[args.fc]
    reps = [rs.Accelerator(spec, rows, seed=1, device=r, max_query_size=args.max_query,
                           fc_mode=fc, queue_depth=args.depth) for r in range(K)]
    P = 2 * args.queries_per_step
    seed = rank_seed(0)
    if args.size_fixed:
        pool_sizes = np.full(P, args.size_fixed, dtype=np.int64)
    else:
        _, pool_sizes = rs.gen_trace(seed, 1000.0, rs.SizeDistribution.log_normal(
            math.log(args.size_median), 0.5), P)
    pool_sizes = np.minimum(pool_sizes, args.max_query)
    device_inputs = args.serve_inputs == "device"
    if device_inputs and K > 1:
        raise SystemExit("--serve-inputs device needs --gpus 1 (a query may go to any replica)")
    bufs, dbufs = [], []
    for q in range(P):
        dn, ix = rs.fill_query(spec, rows, seed, q, int(pool_sizes[q]))
        if device_inputs:
            import torch
            dbufs.append((torch.from_numpy(dn).cuda(0), torch.from_numpy(ix).cuda(0)))
            continue
        hb = rs.PinnedBuffer(dn.nbytes + ix.nbytes)
        raw = hb.view(np.uint8, (dn.nbytes + ix.nbytes,))
        raw[:dn.nbytes] = dn.reshape(-1).view(np.uint8)
        raw[dn.nbytes:] = ix.reshape(-1).view(np.uint8)
        bufs.append((hb, dn.nbytes))
    if device_inputs:
        import torch
        douts = [torch.empty((args.max_query, reps[0].output_dim), device="cuda:0")
                 for _ in range(16)]
    outs = [rs.PinnedBuffer(args.max_query * reps[0].output_dim * 4) for _ in range(16)]
    n = args.serve_n
    dist = rs.SizeDistribution.log_normal(math.log(args.size_median), 0.5)

    def batch_for(sizes_idx):
        sizes = [int(pool_sizes[j]) for j in sizes_idx]
        if device_inputs:
            return reps[0].batch(sizes, [dbufs[j][0].data_ptr() for j in sizes_idx],
                                 [dbufs[j][1].data_ptr() for j in sizes_idx],
                                 [douts[i % 16].data_ptr() for i in range(len(sizes_idx))],
                                 rs.MEM_DEVICE)
        return reps[0].batch(sizes, [bufs[j][0].ptr for j in sizes_idx],
                             [bufs[j][0].ptr + bufs[j][1] for j in sizes_idx],
                             [outs[i % 16].ptr for i in range(len(sizes_idx))], rs.MEM_HOST)

    pool_of = np.arange(n) % P
    prepared = batch_for(pool_of)
    warm = int(0.1 * n)
    host = None
    if args.hybrid_threshold > 0:
        if device_inputs:
            raise SystemExit("--hybrid-threshold serves host queries")
        # DeepRecSched for real: queries <= T as B-item requests on host cores
        host = rs.HostModel(spec, rows, seed=1)
        cores = args.cpu_cores or max(1, (os.cpu_count() or 2) - K - 2)
    offl = {"fraction": None}

    def run_once(arr):
        if host is None:
            return rs.serve(reps, prepared, arr)
        lat, off = rs.serve_hybrid(host, cores, args.cpu_batch, args.hybrid_threshold, reps,
                                   prepared, arr)
        offl["fraction"] = float(np.sum(off * np.array(
            [int(pool_sizes[j]) for j in pool_of])) / np.sum([int(pool_sizes[j]) for j in pool_of]))
        return lat

    def evaluate(lam, eval_idx):
        arr, _ = rs.gen_trace(seed + eval_idx, lam, dist, n)  # Poisson gaps at rate lam
        arr = arr - arr[0]
        t0 = time.time()
        lat = run_once(arr) * 1e-3
        wall = time.time() - t0
        post = lat[warm:]
        p95 = float(np.sort(post)[max(int(math.ceil(0.95 * len(post))), 1) - 1])
        p50 = float(np.sort(post)[max(int(math.ceil(0.50 * len(post))), 1) - 1])
        span = float(np.max(arr + lat) - arr[warm])
        return {"lambda": lam, "p95_ms": p95 * 1e3, "p50_ms": p50 * 1e3,
                "achieved_qps": (n - warm) / span, "wall_s": wall, "feasible": p95 <= sla}

    # warm-up, then a burst (all arrivals at t=0): the saturated throughput
    rs.serve(reps, batch_for(pool_of[:min(n, 2000)]), np.zeros(min(n, 2000)))
    t0 = time.time()
    lat = run_once(np.zeros(n))
    burst_qps = n / (float(lat.max()) * 1e-3)
    evals = []
    lo, hi = 0.5 * burst_qps, 1.5 * burst_qps
    e_lo = evaluate(lo, 0)
    evals.append(e_lo)
    best = e_lo if e_lo["feasible"] else None
    e_hi = evaluate(hi, 1)
    evals.append(e_hi)
    if e_hi["feasible"]:
        best = e_hi
    else:
        k = 2
        while hi / lo > 1.01 and best is not None:
            mid = math.sqrt(lo * hi)
            e = evaluate(mid, k)
            k += 1
            evals.append(e)
            if e["feasible"]:
                lo, best = mid, e
            else:
                hi = mid
    stable = evaluate(0.9 * burst_qps, 99)
    line = {"metric": METRIC + " (real-time serving, --serve)", "mode": "serve",
            "value": best["achieved_qps"] if best else 0.0, "unit": "queries/s", "n_gpus": K,
            "higher_is_better": True, "scaling": "weak", "dtype":
            "fp32" if args.fc == "fp32" else "fp32 SLS / tf32 FC",
            "config": {"workload": args.workload, "model": spec.name, "rows_per_table": rows,
                       "sla_s": sla, "replicas": K, "queries_per_evaluation": n,
                       "distinct_queries": P,
                       "inputs": "device-resident (read in place)" if device_inputs else
                       "host pinned, packed [dense | int64 indices] (reference byte model)",
                       "fc_path": args.fc,
                       "lanes_per_replica": args.depth},
            "qps_at_sla": {"qps": best["achieved_qps"] if best else 0.0,
                           "at_lambda": best["lambda"] if best else 0.0,
                           "p95_ms": best["p95_ms"] if best else None,
                           "p50_ms": best["p50_ms"] if best else None},
            "burst": {"qps": burst_qps, "queries": n,
                      "method": "all n arrivals at t=0: saturated real throughput"},
            "stable_load": stable, "evaluations": evals,
            "hybrid": None if host is None else {
                "threshold": args.hybrid_threshold, "cpu_batch": args.cpu_batch,
                "cpu_cores": cores, "offloaded_item_fraction": offl["fraction"],
                "rule": "S > T whole to the least-loaded replica, else floor(S/B) x B + S mod B "
                        "requests on host worker threads (rs_serve_hybrid, sim.cpp:173-191)"},
            "method": "rs_serve real-time executor: host clock releases, least-outstanding-"
                      "items routing, one dispatcher thread per replica, CUDA-event "
                      "completions; reference search rule (sim.cpp:246-290) over real runs"}
    print(json.dumps(line), flush=True)
    for r in reps:
        r.close()
    if host is not None:
        host.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="cfg3-rmc2",
                    help="cfg3-rmc2 (default) | cfg3-rmc3 | cfg1-rmc1 | cfg5-dien | cfg5-din | "
                         "ncf | wnd | mt-wnd | rmc1 | rmc2 | rmc3 | din | dien")
    ap.add_argument("--sla", type=float, default=0.0, help="override SLA seconds")
    ap.add_argument("--queries-per-step", type=int, default=256)
    ap.add_argument("--pack", type=int, default=1,
                    help="1: each host query in one pinned buffer [dense | indices]")
    ap.add_argument("--size-median", type=float, default=300.0,
                    help="LogNormal(ln m, 0.5) query sizes (SURVEY 8d: 300; 30 = small-query regime)")
    ap.add_argument("--size-fixed", type=int, default=0,
                    help=">0: every query has this many items (BASELINE configs[3] batch sweep)")
    ap.add_argument("--cta-pairs", choices=["auto", "on", "off"], default="auto",
                    help="RS_OPT_CTA_PAIRS (256-row CTA-pair FC tiles); auto = on for "
                         "--size-fixed queues (uniform sizes), off for mixed streams")
    ap.add_argument("--merge", type=int, default=1,
                    help=">1 = labelled query-merging variant (SURVEY 8f-3)")
    ap.add_argument("--dense-bits", type=int, choices=[32, 16], default=32,
                    help="16 = labelled bf16 dense-feature input variant (SURVEY 8f-2)")
    ap.add_argument("--index-bits", type=int, choices=[64, 32], default=64,
                    help="32 = labelled int32-index input variant (SURVEY 8f-2)")
    ap.add_argument("--zipf", type=float, default=0.0,
                    help=">0 = labelled skewed-index variant (SURVEY 8d Zipf(1.05))")
    ap.add_argument("--l2-persist-mb", type=int, default=0,
                    help="hot-row block kept in the L2 persisting set-aside (MiB)")
    ap.add_argument("--max-query", type=int, default=1000)
    ap.add_argument("--fc", choices=["fp32", "tf32", "auto", "bf16"], default="auto",
                    help="bf16 = labelled lower-precision variant (bf16 weights/activations)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--depth", type=int, default=16,
                    help="queries in flight per GPU (lanes): 16 = 8 within 0.4% on cfg3, 2-26% faster for small queries (DESIGN.md §5a)")
    ap.add_argument("--rnn", choices=["gru", "augru"], default="gru",
                    help="AttentionRNN cell (DIEN): AUGRU = the explicit extension of SURVEY D3")
    ap.add_argument("--roofline", choices=["auto", "hbm", "tensor"], default="auto",
                    help="which kernel the roofline object reports (auto: tensor for "
                         "mt-wnd/wnd, else the embedding kernel)")
    ap.add_argument("--serve", action="store_true",
                    help="real-time serving over --gpus replicas in one process (rs_serve)")
    ap.add_argument("--serve-inputs", choices=["host", "device"], default="host",
                    help="--serve: host pinned inputs (e2e) or device-resident (--gpus 1)")
    ap.add_argument("--hybrid-threshold", type=int, default=0,
                    help="--serve: >0 = DeepRecSched hybrid, queries of <= T items on host cores")
    ap.add_argument("--cpu-batch", type=int, default=4,
                    help="--serve --hybrid-threshold: CPU request size B")
    ap.add_argument("--cpu-cores", type=int, default=0,
                    help="--serve --hybrid-threshold: host worker threads (0: nproc - K - 2)")
    ap.add_argument("--serve-n", type=int, default=50_000,
                    help="--serve: queries per evaluation (reference n = 50,000)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.serve:
        run_serve(args)
        return
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
