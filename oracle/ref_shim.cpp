// ORACLE — TEST INFRASTRUCTURE ONLY. A C shim over the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/librecsim_ref.so). It exposes exactly the reference behaviour
// the hot path must reproduce:
//   gen_trace            proj/src/loadgen.cpp:106-125
//   work                 proj/src/model_zoo.cpp:177-245
//   accel_input_bytes /
//   accel_service_time   proj/src/platform.cpp:105-136
//   simulate + EventLogger (Dispatch / AccelStart records)  proj/src/sim.cpp:69-205
//   sla_target           proj/src/autotune.cpp:73-88
//   builtin_model        proj/src/model_zoo.cpp:141-170
#include <cstdint>
#include <cstring>
#include <exception>

#include "oracle.h"
#include "recsim/autotune.hpp"
#include "recsim/loadgen.hpp"
#include "recsim/model_zoo.hpp"
#include "recsim/platform.hpp"
#include "recsim/sim.hpp"

using namespace recsim;

namespace {

ModelSpec to_spec(const or_model& m) {
  ModelSpec s;
  s.name = m.name;
  if (m.has_dense_fc) {
    LayerStack d;
    for (int i = 0; i < m.dense_fc.n; ++i) d.dims.push_back(m.dense_fc.dims[i]);
    s.dense_fc = d;
  }
  for (int i = 0; i < m.predict_fc.n; ++i) s.predict_fc.dims.push_back(m.predict_fc.dims[i]);
  s.num_parallel_predict_stacks = m.stacks;
  s.embeddings.num_tables = m.T;
  s.embeddings.lookups_per_table = m.L;
  s.embeddings.embedding_dim = m.D;
  s.embeddings.pooling = static_cast<Pooling>(m.pooling);
  s.dense_input_dim = m.dense_in;
  if (m.hidden > 0) s.recurrent_hidden_dim = m.hidden;
  return s;
}

void from_spec(const ModelSpec& s, or_model* m) {
  std::memset(m, 0, sizeof(*m));
  std::strncpy(m->name, s.name.c_str(), sizeof(m->name) - 1);
  m->has_dense_fc = s.dense_fc ? 1 : 0;
  if (s.dense_fc) {
    m->dense_fc.n = (int32_t)s.dense_fc->dims.size();
    for (size_t i = 0; i < s.dense_fc->dims.size(); ++i) m->dense_fc.dims[i] = s.dense_fc->dims[i];
  }
  m->predict_fc.n = (int32_t)s.predict_fc.dims.size();
  for (size_t i = 0; i < s.predict_fc.dims.size(); ++i) m->predict_fc.dims[i] = s.predict_fc.dims[i];
  m->stacks = s.num_parallel_predict_stacks;
  m->T = s.embeddings.num_tables;
  m->L = s.embeddings.lookups_per_table;
  m->D = s.embeddings.embedding_dim;
  m->pooling = static_cast<int32_t>(s.embeddings.pooling);
  m->dense_in = s.dense_input_dim;
  m->hidden = s.recurrent_hidden_dim ? *s.recurrent_hidden_dim : 0;
}

SizeDistribution make_dist(int kind, double p0, double p1, double p2, double p3, int64_t max_size) {
  SizeDistribution d;
  d.kind = static_cast<SizeDistribution::Kind>(kind);
  d.p0 = p0; d.p1 = p1; d.p2 = p2; d.p3 = p3;
  d.max_size = max_size;
  return d;
}

// "measured": the box's own cores, priced by the measured per-request table of
// oracle/ref_cpu_adapter.cpp (linked only into librecsim_ref_cpu.so; weak here).
extern "C" __attribute__((weak)) int64_t ref_measured_cores(void);

CpuPlatformSpec shim_cpu(const char* name) {
  if (std::strcmp(name, "measured") == 0 && ref_measured_cores) {
    CpuPlatformSpec p = builtin_cpu("skylake");  // fields other than cores unused
    p.name = "measured";
    p.cores = ref_measured_cores();
    return p;
  }
  return builtin_cpu(name);
}

// 0 ok, -1 invalid_argument, -2 UnknownModel, -3 ConfigError, -4 InvalidDistribution,
// -5 InfeasibleSLA (tune(): no batch size meets the SLA)
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const UnknownModel&) {
    return -2;
  } catch (const ConfigError&) {
    return -3;
  } catch (const InvalidDistribution&) {
    return -4;
  } catch (const InfeasibleSLA&) {
    return -5;
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (...) {
    return -99;
  }
}

}  // namespace

extern "C" {

int ref_builtin_model(const char* name, or_model* out) {
  return guard([&] { from_spec(builtin_model(name), out); });
}

int ref_validate(const or_model* m) { return guard([&] { to_spec(*m).validate(); }); }

int ref_work(const or_model* m, int64_t batch, double* flops, double* bytes, double* gather) {
  return guard([&] {
    WorkBreakdown wb = work(to_spec(*m), batch);
    for (int c = 0; c < kNumOpCategories; ++c) {
      flops[c] = wb.per_category[c].flops;
      bytes[c] = wb.per_category[c].bytes;
    }
    *gather = wb.gather_stream;
  });
}

int ref_accel_input_bytes(const or_model* m, int64_t S, double* out) {
  return guard([&] { *out = accel_input_bytes(to_spec(*m), S); });
}

int ref_accel_service_time_default(const or_model* m, int64_t S, double* total, double* transfer) {
  return guard([&] {
    ServiceTime st = accel_service_time(to_spec(*m), S, builtin_accel("default"));
    *total = st.total;
    *transfer = st.transfer;
  });
}

int ref_sla_target(const char* model, const char* level, double* out) {
  return guard([&] { *out = sla_target(model, level); });
}

int ref_gen_trace(uint64_t seed, double lambda, int kind, double p0, double p1, double p2,
                  double p3, int64_t max_size, int64_t n, double* arrivals, int64_t* sizes) {
  return guard([&] {
    QueryTrace t = gen_trace(seed, lambda, make_dist(kind, p0, p1, p2, p3, max_size), n);
    for (int64_t i = 0; i < n; ++i) {
      arrivals[i] = t.records[(size_t)i].arrival_time;
      sizes[i] = t.records[(size_t)i].size;
    }
  });
}

// Runs the reference simulate() on a gen_trace stream and records every
// Dispatch (kind 1) and AccelStart (kind 3) event as (kind, query, items).
// threshold <= 0 means CPU-only. Returns the number of records in *count.
int ref_simulate_decisions(const or_model* m, const char* cpu, uint64_t seed, double lambda,
                           int kind, double p0, double p1, double p2, double p3,
                           int64_t max_size, int64_t n, int64_t batch, int64_t threshold,
                           int32_t* ev_kind, int64_t* ev_query, int64_t* ev_items,
                           int64_t cap, int64_t* count, double* p95) {
  return guard([&] {
    SchedulerConfig cfg;
    cfg.batch_size = batch;
    cfg.model = to_spec(*m);
    cfg.cpu = shim_cpu(cpu);
    cfg.warmup_fraction = 0.0;
    if (threshold > 0) {
      cfg.offload_threshold = threshold;
      cfg.accel = builtin_accel("default");
    }
    QueryTrace t = gen_trace(seed, lambda, make_dist(kind, p0, p1, p2, p3, max_size), n);
    int64_t k = 0;
    auto logger = [&](const SimEvent& e) {
      if (e.kind != SimEvent::Kind::Dispatch && e.kind != SimEvent::Kind::AccelStart) return;
      if (k < cap) {
        ev_kind[k] = static_cast<int32_t>(e.kind);
        ev_query[k] = e.query;
        ev_items[k] = e.items;
      }
      ++k;
    };
    SimResult r = simulate(t, cfg, logger);
    *count = k;
    if (p95) *p95 = summarize(r).p95;
  });
}

// Reference max_qps_under_sla for a zoo model on a named CPU (with the
// default modeled accelerator when threshold > 0).
int ref_max_qps(const or_model* m, const char* cpu, double sla, uint64_t seed, int kind,
                double p0, double p1, double p2, double p3, int64_t max_size, int64_t n,
                int64_t batch, int64_t threshold, double* qps, double* p95) {
  return guard([&] {
    SchedulerConfig cfg;
    cfg.batch_size = batch;
    cfg.model = to_spec(*m);
    cfg.cpu = shim_cpu(cpu);
    if (threshold > 0) {
      cfg.offload_threshold = threshold;
      cfg.accel = builtin_accel("default");
    }
    TraceGenParams gen;
    gen.base_seed = seed;
    gen.dist = make_dist(kind, p0, p1, p2, p3, max_size);
    gen.n = n;
    QpsResult r = max_qps_under_sla(cfg, sla, gen);
    *qps = r.qps;
    *p95 = r.p95;
  });
}

// Accelerator by name: "default" = the reference's modeled 1080Ti-class spec
// (platform.cpp:174-183); "b200" = the same positive placeholder fields with
// the name the integration adapter (ref_b200_adapter.cpp) routes to the GPU.
static AcceleratorSpec named_accel(const char* name) {
  AcceleratorSpec a = builtin_accel("default");
  if (std::strcmp(name, "default") != 0) a.name = name;
  return a;
}

// accel_service_time (platform.cpp:113-136) on a named accelerator: the whole
// ServiceTime (total, transfer, per-category) — through the B200 adapter for
// "b200" in librecsim_ref_b200.so. Exceptions map to the guard() codes.
int ref_accel_service_time_named(const or_model* m, const char* accel, int64_t S, double* total,
                                 double* transfer, double* per_category) {
  return guard([&] {
    ServiceTime st = accel_service_time(to_spec(*m), S, named_accel(accel));
    *total = st.total;
    *transfer = st.transfer;
    for (int c = 0; c < kNumOpCategories; ++c) per_category[c] = st.per_category[c];
  });
}

// max_qps_under_sla (sim.cpp:246-290) with a named accelerator at threshold T.
int ref_max_qps_accel(const or_model* m, const char* cpu, const char* accel, double sla,
                      uint64_t seed, int kind, double p0, double p1, double p2, double p3,
                      int64_t max_size, int64_t n, int64_t batch, int64_t threshold,
                      double* qps, double* p95, double* frac) {
  return guard([&] {
    SchedulerConfig cfg;
    cfg.batch_size = batch;
    cfg.model = to_spec(*m);
    cfg.cpu = shim_cpu(cpu);
    if (threshold > 0) {
      cfg.offload_threshold = threshold;
      cfg.accel = named_accel(accel);
    }
    TraceGenParams gen;
    gen.base_seed = seed;
    gen.dist = make_dist(kind, p0, p1, p2, p3, max_size);
    gen.n = n;
    QpsResult r = max_qps_under_sla(cfg, sla, gen);
    *qps = r.qps;
    *p95 = r.p95;
    *frac = r.accel_work_fraction;
  });
}

// tune() phase 2's inner loop made explicit (autotune.cpp:159-212): QPS@p95
// of max_qps_under_sla at a fixed batch B for each offload threshold T in
// thresholds[0..n) (T <= 0: CPU only). Out: qps[i], p95[i], accel_fraction[i].
int ref_sweep_threshold(const or_model* m, const char* cpu, const char* accel, double sla,
                        uint64_t seed, int kind, double p0, double p1, double p2, double p3,
                        int64_t max_size, int64_t n, int64_t batch, const int64_t* thresholds,
                        int64_t n_t, double* qps, double* p95, double* frac) {
  return guard([&] {
    for (int64_t i = 0; i < n_t; ++i) {
      SchedulerConfig cfg;
      cfg.batch_size = batch;
      cfg.model = to_spec(*m);
      cfg.cpu = shim_cpu(cpu);
      if (thresholds[i] > 0) {
        cfg.offload_threshold = thresholds[i];
        cfg.accel = named_accel(accel);
      }
      TraceGenParams gen;
      gen.base_seed = seed;
      gen.dist = make_dist(kind, p0, p1, p2, p3, max_size);
      gen.n = n;
      QpsResult r = max_qps_under_sla(cfg, sla, gen);
      qps[i] = r.qps;
      p95[i] = r.p95;
      frac[i] = r.accel_work_fraction;
    }
  });
}

// DeepRecSched tune() (autotune.cpp:90-217) with a named accelerator ("" = CPU only).
int ref_tune(const or_model* m, const char* cpu, const char* accel, double sla, uint64_t seed,
             int kind, double p0, double p1, double p2, double p3, int64_t max_size, int64_t n,
             int seeds, int64_t* batch, int64_t* threshold, double* qps, double* p95,
             double* frac, int64_t* steps) {
  return guard([&] {
    TuneParams tp;
    tp.gen.base_seed = seed;
    tp.gen.dist = make_dist(kind, p0, p1, p2, p3, max_size);
    tp.gen.n = n;
    tp.seeds_to_average = seeds;
    std::optional<AcceleratorSpec> a;
    if (accel && accel[0]) a = named_accel(accel);
    TunedConfig t = tune(to_spec(*m), shim_cpu(cpu), a, sla, tp);
    *batch = t.batch_size;
    *threshold = t.offload_threshold ? *t.offload_threshold : 0;
    *qps = t.qps;
    *p95 = t.p95;
    *frac = t.accel_work_fraction;
    *steps = static_cast<int64_t>(t.search_path.size());
  });
}

}  // extern "C"
