// model.cpp — host mirror of the reference operator API: the eight zoo
// archetypes, ModelSpec validation, per-category work accounting and the
// accelerator input byte model.
//
//   builtin_model      proj/src/model_zoo.cpp:141-170
//   ModelSpec::validate proj/src/model_zoo.cpp:41-59
//   predict_input_dim  proj/src/model_zoo.cpp:113-137
//   work / fc_flops    proj/src/model_zoo.cpp:95-110, 177-245
//   accel_input_bytes  proj/src/platform.cpp:105-111
//   sla_target         proj/src/autotune.cpp:73-88
//
// The reference's arithmetic is in double over integer counts; this file
// keeps that so tests can compare accounting bit-for-bit against the
// compiled reference (tests/test_accounting.py).
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "internal.hpp"

namespace rs {
namespace {

constexpr double kElemBytes = 4.0;  // fp32 activations / embeddings

struct ZooEntry {
  const char* name;
  std::vector<int64_t> dense;    // empty = no dense stack
  std::vector<int64_t> predict;
  int64_t stacks, tables, lookups;
  int32_t pooling;
  int64_t dense_in, hidden;      // hidden 0 = none
};

// The zoo fixes D = 32 for every archetype (model_zoo.cpp:87).
const std::vector<ZooEntry>& zoo() {
  static const std::vector<ZooEntry> z = {
      {"NCF", {}, {256, 256, 128}, 1, 4, 1, RS_POOL_CONCAT, 0, 0},
      {"WND", {}, {1024, 512, 256}, 1, 20, 1, RS_POOL_CONCAT, 1000, 0},
      {"MT-WND", {}, {1024, 512, 256}, 4, 20, 1, RS_POOL_CONCAT, 1000, 0},
      {"DLRM-RMC1", {256, 128, 32}, {256, 64, 1}, 1, 10, 80, RS_POOL_SUM, 256, 0},
      {"DLRM-RMC2", {256, 128, 32}, {512, 128, 1}, 1, 40, 80, RS_POOL_SUM, 256, 0},
      {"DLRM-RMC3", {2560, 512, 32}, {512, 128, 1}, 1, 10, 20, RS_POOL_SUM, 256, 0},
      {"DIN", {}, {200, 80, 2}, 1, 20, 200, RS_POOL_ATTENTION_FC, 0, 0},
      {"DIEN", {}, {200, 80, 2}, 1, 20, 20, RS_POOL_ATTENTION_RNN, 0, 64},
  };
  return z;
}

rs_layer_stack to_stack(const std::vector<int64_t>& dims) {
  rs_layer_stack s{};
  s.n = static_cast<int32_t>(dims.size());
  for (size_t i = 0; i < dims.size(); ++i) s.dims[i] = dims[i];
  return s;
}

void check_stack(const rs_layer_stack& s, const char* what) {
  if (s.n < 1) raise(RS_E_INVALID, std::string(what) + ": empty layer stack");
  if (s.n > RS_MAX_LAYERS) raise(RS_E_INVALID, std::string(what) + ": too many layers");
  for (int i = 0; i < s.n; ++i)
    if (s.dims[i] < 1) raise(RS_E_INVALID, std::string(what) + ": layer width < 1");
}

// Sum over the stack of 2 * d_in * d_out for one item.
double chain_flops(int64_t in, const rs_layer_stack& s) {
  double f = 0;
  for (int i = 0; i < s.n; ++i) {
    f += 2.0 * static_cast<double>(in) * static_cast<double>(s.dims[i]);
    in = s.dims[i];
  }
  return f;
}

// Input plus every layer output, in bytes, for one item.
double chain_bytes(int64_t in, const rs_layer_stack& s) {
  double elems = static_cast<double>(in);
  for (int i = 0; i < s.n; ++i) elems += static_cast<double>(s.dims[i]);
  return elems * kElemBytes;
}

}  // namespace

void validate_model(const rs_model_desc& m) {
  check_stack(m.predict_fc, "predict_fc");
  if (m.has_dense_fc) check_stack(m.dense_fc, "dense_fc");
  if (m.num_parallel_predict_stacks < 1)
    raise(RS_E_INVALID, "num_parallel_predict_stacks < 1");
  if (m.num_tables < 0) raise(RS_E_INVALID, "num_tables < 0");
  if (m.num_tables > 0 && m.lookups_per_table < 1)
    raise(RS_E_INVALID, "lookups_per_table < 1");
  if (m.num_tables > 0 && (m.embedding_dim < 8 || m.embedding_dim > 256))
    raise(RS_E_INVALID, "embedding_dim outside [8, 256]");
  if (m.pooling < RS_POOL_SUM || m.pooling > RS_POOL_ATTENTION_RNN)
    raise(RS_E_INVALID, "unknown pooling");
  if (m.pooling == RS_POOL_ATTENTION_RNN && m.recurrent_hidden_dim <= 0)
    raise(RS_E_INVALID, "AttentionRNN requires recurrent_hidden_dim");
  if (m.dense_input_dim < 0) raise(RS_E_INVALID, "dense_input_dim < 0");
}

int64_t dense_out_dim(const rs_model_desc& m) {
  return m.has_dense_fc ? m.dense_fc.dims[m.dense_fc.n - 1] : m.dense_input_dim;
}

int64_t sparse_out_dim(const rs_model_desc& m) {
  switch (m.pooling) {
    case RS_POOL_SUM: return m.embedding_dim;  // one summed vector (D9)
    case RS_POOL_CONCAT: return m.num_tables * m.lookups_per_table * m.embedding_dim;
    case RS_POOL_ATTENTION_FC: return m.num_tables * m.embedding_dim;
    case RS_POOL_ATTENTION_RNN: return m.num_tables * m.recurrent_hidden_dim;
  }
  return 0;
}

int64_t interaction_pairs(const rs_model_desc& m) {
  if (m.pooling != RS_POOL_SUM || !m.has_dense_fc) return 0;
  const int64_t v = m.num_tables + 1;  // pooled tables plus the dense vector
  return v * (v - 1) / 2;
}

int64_t predict_input_dim(const rs_model_desc& m) {
  const int64_t w = dense_out_dim(m) + sparse_out_dim(m) + interaction_pairs(m);
  return w < 1 ? 1 : w;
}

rs_work_breakdown work(const rs_model_desc& m, int64_t batch) {
  if (batch < 1) raise(RS_E_INVALID, "batch < 1");
  rs_work_breakdown wb{};
  const double b = static_cast<double>(batch);
  const double D = static_cast<double>(m.embedding_dim);
  const double T = static_cast<double>(m.num_tables);
  const double L = static_cast<double>(m.lookups_per_table);

  if (m.has_dense_fc) {
    wb.flops[RS_OP_DENSE_FC] = b * chain_flops(m.dense_input_dim, m.dense_fc);
    wb.bytes[RS_OP_DENSE_FC] = b * chain_bytes(m.dense_input_dim, m.dense_fc);
  }
  if (m.num_tables > 0) {
    wb.gather_stream = b * L;
    wb.bytes[RS_OP_EMBEDDING_LOOKUP] = b * T * L * D * kElemBytes;
    switch (m.pooling) {
      case RS_POOL_SUM:
        wb.flops[RS_OP_POOLING] = b * T * L * D;
        wb.bytes[RS_OP_POOLING] = b * T * D * kElemBytes;
        break;
      case RS_POOL_CONCAT:
        wb.bytes[RS_OP_POOLING] = b * T * L * D * kElemBytes;
        break;
      case RS_POOL_ATTENTION_FC:
        wb.flops[RS_OP_ATTENTION] = b * T * L * 2.0 * D * D;
        wb.bytes[RS_OP_ATTENTION] = b * T * L * kElemBytes;
        wb.flops[RS_OP_POOLING] = 2.0 * b * T * L * D;
        wb.bytes[RS_OP_POOLING] = b * T * D * kElemBytes;
        break;
      case RS_POOL_ATTENTION_RNN: {
        const double h = static_cast<double>(m.recurrent_hidden_dim);
        wb.flops[RS_OP_RECURRENT] = b * T * L * 3.0 * 2.0 * h * h;
        wb.bytes[RS_OP_RECURRENT] = b * T * L * h * kElemBytes;
        wb.flops[RS_OP_POOLING] = 2.0 * b * T * L * D;
        wb.bytes[RS_OP_POOLING] = b * T * h * kElemBytes;
        break;
      }
    }
  }
  if (m.pooling == RS_POOL_SUM && m.has_dense_fc && m.num_tables > 0) {
    const double v = T + 1.0;
    const double pairs = v * (v - 1.0) / 2.0;
    wb.flops[RS_OP_INTERACTION] = 2.0 * b * pairs * D;
    wb.bytes[RS_OP_INTERACTION] = b * pairs * kElemBytes;
  }
  const int64_t p_in = predict_input_dim(m);
  const double N = static_cast<double>(m.num_parallel_predict_stacks);
  wb.flops[RS_OP_PREDICT_FC] = b * N * chain_flops(p_in, m.predict_fc);
  wb.bytes[RS_OP_PREDICT_FC] = b * N * chain_bytes(p_in, m.predict_fc);
  return wb;
}

double accel_input_bytes(const rs_model_desc& m, int64_t query_size) {
  const double per_item = static_cast<double>(m.dense_input_dim) * 4.0 +
                          static_cast<double>(m.num_tables) *
                              static_cast<double>(m.lookups_per_table) * 8.0;
  return per_item * static_cast<double>(query_size);
}

}  // namespace rs

// ---- C-ABI ---------------------------------------------------------------
using namespace rs;

extern "C" int rs_model_builtin(const char* name, rs_model_desc* out) {
  return guarded([&] {
    if (!name || !out) raise(RS_E_INVALID, "null argument");
    for (const auto& z : zoo()) {
      if (std::strcmp(z.name, name) != 0) continue;
      rs_model_desc m{};
      std::strncpy(m.name, z.name, RS_NAME_LEN - 1);
      m.has_dense_fc = z.dense.empty() ? 0 : 1;
      m.dense_fc = to_stack(z.dense);
      m.predict_fc = to_stack(z.predict);
      m.num_parallel_predict_stacks = z.stacks;
      m.num_tables = z.tables;
      m.lookups_per_table = z.lookups;
      m.embedding_dim = 32;
      m.pooling = z.pooling;
      m.dense_input_dim = z.dense_in;
      m.recurrent_hidden_dim = z.hidden;
      validate_model(m);
      *out = m;
      return;
    }
    raise(RS_E_UNKNOWN_MODEL, std::string("unknown model: ") + name);
  });
}

extern "C" int rs_zoo_names(const char** names, int cap, int* count) {
  return guarded([&] {
    const auto& z = zoo();
    if (count) *count = static_cast<int>(z.size());
    for (int i = 0; names && i < cap && i < static_cast<int>(z.size()); ++i)
      names[i] = z[i].name;
  });
}

extern "C" int rs_model_validate(const rs_model_desc* m) {
  return guarded([&] {
    if (!m) raise(RS_E_INVALID, "null model");
    validate_model(*m);
  });
}

extern "C" int rs_work(const rs_model_desc* m, int64_t batch, rs_work_breakdown* out) {
  return guarded([&] {
    if (!m || !out) raise(RS_E_INVALID, "null argument");
    *out = work(*m, batch);
  });
}

extern "C" int rs_predict_input_dim(const rs_model_desc* m, int64_t* out) {
  return guarded([&] {
    if (!m || !out) raise(RS_E_INVALID, "null argument");
    *out = predict_input_dim(*m);
  });
}

extern "C" int rs_accel_input_bytes(const rs_model_desc* m, int64_t query_size,
                                    double* out) {
  return guarded([&] {
    if (!m || !out) raise(RS_E_INVALID, "null argument");
    *out = accel_input_bytes(*m, query_size);
  });
}

extern "C" int rs_sla_target(const char* model_name, const char* level, double* out) {
  return guarded([&] {
    if (!model_name || !level || !out) raise(RS_E_INVALID, "null argument");
    static const struct { const char* name; double medium; } kSla[] = {
        {"DLRM-RMC1", 0.100}, {"DLRM-RMC2", 0.400}, {"DLRM-RMC3", 0.100},
        {"NCF", 0.005},       {"WND", 0.025},       {"MT-WND", 0.025},
        {"DIN", 0.100},       {"DIEN", 0.035}};
    double medium = -1;
    for (const auto& s : kSla)
      if (std::strcmp(s.name, model_name) == 0) medium = s.medium;
    if (medium < 0) raise(RS_E_UNKNOWN_MODEL, std::string("unknown model: ") + model_name);
    if (std::strcmp(level, "low") == 0) *out = 0.5 * medium;
    else if (std::strcmp(level, "medium") == 0) *out = medium;
    else if (std::strcmp(level, "high") == 0) *out = 1.5 * medium;
    else raise(RS_E_INVALID, std::string("unknown SLA level: ") + level);
  });
}
