// Reference-side integration adapter (built into oracle/_ref/librecsim_ref_b200.so
// together with the UNMODIFIED reference sources).
//
// The reference prices every offloaded query with the pure cost function
//   recsim::accel_service_time(const ModelSpec&, int64_t, const AcceleratorSpec&)
//   (/root/reference/proj/include/recsim/platform.hpp:83-84,
//    /root/reference/proj/src/platform.cpp:113-136)
// which simulate()'s accel_time memo (proj/src/sim.cpp:81-88) and tune()'s
// phase-2 gate (proj/src/autotune.cpp:167-168) call. This file is linked with
//   -Wl,--wrap=_ZN6recsim18accel_service_timeERKNS_9ModelSpecElRKNS_15AcceleratorSpecE
// so those call sites reach __wrap_... below: for an AcceleratorSpec named
// "b200" the service time is MEASURED on the GPU through the C-ABI
// (rs_service_time: H2D + forward + D2H of a synthetic query of that size,
// memoised per size), every other spec falls through to the original model.
// Nothing in the reference is edited; the same three-line hook is what a
// maintainer would add inside accel_service_time itself.
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../include/rs_accel.h"
#include "recsim/loadgen.hpp"
#include "recsim/model_zoo.hpp"
#include "recsim/platform.hpp"
#include "recsim/sim.hpp"

using recsim::AcceleratorSpec;
using recsim::ModelSpec;
using recsim::ServiceTime;

#define RS_WRAPPED _ZN6recsim18accel_service_timeERKNS_9ModelSpecElRKNS_15AcceleratorSpecE
#define RS_CAT2(a, b) a##b
#define RS_CAT(a, b) RS_CAT2(a, b)

extern "C" ServiceTime RS_CAT(__real_, RS_WRAPPED)(const ModelSpec&, std::int64_t,
                                                    const AcceleratorSpec&);

namespace {

std::mutex g_mu;
// one replica per distinct model SHAPE (not per name: two inline specs may
// share a name), on the device and with the row count the environment names
std::map<std::string, rs_accel*> g_accels;

rs_model_desc to_desc(const ModelSpec& s) {
  rs_model_desc d{};
  std::strncpy(d.name, s.name.c_str(), RS_NAME_LEN - 1);
  d.has_dense_fc = s.dense_fc ? 1 : 0;
  if (s.dense_fc) {
    d.dense_fc.n = static_cast<int32_t>(s.dense_fc->dims.size());
    for (size_t i = 0; i < s.dense_fc->dims.size(); ++i) d.dense_fc.dims[i] = s.dense_fc->dims[i];
  }
  d.predict_fc.n = static_cast<int32_t>(s.predict_fc.dims.size());
  for (size_t i = 0; i < s.predict_fc.dims.size(); ++i) d.predict_fc.dims[i] = s.predict_fc.dims[i];
  d.num_parallel_predict_stacks = s.num_parallel_predict_stacks;
  d.num_tables = s.embeddings.num_tables;
  d.lookups_per_table = s.embeddings.lookups_per_table;
  d.embedding_dim = s.embeddings.embedding_dim;
  d.pooling = static_cast<int32_t>(s.embeddings.pooling);
  d.dense_input_dim = s.dense_input_dim;
  d.recurrent_hidden_dim = s.recurrent_hidden_dim ? *s.recurrent_hidden_dim : 0;
  return d;
}

// The full operator shape as the cache key (every ModelSpec field).
std::string shape_key(const rs_model_desc& d) {
  std::string k = d.name;
  auto add = [&](int64_t v) { k += ':' + std::to_string(v); };
  add(d.has_dense_fc);
  for (int i = 0; i < d.dense_fc.n; ++i) add(d.dense_fc.dims[i]);
  k += '|';
  for (int i = 0; i < d.predict_fc.n; ++i) add(d.predict_fc.dims[i]);
  k += '|';
  add(d.num_parallel_predict_stacks); add(d.num_tables); add(d.lookups_per_table);
  add(d.embedding_dim); add(d.pooling); add(d.dense_input_dim); add(d.recurrent_hidden_dim);
  return k;
}

// RS_E_* -> the exception type the reference itself throws for that failure
// (SURVEY §8b "Errors"), so CHECK_THROWS_AS-style callers keep working.
[[noreturn]] void rethrow(int rc, const char* where) {
  const std::string msg = std::string(where) + ": " + rs_last_error();
  switch (rc) {
    case RS_E_INVALID: throw std::invalid_argument(msg);     // platform.cpp:115, :65-69
    case RS_E_UNKNOWN_MODEL: throw recsim::UnknownModel(msg);  // model_zoo.hpp:15-18
    case RS_E_CONFIG: throw recsim::ConfigError(msg);          // sim.hpp:15-17
    case RS_E_DISTRIBUTION: throw recsim::InvalidDistribution(msg);  // loadgen.hpp:12-14
    case RS_E_EMPTY: throw recsim::EmptyResult(msg);           // sim.hpp:19-21
    case RS_E_CAPACITY: throw std::invalid_argument(msg);      // query_size out of range
    default: throw std::runtime_error(msg);  // device / CUDA failures: no reference analogue
  }
}

rs_accel* accel_for(const ModelSpec& m) {
  const rs_model_desc d = to_desc(m);
  const std::string key = shape_key(d);
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_accels.find(key);
  if (it != g_accels.end()) return it->second;
  const char* rows = std::getenv("RS_B200_ROWS");
  const char* dev = std::getenv("RS_B200_DEVICE");
  rs_init_desc init{};
  init.seed = 1;
  init.rows_per_table = rows ? std::atoll(rows) : 1000000;
  init.max_query_size = 1000;  // the reference's size-distribution cap (sim.hpp:78)
  init.fc_mode = RS_FC_AUTO;
  rs_accel* a = nullptr;
  const int rc = rs_accel_create(&d, &init, dev ? std::atoi(dev) : 0, &a);
  if (rc != RS_OK) rethrow(rc, "rs_accel_create");
  g_accels[key] = a;
  return a;
}

}  // namespace

extern "C" ServiceTime RS_CAT(__wrap_, RS_WRAPPED)(const ModelSpec& model, std::int64_t query_size,
                                                    const AcceleratorSpec& spec) {
  if (spec.name != "b200") return RS_CAT(__real_, RS_WRAPPED)(model, query_size, spec);
  if (query_size < 1) throw std::invalid_argument("query_size < 1");
  // memoised per (shape, S) like simulate()'s accel_time cache (sim.cpp:81-88)
  static std::map<std::pair<std::string, std::int64_t>, ServiceTime> memo;
  rs_accel* a = accel_for(model);
  const auto key = std::make_pair(shape_key(to_desc(model)), query_size);
  {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  // the whole measured ServiceTime: total (H2D + forward + D2H), transfer
  // (H2D + D2H) and the compute time split over the operator categories from
  // measured stage times (rs_service_breakdown)
  ServiceTime st;
  double per[RS_NUM_OP_CATEGORIES] = {};
  const int rc = rs_service_breakdown(a, query_size, &st.total, &st.transfer, per);
  if (rc != RS_OK) rethrow(rc, "rs_service_breakdown");
  for (int c = 0; c < RS_NUM_OP_CATEGORIES; ++c) st.per_category[c] = per[c];
  std::lock_guard<std::mutex> lock(g_mu);
  memo[key] = st;
  return st;
}

// B200 accelerator spec for the reference's AcceleratorSpec::validate
// (platform.cpp:65-69 needs positive fields; only the name is consulted).
extern "C" void ref_b200_release() {
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto& kv : g_accels) rs_accel_destroy(kv.second);
  g_accels.clear();
}
