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
#include "recsim/platform.hpp"

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

rs_accel* accel_for(const ModelSpec& m) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_accels.find(m.name);
  if (it != g_accels.end()) return it->second;
  const char* rows = std::getenv("RS_B200_ROWS");
  rs_init_desc init{};
  init.seed = 1;
  init.rows_per_table = rows ? std::atoll(rows) : 1000000;
  init.max_query_size = 1000;
  init.fc_mode = RS_FC_AUTO;
  rs_model_desc d = to_desc(m);
  rs_accel* a = nullptr;
  if (rs_accel_create(&d, &init, 0, &a) != RS_OK)
    throw std::runtime_error(std::string("rs_accel_create: ") + rs_last_error());
  g_accels[m.name] = a;
  return a;
}

}  // namespace

extern "C" ServiceTime RS_CAT(__wrap_, RS_WRAPPED)(const ModelSpec& model, std::int64_t query_size,
                                                    const AcceleratorSpec& spec) {
  if (spec.name != "b200") return RS_CAT(__real_, RS_WRAPPED)(model, query_size, spec);
  if (query_size < 1) throw std::invalid_argument("query_size < 1");
  double seconds = 0;
  if (rs_service_time(accel_for(model), query_size, &seconds) != RS_OK)
    throw std::runtime_error(std::string("rs_service_time: ") + rs_last_error());
  ServiceTime st;
  st.total = seconds;
  return st;
}

// B200 accelerator spec for the reference's AcceleratorSpec::validate
// (platform.cpp:65-69 needs positive fields; only the name is consulted).
extern "C" void ref_b200_release() {
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto& kv : g_accels) rs_accel_destroy(kv.second);
  g_accels.clear();
}
