// internal.hpp — shared host-side helpers behind the rs_* C-ABI.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../../include/rs_accel.h"

namespace rs {

// Thread-local last-error plumbing: every ABI function returns a code and
// leaves a message; no exception ever crosses the ABI.
int fail(int code, const std::string& msg);
void clear_error();

// Typed failure used inside the library; converted to a code at the ABI.
struct Error {
  int code;
  std::string msg;
};
[[noreturn]] void raise(int code, const std::string& msg);

template <class F>
int guarded(F&& f) {
  try {
    clear_error();
    f();
    return RS_OK;
  } catch (const Error& e) {
    return fail(e.code, e.msg);
  } catch (const std::exception& e) {
    return fail(RS_E_INVALID, e.what());
  } catch (...) {
    return fail(RS_E_INVALID, "unknown exception");
  }
}

// ---- model descriptor helpers (model.cpp) ----
void validate_model(const rs_model_desc& m);
int64_t predict_input_dim(const rs_model_desc& m);
int64_t dense_out_dim(const rs_model_desc& m);
int64_t sparse_out_dim(const rs_model_desc& m);
int64_t interaction_pairs(const rs_model_desc& m);
rs_work_breakdown work(const rs_model_desc& m, int64_t batch);
double accel_input_bytes(const rs_model_desc& m, int64_t query_size);

// ---- host-core operators (host_sls.cpp, host_fc.cpp) ----
// Canonical-order SLS of bags [b0, b1) (bag = item*T + t); returns the first
// bad (bag*L + lookup) or -1.
int64_t host_pool_bags(const float* tables, int64_t rows, int T, int L, int D,
                       const int64_t* idx, float* pooled, int64_t b0, int64_t b1);
// y[m][0..N) = act(b + x[m][0..K) . wt[0..K)[n]) for rows [m0, m1); x row
// stride K, y row stride N, wt the transposed weight [K][N].
void host_fc_rows(const float* x, int64_t m0, int64_t m1, int K, int N, const float* wt,
                  const float* b, int relu, float* y);

// Host forward of items [m0, m1) of one request on the calling thread
// (host_model.cpp); returns the first bad index position or -1.
int64_t host_forward_rows(const rs_host_model* h, const float* dense, const int64_t* idx,
                          float* out, int64_t m0, int64_t m1);
// Cores this process may run on (sched_getaffinity; cgroup cpusets included).
int host_cores();

}  // namespace rs
