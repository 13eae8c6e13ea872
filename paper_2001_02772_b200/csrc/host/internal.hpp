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

}  // namespace rs
