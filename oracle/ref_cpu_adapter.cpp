// ORACLE — TEST INFRASTRUCTURE ONLY (the CPU baseline of bench.py).
//
// The reference prices each CPU request of b items with the pure cost model
//   recsim::cpu_service_time(const WorkBreakdown&, b, active_cores, const CpuPlatformSpec&)
//   (/root/reference/proj/src/platform.cpp:71-97; called by simulate()'s
//    dispatch_cpu, proj/src/sim.cpp:114-124, and by max_qps_under_sla's
//    capacity bracket, :257-262).
// Linked with --wrap of both overloads into oracle/_ref/librecsim_ref_cpu.so
// together with the UNMODIFIED reference sources: for the CpuPlatformSpec named
// "measured" the time is looked up in a table MEASURED on this host (the
// oracle's fp32 forward, oracle/forward.c or_time_requests, timed with 1 and
// with all cores busy; linear in b between measured sizes and linear in the
// active-core count between the two), every other platform falls through to
// the reference model. The reference's own simulate() / max_qps_under_sla() /
// tune() then run unchanged on the box's real CPU cost: split rule, C-core
// FIFO, exact p95 and lambda bisection are the reference's code.
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "recsim/model_zoo.hpp"
#include "recsim/platform.hpp"

using recsim::CpuPlatformSpec;
using recsim::ModelSpec;
using recsim::ServiceTime;
using recsim::WorkBreakdown;

#define RS_WB _ZN6recsim16cpu_service_timeERKNS_13WorkBreakdownEllRKNS_15CpuPlatformSpecE
#define RS_MS _ZN6recsim16cpu_service_timeERKNS_9ModelSpecEllRKNS_15CpuPlatformSpecE
#define RS_CAT2(a, b) a##b
#define RS_CAT(a, b) RS_CAT2(a, b)

extern "C" ServiceTime RS_CAT(__real_, RS_WB)(const WorkBreakdown&, std::int64_t, std::int64_t,
                                               const CpuPlatformSpec&);
extern "C" ServiceTime RS_CAT(__real_, RS_MS)(const ModelSpec&, std::int64_t, std::int64_t,
                                               const CpuPlatformSpec&);

namespace {

struct Table {
  std::vector<std::int64_t> b;   // ascending request sizes
  std::vector<double> t1, tc;    // seconds with 1 / `cores` active cores
  std::int64_t cores = 1;
};
std::mutex g_mu;
Table g_table;

double interp(const std::vector<double>& t, const std::vector<std::int64_t>& b, std::int64_t x) {
  if (b.size() == 1) return t[0] * static_cast<double>(x) / static_cast<double>(b[0]);
  size_t hi = 1;
  while (hi + 1 < b.size() && b[hi] < x) ++hi;
  const size_t lo = hi - 1;
  const double f = static_cast<double>(x - b[lo]) / static_cast<double>(b[hi] - b[lo]);
  return std::max(1e-9, t[lo] + f * (t[hi] - t[lo]));  // linear (extrapolated past the ends)
}

ServiceTime measured(std::int64_t batch, std::int64_t active) {
  if (batch < 1) throw std::invalid_argument("batch < 1");
  std::lock_guard<std::mutex> lock(g_mu);
  const Table& T = g_table;
  if (T.b.empty()) throw std::invalid_argument("measured CPU table not set");
  if (active < 1 || active > T.cores) throw std::invalid_argument("active_cores outside [1, cores]");
  const double a = interp(T.t1, T.b, batch), c = interp(T.tc, T.b, batch);
  const double f = T.cores > 1 ? static_cast<double>(active - 1) / static_cast<double>(T.cores - 1) : 1.0;
  ServiceTime st;
  st.total = a + f * (c - a);
  return st;
}

}  // namespace

extern "C" ServiceTime RS_CAT(__wrap_, RS_WB)(const WorkBreakdown& wb, std::int64_t batch,
                                               std::int64_t active, const CpuPlatformSpec& p) {
  if (p.name != "measured") return RS_CAT(__real_, RS_WB)(wb, batch, active, p);
  return measured(batch, active);
}

extern "C" ServiceTime RS_CAT(__wrap_, RS_MS)(const ModelSpec& m, std::int64_t batch,
                                               std::int64_t active, const CpuPlatformSpec& p) {
  if (p.name != "measured") return RS_CAT(__real_, RS_MS)(m, batch, active, p);
  return measured(batch, active);
}

extern "C" int64_t ref_measured_cores(void) {
  std::lock_guard<std::mutex> lock(g_mu);
  return g_table.cores;
}

// n request sizes (ascending) with their measured seconds at 1 and at `cores`
// busy cores. Returns 0, or -1 on a malformed table.
extern "C" int ref_cpu_set_table(int n, const int64_t* b, const double* t1, const double* tc,
                                 int64_t cores) {
  if (n < 1 || cores < 1) return -1;
  for (int i = 1; i < n; ++i)
    if (b[i] <= b[i - 1]) return -1;
  std::lock_guard<std::mutex> lock(g_mu);
  g_table.b.assign(b, b + n);
  g_table.t1.assign(t1, t1 + n);
  g_table.tc.assign(tc, tc + n);
  g_table.cores = cores;
  return 0;
}
