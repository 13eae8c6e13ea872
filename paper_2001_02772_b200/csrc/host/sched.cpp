// sched.cpp — host side of the scheduler interface: error plumbing, the
// split/offload routing decision, bit-exact query streams, synthetic query
// inputs and the QPS-under-SLA search over measured service times.
//
//   routing            proj/src/sim.cpp:173-191 (strict S > T; floor/rem split)
//   Rng / gen_trace    proj/include/recsim/rng.hpp:14-48, proj/src/loadgen.cpp:80-125
//   SizeDistribution   proj/include/recsim/loadgen.hpp:23-45, loadgen.cpp:15-68
//   max_qps_under_sla  proj/src/sim.cpp:207-290 (exact p95, geometric bisection)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>

#include "../spec.h"
#include "internal.hpp"

namespace rs {

namespace {
thread_local std::string g_last_error;
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
void clear_error() { g_last_error.clear(); }
[[noreturn]] void raise(int code, const std::string& msg) { throw Error{code, msg}; }

namespace {

// Draw stream pinned to mt19937_64 with explicit inverse-CDF samplers; the
// expression order matches rng.hpp so every double is bit-identical.
class Stream {
 public:
  explicit Stream(uint64_t seed) : mt_(seed) {}
  double u01() { return static_cast<double>(mt_() >> 11) * 0x1.0p-53; }
  double u01_open_low() { return 1.0 - u01(); }
  double exp_gap(double rate) { return -std::log(u01_open_low()) / rate; }
  double gauss(double mean, double sd) {
    const double a = u01_open_low();
    const double b = u01();
    const double z = std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * M_PI * b);
    return mean + sd * z;
  }
  double lognormal(double mu, double sigma) { return std::exp(gauss(mu, sigma)); }
  double pareto(double xmin, double alpha) {
    return xmin * std::pow(u01_open_low(), -1.0 / alpha);
  }

 private:
  std::mt19937_64 mt_;
};

void check_dist(const rs_size_dist& d) {
  for (double p : {d.p0, d.p1, d.p2, d.p3})
    if (!std::isfinite(p)) raise(RS_E_DISTRIBUTION, "non-finite distribution parameter");
  if (d.max_size < 1) raise(RS_E_DISTRIBUTION, "max_size < 1");
  if (d.kind < RS_DIST_FIXED || d.kind > RS_DIST_PRODUCTION_HEAVY_TAIL)
    raise(RS_E_DISTRIBUTION, "unknown distribution kind");
  if (d.kind == RS_DIST_PRODUCTION_HEAVY_TAIL) {
    if (d.p2 <= 0) raise(RS_E_DISTRIBUTION, "tail_alpha must be positive");
    if (d.p3 < 0 || d.p3 > 1) raise(RS_E_DISTRIBUTION, "tail_weight outside [0, 1]");
  }
}

int64_t draw_size(Stream& s, const rs_size_dist& d) {
  double x = 0;
  switch (d.kind) {
    case RS_DIST_FIXED: x = d.p0; break;
    case RS_DIST_NORMAL: x = s.gauss(d.p0, d.p1); break;
    case RS_DIST_LOGNORMAL: x = s.lognormal(d.p0, d.p1); break;
    case RS_DIST_PRODUCTION_HEAVY_TAIL: {
      const bool in_tail = s.u01() < d.p3;
      x = in_tail ? s.pareto(std::exp(d.p0), d.p2) : s.lognormal(d.p0, d.p1);
      break;
    }
  }
  const int64_t v = static_cast<int64_t>(std::llround(x));
  return std::clamp<int64_t>(v, 1, d.max_size);
}

double order_stat(std::vector<double>& v, double pct) {
  std::sort(v.begin(), v.end());
  size_t k = static_cast<size_t>(std::ceil(pct / 100.0 * static_cast<double>(v.size())));
  k = std::max<size_t>(k, 1) - 1;
  return v[std::min(k, v.size() - 1)];
}

struct QpsEval {
  rs_qps_result r;
  bool ok;
};

// One open-loop replay of the measured stream at rate `lambda` over
// `servers` FIFO replicas (least outstanding work, ties to lowest index).
QpsEval replay(const double* service, const double* extra, int64_t n, int servers,
               double lambda, uint64_t seed, double warmup_fraction, double sla) {
  Stream gaps(seed);
  std::vector<double> free_at(static_cast<size_t>(servers), 0.0);
  const int64_t warm = static_cast<int64_t>(std::floor(warmup_fraction * static_cast<double>(n)));
  std::vector<double> lat;
  lat.reserve(static_cast<size_t>(n - warm));
  double now = 0, first_pw_arrival = 0, last_done = 0;
  for (int64_t i = 0; i < n; ++i) {
    now += gaps.exp_gap(lambda);
    int best = 0;
    double best_backlog = std::max(0.0, free_at[0] - now);
    for (int k = 1; k < servers; ++k) {
      const double b = std::max(0.0, free_at[static_cast<size_t>(k)] - now);
      if (b < best_backlog) { best = k; best_backlog = b; }
    }
    const double start = std::max(now, free_at[static_cast<size_t>(best)]);
    const double done = start + service[i];
    free_at[static_cast<size_t>(best)] = done;
    last_done = std::max(last_done, done);
    if (i == warm) first_pw_arrival = now;
    if (i >= warm) lat.push_back(done - now + (extra ? std::max(0.0, extra[i]) : 0.0));
  }
  QpsEval e{};
  if (lat.empty()) raise(RS_E_EMPTY, "no post-warmup queries");
  const double span = last_done - first_pw_arrival;
  e.r.qps = span > 0 ? static_cast<double>(lat.size()) / span : 0;
  e.r.at_lambda = lambda;
  std::vector<double> v = lat;
  e.r.p95 = order_stat(v, 95);
  e.r.p50 = order_stat(v, 50);
  e.ok = e.r.p95 <= sla;
  return e;
}

}  // namespace
}  // namespace rs

using namespace rs;

extern "C" const char* rs_last_error(void) { return g_last_error.c_str(); }
extern "C" int rs_abi_version(void) { return RS_ABI_VERSION; }

extern "C" int rs_route(int64_t query_size, int64_t batch_size, int64_t threshold,
                        int32_t* offload, int64_t* requests, int64_t cap,
                        int64_t* n_requests) {
  return guarded([&] {
    if (!offload || !n_requests) raise(RS_E_INVALID, "null argument");
    if (batch_size < 1) raise(RS_E_CONFIG, "batch_size < 1");
    if (query_size < 1) raise(RS_E_INVALID, "query_size < 1");
    *n_requests = 0;
    if (threshold > 0 && query_size > threshold) {  // whole query to the accelerator
      *offload = 1;
      return;
    }
    *offload = 0;
    const int64_t full = query_size / batch_size;
    const int64_t rem = query_size % batch_size;
    const int64_t total = full + (rem > 0 ? 1 : 0);
    if (total > cap || (!requests && total > 0))
      raise(RS_E_CAPACITY, "request buffer too small");
    for (int64_t i = 0; i < full; ++i) requests[i] = batch_size;
    if (rem > 0) requests[full] = rem;
    *n_requests = total;
  });
}

extern "C" int rs_dist_production(rs_size_dist* out) {
  return guarded([&] {
    if (!out) raise(RS_E_INVALID, "null argument");
    *out = rs_size_dist{RS_DIST_PRODUCTION_HEAVY_TAIL, std::log(300.0), 0.5, 1.1, 0.25, 1000};
  });
}

extern "C" int rs_gen_trace(uint64_t seed, double lambda, const rs_size_dist* dist,
                            int64_t n, double* arrival_times, int64_t* sizes) {
  return guarded([&] {
    if (!dist) raise(RS_E_INVALID, "null distribution");
    if (lambda <= 0 || !std::isfinite(lambda))
      raise(RS_E_DISTRIBUTION, "lambda must be positive and finite");
    if (n < 1) raise(RS_E_INVALID, "n < 1");
    check_dist(*dist);
    Stream s(seed);
    double t = 0;
    for (int64_t i = 0; i < n; ++i) {
      t += s.exp_gap(lambda);
      const int64_t sz = draw_size(s, *dist);
      if (arrival_times) arrival_times[i] = t;
      if (sizes) sizes[i] = sz;
    }
  });
}

extern "C" int rs_qps_under_sla(const double* service_s, const double* extra_s, int64_t n,
                                int32_t servers, double sla_s, double warmup_fraction,
                                uint64_t base_seed, double lambda_hi, rs_qps_result* out) {
  return guarded([&] {
    if (!service_s || !out) raise(RS_E_INVALID, "null argument");
    if (n < 1) raise(RS_E_INVALID, "n < 1");
    if (servers < 1) raise(RS_E_CONFIG, "servers < 1");
    if (sla_s <= 0) raise(RS_E_INVALID, "sla <= 0");
    if (warmup_fraction < 0 || warmup_fraction > 0.5)
      raise(RS_E_CONFIG, "warmup_fraction outside [0, 0.5]");
    double mean = 0;
    for (int64_t i = 0; i < n; ++i) mean += service_s[i];
    mean /= static_cast<double>(n);
    double hi = lambda_hi > 0 ? lambda_hi : 2.0 * servers / std::max(mean, 1e-12);
    hi = std::max(hi, 2.0);
    uint64_t idx = 0;
    int evals = 0;
    auto eval = [&](double lam) {
      ++evals;
      return replay(service_s, extra_s, n, servers, lam, base_seed + idx++, warmup_fraction,
                    sla_s);
    };
    double lo = 1.0;
    QpsEval lo_e = eval(lo);
    if (!lo_e.ok) {
      *out = rs_qps_result{0, 0, lo_e.r.p95, lo_e.r.p50, evals};
      return;
    }
    QpsEval hi_e = eval(hi);
    if (hi_e.ok) {
      *out = hi_e.r;
      out->evaluations = evals;
      return;
    }
    rs_qps_result best = lo_e.r;
    while (hi / lo > 1.01) {
      const double mid = std::sqrt(lo * hi);
      QpsEval e = eval(mid);
      if (e.ok) {
        lo = mid;
        best = e.r;
      } else {
        hi = mid;
      }
    }
    *out = best;
    out->evaluations = evals;
  });
}

extern "C" int rs_fill_query(const rs_model_desc* m, int64_t rows_per_table, uint64_t seed,
                             uint64_t query_id, int64_t size, float* dense,
                             int64_t* indices) {
  return guarded([&] {
    if (!m) raise(RS_E_INVALID, "null model");
    if (size < 1) raise(RS_E_INVALID, "size < 1");
    if (m->num_tables > 0 && rows_per_table < 1) raise(RS_E_INVALID, "rows_per_table < 1");
    const uint64_t nd = static_cast<uint64_t>(size * m->dense_input_dim);
    if (dense && nd) {
      const uint64_t k = stream_key(seed, id_query_dense(query_id));
      for (uint64_t i = 0; i < nd; ++i) dense[i] = unit(splitmix64(k + i));
    }
    const uint64_t ni = static_cast<uint64_t>(size * m->num_tables * m->lookups_per_table);
    if (indices && ni) {
      const uint64_t k = stream_key(seed, id_query_idx(query_id));
      for (uint64_t i = 0; i < ni; ++i)
        indices[i] = index_from_hash(splitmix64(k + i), rows_per_table);
    }
  });
}

extern "C" int rs_fill_query_zipf(const rs_model_desc* m, int64_t rows_per_table, uint64_t seed,
                                  uint64_t query_id, int64_t size, double alpha, float* dense,
                                  int64_t* indices) {
  return guarded([&] {
    if (!(alpha > 0.0)) raise(RS_E_INVALID, "zipf alpha must be > 0");
    int rc = rs_fill_query(m, rows_per_table, seed, query_id, size, dense, nullptr);
    if (rc != RS_OK) raise(rc, rs_last_error());
    const uint64_t ni = static_cast<uint64_t>(size * m->num_tables * m->lookups_per_table);
    if (!indices || !ni) return;
    // inverse CDF of x^-alpha on [1, N+1): x = (1 + u((N+1)^(1-a) - 1))^(1/(1-a))
    // (a = 1: x = (N+1)^u); index = floor(x) - 1
    const double n1 = static_cast<double>(rows_per_table) + 1.0;
    const bool one = std::fabs(alpha - 1.0) < 1e-12;
    const double e = 1.0 - alpha;
    const double span = one ? std::log(n1) : std::pow(n1, e) - 1.0;
    const uint64_t k = stream_key(seed, id_query_idx(query_id));
    for (uint64_t i = 0; i < ni; ++i) {
      const double u = static_cast<double>(splitmix64(k + i) >> 11) * 0x1.0p-53;
      const double x = one ? std::exp(u * span) : std::pow(1.0 + u * span, 1.0 / e);
      int64_t r = static_cast<int64_t>(x) - 1;
      indices[i] = r < 0 ? 0 : (r >= rows_per_table ? rows_per_table - 1 : r);
    }
  });
}
