// host_model.cpp — the whole forward pass of one model on the host cores: the
// CPU side of DeepRecSched's split. The reference sends
// every query of size <= T to a CPU core as floor(S/B) requests of B items
// plus one of S mod B (proj/src/sim.cpp:184-188), each priced by
// cpu_service_time (proj/src/platform.cpp:71-97) and served whole by one core
// (sim.cpp:114-124; "a single Caffe2 worker and Intel MKL thread",
// PAPER.md:643). rs_host_forward executes such a request for real, with the
// same operator order and tensor widths as the device graph (work(),
// proj/src/model_zoo.cpp:177-245; predict_input_dim, :113-137) and the same
// parameters (spec.h), so a query gives the same logits on
// either side of the split within the fp32 tolerance rule (tests/parity_rule.py)
// — the embedding sums are even bit-identical (canonical SLS order).
//
// Layout: tables [T][rows][D] fp32 in host memory (filled on all cores at
// create: 82 GB for BASELINE configs[2]); every FC weight kept transposed
// [in][out] once, so a request never transposes (host_fc.cpp's register tile
// streams W^T rows). One request = one thread; rs_host_forward with
// threads > 1 deals a request's items to threads (a query run whole).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <sched.h>

#include "../spec.h"
#include "internal.hpp"

namespace rs {
namespace {

struct HostFc {
  int64_t in = 0, out = 0;
  int relu = 0;
  std::vector<float> wt;  // [stacks][in][out]
  std::vector<float> b;   // [stacks][out]
};

}  // namespace

int host_cores() {
  cpu_set_t set;
  CPU_ZERO(&set);
  if (sched_getaffinity(0, sizeof(set), &set) == 0) {
    const int n = CPU_COUNT(&set);
    if (n > 0) return n;
  }
  return (int)std::max(1u, std::thread::hardware_concurrency());
}

}  // namespace rs

struct rs_host_model {
  rs_model_desc m{};
  rs_init_desc init{};
  int64_t T = 0, L = 0, D = 0, H = 0, stacks = 1, rows = 0;
  int64_t dense_in = 0, dense_out = 0, p_in = 0, out_dim = 0, out_w = 0, pooled_dim = 0;
  std::unique_ptr<float[]> tables;
  std::vector<rs::HostFc> dense, pred;
  std::vector<float> att;                        // [T][D][D]
  std::vector<float> wih, whh, bih, bhh, watt;   // GRU per table
};

namespace rs {
namespace {

void parallel_for(int64_t n, int threads, const std::function<void(int64_t, int64_t)>& f) {
  threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n));
  if (threads == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(threads);
  for (int i = 0; i < threads; ++i)
    th.emplace_back([&, i] { f(n * i / threads, n * (i + 1) / threads); });
  for (auto& t : th) t.join();
}

HostFc make_fc(uint64_t seed, int64_t in, int64_t out, int relu, int64_t stacks,
               uint64_t (*wid)(int64_t, int64_t), uint64_t (*bid)(int64_t, int64_t),
               int64_t layer) {
  HostFc f;
  f.in = in; f.out = out; f.relu = relu;
  f.wt.assign((size_t)(stacks * in * out), 0.f);
  f.b.assign((size_t)(stacks * out), 0.f);
  const float bound = 1.0f / sqrtf((float)in);
  for (int64_t z = 0; z < stacks; ++z) {
    const uint64_t kw = stream_key(seed, wid(z, layer)), kb = stream_key(seed, bid(z, layer));
    for (int64_t o = 0; o < out; ++o) {
      for (int64_t i = 0; i < in; ++i)
        f.wt[(size_t)((z * in + i) * out + o)] = param(kw, (uint64_t)(o * in + i), bound);
      f.b[(size_t)(z * out + o)] = param(kb, (uint64_t)o, bound);
    }
  }
  return f;
}

uint64_t dwid(int64_t, int64_t l) { return id_dense_w(l); }
uint64_t dbid(int64_t, int64_t l) { return id_dense_b(l); }
uint64_t pwid(int64_t s, int64_t l) { return id_pred_w(s, l); }
uint64_t pbid(int64_t s, int64_t l) { return id_pred_b(s, l); }

std::vector<float> gen(uint64_t seed, uint64_t id, int64_t n, float bound) {
  std::vector<float> v((size_t)n);
  const uint64_t k = stream_key(seed, id);
  for (int64_t i = 0; i < n; ++i) v[(size_t)i] = param(k, (uint64_t)i, bound);
  return v;
}

float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

// Items [m0, m1) of one request, single thread. dense f32[S][dense_in],
// idx i64[S][T][L], out f32[S][out_w] (all indexed by absolute item).
int64_t forward_rows(const rs_host_model* h, const float* dense, const int64_t* idx, float* out,
                     int64_t m0, int64_t m1) {
  const rs_model_desc& m = h->m;
  const int64_t b = m1 - m0, T = h->T, L = h->L, D = h->D, p_in = h->p_in, dout = h->dense_out;
  if (b <= 0) return -1;
  std::vector<float> X((size_t)(b * p_in), 0.f), tmp[2];
  // ---- DenseFC (ReLU after every layer) or the raw dense features
  if (m.has_dense_fc) {
    const float* a = dense + m0 * h->dense_in;
    int64_t k = h->dense_in;
    for (size_t l = 0; l < h->dense.size(); ++l) {
      const HostFc& f = h->dense[l];
      tmp[l & 1].resize((size_t)(b * f.out));
      host_fc_rows(a, 0, b, (int)k, (int)f.out, f.wt.data(), f.b.data(), 1, tmp[l & 1].data());
      a = tmp[l & 1].data();
      k = f.out;
    }
    for (int64_t i = 0; i < b; ++i) std::memcpy(&X[(size_t)(i * p_in)], a + i * dout, 4 * dout);
  } else {
    for (int64_t i = 0; i < b; ++i)
      std::memcpy(&X[(size_t)(i * p_in)], dense + (m0 + i) * h->dense_in, 4 * h->dense_in);
  }
  // ---- EmbeddingLookup + pooling
  const float* tab = h->tables.get();
  auto row = [&](int64_t t, int64_t r) { return tab + (t * h->rows + r) * D; };
  if (T > 0) {
    const int64_t* qi = idx + m0 * T * L;
    switch (m.pooling) {
      case RS_POOL_SUM: {
        std::vector<float> P((size_t)(b * T * D));
        const int64_t bad = host_pool_bags(tab, h->rows, (int)T, (int)L, (int)D, qi, P.data(), 0,
                                           b * T);
        if (bad >= 0) return m0 * T * L + bad;
        for (int64_t i = 0; i < b; ++i) {
          float* x = &X[(size_t)(i * p_in)];
          const float* Pi = &P[(size_t)(i * T * D)];
          for (int64_t c = 0; c < D; ++c) {  // summed embedding (D9)
            float s = 0.f;
            for (int64_t t = 0; t < T; ++t) s += Pi[t * D + c];
            x[dout + c] = s;
          }
          if (m.has_dense_fc) {  // triu dots over v0 = dense_out, v_t = pooled_t
            int64_t p = 0;
            for (int64_t a = 1; a <= T; ++a)
              for (int64_t j = 0; j < a; ++j, ++p) {
                const float* va = Pi + (a - 1) * D;
                const float* vj = j == 0 ? x : Pi + (j - 1) * D;
                float d = 0.f;
                for (int64_t c = 0; c < D; ++c) d += va[c] * vj[c];
                x[dout + D + p] = d;
              }
          }
        }
        break;
      }
      case RS_POOL_CONCAT:
        for (int64_t i = 0; i < b; ++i)
          for (int64_t k = 0; k < T * L; ++k) {
            const int64_t r = qi[i * T * L + k];
            if ((uint64_t)r >= (uint64_t)h->rows) return (m0 + i) * T * L + k;
            std::memcpy(&X[(size_t)(i * p_in + dout + k * D)], row(k / L, r), 4 * D);
          }
        break;
      case RS_POOL_ATTENTION_FC: {
        std::vector<float> u((size_t)D);
        for (int64_t i = 0; i < b; ++i)
          for (int64_t t = 0; t < T; ++t) {
            const int64_t* bi = qi + (i * T + t) * L;
            for (int64_t l = 0; l < L; ++l)
              if ((uint64_t)bi[l] >= (uint64_t)h->rows) return ((m0 + i) * T + t) * L + l;
            const float* q = row(t, bi[0]);
            const float* W = &h->att[(size_t)(t * D * D)];
            for (int64_t c = 0; c < D; ++c) {  // u = W_t^T q
              float a = 0.f;
              for (int64_t r = 0; r < D; ++r) a += W[r * D + c] * q[r];
              u[(size_t)c] = a;
            }
            float* o = &X[(size_t)(i * p_in + dout + t * D)];
            for (int64_t l = 0; l < L; ++l) {
              const float* e = row(t, bi[l]);
              float sc = 0.f;
              for (int64_t c = 0; c < D; ++c) sc += u[(size_t)c] * e[c];
              const float a = sigm(sc);
              for (int64_t c = 0; c < D; ++c) o[c] += a * e[c];
            }
          }
        break;
      }
      case RS_POOL_ATTENTION_RNN: {
        const int64_t H = h->H, H3 = 3 * H;
        const bool augru = h->init.rnn_cell == RS_RNN_AUGRU;
        std::vector<float> hs((size_t)H), gi((size_t)H3), gh((size_t)H3), ua((size_t)D);
        for (int64_t i = 0; i < b; ++i)
          for (int64_t t = 0; t < T; ++t) {
            const int64_t* bi = qi + (i * T + t) * L;
            for (int64_t l = 0; l < L; ++l)
              if ((uint64_t)bi[l] >= (uint64_t)h->rows) return ((m0 + i) * T + t) * L + l;
            const float* wih = &h->wih[(size_t)(t * H3 * D)];
            const float* whh = &h->whh[(size_t)(t * H3 * H)];
            const float* bih = &h->bih[(size_t)(t * H3)];
            const float* bhh = &h->bhh[(size_t)(t * H3)];
            std::fill(hs.begin(), hs.end(), 0.f);
            if (augru) {  // ua = W_a^T x_0
              const float* x0 = row(t, bi[0]);
              const float* wa = &h->watt[(size_t)(t * D * D)];
              for (int64_t c = 0; c < D; ++c) {
                float a = 0.f;
                for (int64_t r = 0; r < D; ++r) a += x0[r] * wa[r * D + c];
                ua[(size_t)c] = a;
              }
            }
            for (int64_t l = 0; l < L; ++l) {
              const float* x = row(t, bi[l]);
              for (int64_t r = 0; r < H3; ++r) {
                float a = bih[r], g = bhh[r];
                for (int64_t c = 0; c < D; ++c) a += wih[r * D + c] * x[c];
                for (int64_t k = 0; k < H; ++k) g += whh[r * H + k] * hs[(size_t)k];
                gi[(size_t)r] = a;
                gh[(size_t)r] = g;
              }
              float att = 1.f;
              if (augru) {
                float sc = 0.f;
                for (int64_t c = 0; c < D; ++c) sc += ua[(size_t)c] * x[c];
                att = sigm(sc);
              }
              for (int64_t j = 0; j < H; ++j) {
                const float r = sigm(gi[(size_t)j] + gh[(size_t)j]);
                const float z = sigm(gi[(size_t)(H + j)] + gh[(size_t)(H + j)]);
                const float n = tanhf(gi[(size_t)(2 * H + j)] + r * gh[(size_t)(2 * H + j)]);
                if (augru) {
                  const float uu = att * (1.f - z);
                  hs[(size_t)j] = (1.f - uu) * hs[(size_t)j] + uu * n;
                } else {
                  hs[(size_t)j] = (1.f - z) * n + z * hs[(size_t)j];
                }
              }
            }
            std::memcpy(&X[(size_t)(i * p_in + dout + t * H)], hs.data(), 4 * H);
          }
        break;
      }
    }
  }
  // ---- PredictFC: N stacks on the shared input, ReLU on hidden layers
  for (int64_t z = 0; z < h->stacks; ++z) {
    const float* a = X.data();
    int64_t k = p_in;
    for (size_t l = 0; l < h->pred.size(); ++l) {
      const HostFc& f = h->pred[l];
      tmp[l & 1].resize((size_t)(b * f.out));
      host_fc_rows(a, 0, b, (int)k, (int)f.out, f.wt.data() + z * f.in * f.out,
                   f.b.data() + z * f.out, f.relu, tmp[l & 1].data());
      a = tmp[l & 1].data();
      k = f.out;
    }
    for (int64_t i = 0; i < b; ++i)
      std::memcpy(out + (m0 + i) * h->out_w + z * h->out_dim, a + i * h->out_dim,
                  4 * h->out_dim);
  }
  return -1;
}

}  // namespace

int64_t host_forward_rows(const rs_host_model* h, const float* dense, const int64_t* idx,
                          float* out, int64_t m0, int64_t m1) {
  return forward_rows(h, dense, idx, out, m0, m1);
}

}  // namespace rs

using namespace rs;

extern "C" int rs_host_model_create(const rs_model_desc* model, const rs_init_desc* init,
                                    int32_t threads, rs_host_model** out) {
  return guarded([&] {
    if (!model || !init || !out) raise(RS_E_INVALID, "null argument");
    *out = nullptr;
    validate_model(*model);
    auto h = std::make_unique<rs_host_model>();
    const rs_model_desc& m = *model;
    h->m = m;
    h->init = *init;
    h->T = m.num_tables; h->L = m.lookups_per_table; h->D = m.embedding_dim;
    h->H = m.recurrent_hidden_dim; h->stacks = m.num_parallel_predict_stacks;
    h->rows = init->rows_per_table;
    h->dense_in = m.dense_input_dim;
    h->dense_out = dense_out_dim(m);
    h->p_in = predict_input_dim(m);
    h->out_dim = m.predict_fc.dims[m.predict_fc.n - 1];
    h->out_w = h->stacks * h->out_dim;
    if (h->T > 0 && h->rows < 1) raise(RS_E_INVALID, "rows_per_table < 1");
    if (m.pooling == RS_POOL_SUM && m.has_dense_fc && h->T > 0 && h->dense_out != h->D)
      raise(RS_E_INVALID, "dot interaction needs dense stack output == embedding_dim (D2)");
    if (m.pooling == RS_POOL_ATTENTION_RNN && h->T > 0 && h->H < 1)
      raise(RS_E_INVALID, "AttentionRNN needs recurrent_hidden_dim");
    const int nt = threads > 0 ? threads : host_cores();
    if (h->T > 0) {
      const int64_t n = h->T * h->rows * h->D;
      h->tables.reset(new (std::nothrow) float[(size_t)n]);
      if (!h->tables) raise(RS_E_OOM, "host tables");
      float* tab = h->tables.get();
      const int64_t per = h->rows * h->D;
      const uint64_t seed = init->seed;
      parallel_for(n, nt, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b;) {
          const int64_t t = i / per, end = std::min(b, (t + 1) * per);
          const uint64_t key = stream_key(seed, id_table(t));
          for (int64_t e = i - t * per; i < end; ++i, ++e) tab[i] = param(key, (uint64_t)e, kTableScale);
        }
      });
    }
    if (m.has_dense_fc) {
      int64_t in = h->dense_in;
      for (int l = 0; l < m.dense_fc.n; ++l) {
        h->dense.push_back(make_fc(init->seed, in, m.dense_fc.dims[l], 1, 1, dwid, dbid, l));
        in = m.dense_fc.dims[l];
      }
    }
    {
      int64_t in = h->p_in;
      for (int l = 0; l < m.predict_fc.n; ++l) {
        h->pred.push_back(make_fc(init->seed, in, m.predict_fc.dims[l],
                                  l + 1 < m.predict_fc.n ? 1 : 0, h->stacks, pwid, pbid, l));
        in = m.predict_fc.dims[l];
      }
    }
    const int64_t T = h->T, D = h->D, H = h->H;
    if (m.pooling == RS_POOL_ATTENTION_FC)
      for (int64_t t = 0; t < T; ++t) {
        auto v = gen(init->seed, id_att_w(t), D * D, 1.0f / sqrtf((float)D));
        h->att.insert(h->att.end(), v.begin(), v.end());
      }
    if (m.pooling == RS_POOL_ATTENTION_RNN)
      for (int64_t t = 0; t < T; ++t) {
        const float bh = 1.0f / sqrtf((float)H), bd = 1.0f / sqrtf((float)D);
        auto a0 = gen(init->seed, id_gru(t, 0), 3 * H * D, bh);
        auto a1 = gen(init->seed, id_gru(t, 1), 3 * H * H, bh);
        auto a2 = gen(init->seed, id_gru(t, 2), 3 * H, bh);
        auto a3 = gen(init->seed, id_gru(t, 3), 3 * H, bh);
        auto a4 = gen(init->seed, id_gru(t, 4), D * D, bd);
        h->wih.insert(h->wih.end(), a0.begin(), a0.end());
        h->whh.insert(h->whh.end(), a1.begin(), a1.end());
        h->bih.insert(h->bih.end(), a2.begin(), a2.end());
        h->bhh.insert(h->bhh.end(), a3.begin(), a3.end());
        h->watt.insert(h->watt.end(), a4.begin(), a4.end());
      }
    *out = h.release();
  });
}

extern "C" int rs_host_model_destroy(rs_host_model* h) {
  return guarded([&] { delete h; });
}

extern "C" int rs_host_forward(rs_host_model* h, const rs_query* q, float* out,
                               int32_t threads) {
  return guarded([&] {
    if (!h || !q || !out) raise(RS_E_INVALID, "null argument");
    if (q->size < 1) raise(RS_E_INVALID, "query_size < 1");
    if (q->location != RS_MEM_HOST) raise(RS_E_INVALID, "host forward takes host memory");
    if (q->index_type != 0) raise(RS_E_INVALID, "host forward takes the reference byte model");
    if (h->dense_in > 0 && !q->dense) raise(RS_E_INVALID, "null dense features");
    if (h->T > 0 && !q->indices) raise(RS_E_INVALID, "null indices");
    const int nt = threads > 0 ? threads : 1;
    std::vector<int64_t> bad((size_t)nt, -1);
    const int64_t S = q->size;
    const int use = (int)std::max<int64_t>(1, std::min<int64_t>(nt, S));
    std::vector<std::thread> th;
    for (int i = 0; i < use; ++i) {
      auto job = [&, i] {
        bad[(size_t)i] = forward_rows(h, q->dense, q->indices, out, S * i / use,
                                      S * (i + 1) / use);
      };
      if (use == 1) job();
      else th.emplace_back(job);
    }
    for (auto& t : th) t.join();
    for (int64_t v : bad)
      if (v >= 0)
        raise(RS_E_INDEX, "embedding index " + std::to_string(q->indices[v]) +
                              " outside [0, rows_per_table)");
  });
}
