// accel.cu — rs_accel: one model replica on one B200, behind the C-ABI of
// include/rs_accel.h. Replaces the modeled accelerator of the reference
// (AcceleratorSpec + accel_service_time, proj/include/recsim/platform.hpp:48-68,
// proj/src/platform.cpp:113-136) with real execution.
//
// Execution model:
//  * tables and weights are device-resident for the handle's lifetime
//    (one allocation for all T tables, [T][rows][D] fp32);
//  * each CUDA stream that calls in gets a scratch SLOT (staging buffers,
//    activations, a device query descriptor) and a CUDA graph captured once
//    for that slot. All kernels read the item count S from the device
//    descriptor, so one graph serves every query size <= max_query_size;
//  * a call = async H2D of the query's dense features and indices (pinned
//    host memory) + 16-byte descriptor update + cudaGraphLaunch + async D2H
//    of the logits and the error word, all on the caller's stream.
//  * the descriptor update has value semantics (event-guarded pinned ring,
//    or cuStreamBatchMemOp writes), so the host may run any number of
//    queries ahead of the GPU.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <thread>
#include <memory>
#include <mutex>
#include <vector>

#include "../kernels/common.cuh"
#include "../kernels/kernels.hpp"
#include "internal.hpp"

namespace rs {
bool gru_supported(int D, int H);

namespace {

#define RS_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      raise(e_ == cudaErrorMemoryAllocation ? RS_E_OOM : RS_E_CUDA,                    \
            std::string(#call) + ": " + cudaGetErrorString(e_));                       \
  } while (0)

constexpr int kDescRing = 256;

using BatchMemOpFn = CUresult (*)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

#if RS_EXPERIMENTS
BatchMemOpFn batch_memop_fn() {
  static BatchMemOpFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<BatchMemOpFn>(p);
  }();
  return fn;
}
#endif

struct FcLayer {
  int64_t in = 0, out = 0, ldk = 0;
  int relu = 0;
  int batch = 1;
  float* W = nullptr;  // [batch][out][ldk]
  float* b = nullptr;  // [batch][out]
  // RS_FC_BF16: the same weights rounded to bfloat16, [batch][out][ldk16],
  // ldk16 = round8(in) (16-byte rows for TMA)
  uint16_t* W16 = nullptr;
  int64_t ldk16 = 0;
};

struct Slot {
  cudaStream_t cap = nullptr;  // capture stream
  QDesc* d_q = nullptr;
  int* d_err = nullptr;
  int* h_err = nullptr;        // pinned error word read-back
  QDesc* h_q = nullptr;        // pinned descriptor ring [kDescRing]
  cudaEvent_t q_ev[kDescRing] = {};  // last copy out of each ring entry
  int ring = 0;
  float* dense_stage = nullptr;
  float* dense_raw = nullptr;   // contiguous H2D landing zone for strided dense
  int64_t* idx_stage = nullptr;
  int32_t* idx32_stage = nullptr;  // H2D landing zone of RS_INDEX_I32 queries
  uint8_t* landing = nullptr;      // one-DMA landing zone for packed host inputs
  const int32_t* idx32_src = nullptr;  // where this query's int32 indices landed
  SplitKPool splitk;                   // split-K workspaces of this slot's graphs
  float* act[2] = {nullptr, nullptr};
  float* pooled = nullptr;
  float* X = nullptr;
  float* pact[2] = {nullptr, nullptr};
  // RS_FC_BF16 activations: the stacks' inputs and hidden layers as bfloat16
  uint16_t* X16 = nullptr;
  uint16_t* dense16 = nullptr;
  uint16_t* act16[2] = {nullptr, nullptr};
  uint16_t* pact16[2] = {nullptr, nullptr};
  float* out = nullptr;
  cudaGraphExec_t graph[7] = {};  // GraphKind
  int kernels[7] = {};
  // kGraphWide: capturing it (pairs), its CTA-pair layers, whether one of them
  // is a single stack, and the smallest query it serves
  bool pairs = false;
  bool wide_tried = false;
  // a lane of the pipelined queue: its graphs capture without PDL edges
  // (cfg3 RMC2 -1.2%, cfg3 RMC3 -2.9%, zoo RMC3 -5.9% us/query) and with one
  // resident wave of gather CTAs (cfg3 RMC2 -1.6%, RMC1 -7%); DESIGN.md §5a
  bool lane = false;
  int pair_layers = 0;
  bool pair_single = false;
  int64_t pair_min = 0;
  int tc_layers = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // event-record nodes around the embedding kernel (pool graph and the
  // stage-timed forward graph) and around the predict stack (stage-timed)
  cudaEvent_t kev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ready = nullptr, free = nullptr;  // pipelined queue hand-off
  cudaEvent_t computed = nullptr;               // forward done (result copy may start)
  cudaStream_t cap2 = nullptr;                  // capture: parallel graph branch
  // SM-partitioned slots (rs_forward_many lanes when the device is split):
  // capture streams on the dense and the gather green contexts
  cudaStream_t gcap_d = nullptr, gcap_e = nullptr;
  int emb_sms = 0, dense_sms = 0;  // SMs the gather / dense grids are sized for
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<void*> allocs;
};

}  // namespace
}  // namespace rs

struct rs_accel {
  rs_model_desc m{};
  rs_init_desc init{};
  int device = 0;
  int sm_count = 0;
  int64_t l2_bytes = 0;
  cudaStream_t own = nullptr;
  // geometry
  int64_t T = 0, L = 0, D = 0, H = 0, stacks = 1;
  int64_t dense_in = 0, ld_dense = 0, dense_out = 0;
  int64_t p_in = 0, ld_x = 0, out_dim = 0, out_w = 0;
  int64_t pooled_dim = 0;
  int64_t max_dense_w = 0, max_pred_w = 0;
  int64_t ld_x16 = 0, ld_dense16 = 0;  // bf16 row strides (round8)
  // device state
  float* tables = nullptr;
  // L2-persisting hot block: rows [0, hot_rows) of every table, [T][hot_rows][D]
  float* hot = nullptr;
  int64_t hot_rows = 0;
  size_t hot_bytes = 0;
  std::vector<rs::FcLayer> dense_layers, pred_layers;
  float* att_w = nullptr;
  float *gru_wih = nullptr, *gru_whh = nullptr, *gru_bih = nullptr, *gru_bhh = nullptr,
        *gru_watt = nullptr;
  std::vector<void*> allocs;
  int64_t table_bytes = 0, weight_bytes = 0;
  std::mutex mu;
  std::map<cudaStream_t, std::unique_ptr<rs::Slot>> slots;
  // rs_forward_many queue: `depth` lanes, each a compute stream + a slot
  static constexpr int kMaxLanes = 16;
  int depth = 2;
  int64_t merge_queries = 1;  // RS_OPT_MERGE_QUERIES (1 = one query per launch)
  int stage_timing = 0;       // RS_OPT_STAGE_TIMING
  // RS_OPT_CTA_PAIRS (RS_TC2=1 sets the default, for tools/env_sweep.py)
  int cta_pairs = [] {
    const char* e = getenv("RS_TC2");
    return e && atoi(e) == 1 ? 1 : 0;
  }();
  // Uniform shared-memory carveout (% of the unified L1/shared array) set on
  // every kernel node of the forward graphs, with the tcgen05 FC tiles held
  // to a shared-memory budget that fits it: an SM never has to drain to
  // switch its L1/shared split when a 192 KB FC tile lands between gather
  // CTAs, and the gathers keep their L1 for in-flight loads.
  // 0 = the driver's per-kernel choice and the deep FC tiles.
  int carveout_pct = 0;
  int fc_smem_kb = 0;         // FC tile shared-memory budget (0 = none)
  int inter_threads = 256;    // interaction CTA size (64: co-resident with the gathers)
  int pair_capped = 0;        // CTA-pair FC tiles within the capped shared memory
  int pairs_all = 0;          // CTA-pair FC tiles (4-deep) in every tcgen05 graph
  std::unique_ptr<rs::Slot> pipe[kMaxLanes];
  cudaStream_t lane[kMaxLanes] = {};
  cudaEvent_t lane_join[kMaxLanes] = {};
  cudaStream_t copy = nullptr;
  cudaStream_t copy_more[3] = {};  // further copy streams: queries rotate (RS_COPY_STREAMS)
  // device->host result copies of host queries, off the lanes (RS_D2H_STREAMS)
  cudaStream_t d2h[2] = {};
  cudaEvent_t d2h_join[2] = {};
  cudaEvent_t copy_gate = nullptr;
  std::mutex many_mu;
  std::vector<cudaEvent_t> evpool, evstart;
  std::map<int64_t, double> service_memo;
  rs::BatchMemOpFn memops = nullptr;  // null: pageable-copy descriptor writes
  // SM partition for the pipelined queue (green contexts): the gathers run
  // on emb_sms SMs, the latency-bound dense kernels on part_dense_sms.
  CUgreenCtx g_dense = nullptr, g_emb = nullptr;
  int part_dense_sms = 0, part_emb_sms = 0;
};

namespace rs {
namespace {

void* dmalloc(rs_accel* a, std::vector<void*>& list, size_t bytes, bool zero = true) {
  void* p = nullptr;
  RS_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  list.push_back(p);
  if (zero) RS_CUDA(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
  (void)a;
  return p;
}

void upload(void* dst, const std::vector<float>& v) {
  RS_CUDA(cudaMemcpy(dst, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice));
}

float fan_bound(int64_t fan_in) { return 1.0f / sqrtf(static_cast<float>(fan_in)); }

// fp32 -> bfloat16 bits, round to nearest even (finite inputs)
uint16_t to_bf16_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// Weights and biases of one FC stack layer, [batch][out][ldk] with zero pad.
FcLayer make_layer(rs_accel* a, int64_t in, int64_t out, int relu, int batch,
                   uint64_t (*wid)(int64_t, int64_t), uint64_t (*bid)(int64_t, int64_t),
                   int64_t layer) {
  FcLayer f;
  f.in = in; f.out = out; f.ldk = round_up(in, 4); f.relu = relu; f.batch = batch;
  const float bound = fan_bound(in);
  std::vector<float> w((size_t)(batch * out * f.ldk), 0.f), b((size_t)(batch * out));
  for (int z = 0; z < batch; ++z) {
    const uint64_t kw = stream_key(a->init.seed, wid(z, layer));
    const uint64_t kb = stream_key(a->init.seed, bid(z, layer));
    for (int64_t o = 0; o < out; ++o) {
      for (int64_t i = 0; i < in; ++i)
        w[(size_t)((z * out + o) * f.ldk + i)] = param(kw, (uint64_t)(o * in + i), bound);
      b[(size_t)(z * out + o)] = param(kb, (uint64_t)o, bound);
    }
  }
  f.W = static_cast<float*>(dmalloc(a, a->allocs, w.size() * sizeof(float), false));
  f.b = static_cast<float*>(dmalloc(a, a->allocs, b.size() * sizeof(float), false));
  upload(f.W, w);
  upload(f.b, b);
  a->weight_bytes += (int64_t)((w.size() + b.size()) * sizeof(float));
  if (a->init.fc_mode == RS_FC_BF16) {
    f.ldk16 = round_up(in, 8);
    std::vector<uint16_t> h((size_t)(batch * out * f.ldk16), 0);
    for (int z = 0; z < batch; ++z)
      for (int64_t o = 0; o < out; ++o)
        for (int64_t i = 0; i < in; ++i)
          h[(size_t)((z * out + o) * f.ldk16 + i)] =
              to_bf16_bits(w[(size_t)((z * out + o) * f.ldk + i)]);
    f.W16 = static_cast<uint16_t*>(dmalloc(a, a->allocs, h.size() * 2, false));
    RS_CUDA(cudaMemcpy(f.W16, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
    a->weight_bytes += (int64_t)(h.size() * 2);
  }
  return f;
}

uint64_t dense_wid(int64_t, int64_t l) { return id_dense_w(l); }
uint64_t dense_bid(int64_t, int64_t l) { return id_dense_b(l); }
uint64_t pred_wid(int64_t s, int64_t l) { return id_pred_w(s, l); }
uint64_t pred_bid(int64_t s, int64_t l) { return id_pred_b(s, l); }

std::vector<float> fill_param(uint64_t seed, uint64_t id, int64_t n, float bound) {
  std::vector<float> v((size_t)n);
  const uint64_t k = stream_key(seed, id);
  for (int64_t i = 0; i < n; ++i) v[(size_t)i] = param(k, (uint64_t)i, bound);
  return v;
}

// L2 persistence for skewed (Zipf) index streams: rows
// [0, hot_rows) of every table are copied into one contiguous block that an
// access-policy window keeps in the persisting L2 set-aside, so hot rows stay
// resident while the cold gathers stream past them. A pure copy — the SLS
// result does not depend on which of the two copies a row is read from.
struct HotDevice {
  int users = 0;
  size_t saved_limit = 0;
};
std::mutex& hot_mu() {
  static std::mutex m;
  return m;
}
std::map<int, HotDevice>& hot_devices() {
  static std::map<int, HotDevice> d;
  return d;
}

void setup_hot(rs_accel* a) {
  cudaDeviceProp prop;
  RS_CUDA(cudaGetDeviceProperties(&prop, a->device));
  size_t want = (size_t)a->init.l2_persist_mb << 20;
  want = std::min(want, (size_t)prop.persistingL2CacheMaxSize);
  want = std::min(want, (size_t)prop.accessPolicyMaxWindowSize);
  const size_t per_row = (size_t)a->T * a->D * sizeof(float);  // one row of every table
  const int64_t hr = std::min<int64_t>(a->init.rows_per_table, (int64_t)(want / per_row));
  if (hr < 1) return;
  a->hot_rows = hr;
  a->hot_bytes = (size_t)hr * per_row;
  a->hot = static_cast<float*>(dmalloc(a, a->allocs, a->hot_bytes, false));
  const size_t w = (size_t)hr * a->D * sizeof(float);
  RS_CUDA(cudaMemcpy2DAsync(a->hot, w, a->tables, (size_t)a->init.rows_per_table * a->D * sizeof(float),
                            w, (size_t)a->T, cudaMemcpyDeviceToDevice, a->own));
  size_t cur = 0;
  RS_CUDA(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
  std::lock_guard<std::mutex> g(hot_mu());
  HotDevice& hd = hot_devices()[a->device];
  if (hd.users++ == 0) hd.saved_limit = cur;  // the first hot handle remembers the limit
  if (cur < a->hot_bytes) RS_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, a->hot_bytes));
}

// The last hot-block handle of a device drops the persisting lines and puts
// the set-aside limit back; earlier ones leave other handles' blocks alone.
void release_hot(rs_accel* a) {
  std::lock_guard<std::mutex> g(hot_mu());
  HotDevice& hd = hot_devices()[a->device];
  if (--hd.users > 0) return;
  cudaCtxResetPersistingL2Cache();
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, hd.saved_limit);
}


void build_model(rs_accel* a) {
  const rs_model_desc& m = a->m;
  a->T = m.num_tables;
  a->L = m.lookups_per_table;
  a->D = m.embedding_dim;
  a->H = m.recurrent_hidden_dim;
  a->stacks = m.num_parallel_predict_stacks;
  a->dense_in = m.dense_input_dim;
  a->ld_dense = round_up(std::max<int64_t>(a->dense_in, 1), 4);
  a->dense_out = dense_out_dim(m);
  a->p_in = predict_input_dim(m);
  a->ld_x = round_up(a->p_in, 4);
  a->ld_x16 = round_up(a->p_in, 8);
  a->ld_dense16 = round_up(std::max<int64_t>(a->dense_in, 1), 8);
  a->out_dim = m.predict_fc.dims[m.predict_fc.n - 1];
  a->out_w = a->stacks * a->out_dim;
  switch (m.pooling) {
    case RS_POOL_SUM: a->pooled_dim = a->T * a->D; break;
    case RS_POOL_CONCAT: a->pooled_dim = a->T * a->L * a->D; break;
    case RS_POOL_ATTENTION_FC: a->pooled_dim = a->T * a->D; break;
    case RS_POOL_ATTENTION_RNN: a->pooled_dim = a->T * a->H; break;
  }
  if (m.pooling == RS_POOL_SUM && m.has_dense_fc && a->T > 0 && a->dense_out != a->D)
    raise(RS_E_INVALID,
          "dot interaction needs the dense stack output width to equal embedding_dim "
          "(SURVEY.md D2; the reference never checks this)");
  if (m.pooling == RS_POOL_ATTENTION_FC && a->T > 0 && !din_supported(a->D))
    raise(RS_E_INVALID, "AttentionFC requires a power-of-two embedding_dim");
  if (m.pooling == RS_POOL_ATTENTION_RNN && a->T > 0 && !gru_supported((int)a->D, (int)a->H))
    raise(RS_E_INVALID, "AttentionRNN shape unsupported (needs embedding_dim % 4 == 0)");
  if (a->T > 0 && a->init.rows_per_table < 1) raise(RS_E_INVALID, "rows_per_table < 1");

  // tables
  if (a->T > 0) {
    a->table_bytes = a->T * a->init.rows_per_table * a->D * (int64_t)sizeof(float);
    a->tables = static_cast<float*>(dmalloc(a, a->allocs, (size_t)a->table_bytes, false));
    launch_init_tables(a->tables, a->T, a->init.rows_per_table, a->D, a->init.seed,
                       a->sm_count, a->own);
    RS_CUDA(cudaGetLastError());
    if (m.pooling == RS_POOL_SUM && a->init.l2_persist_mb > 0) setup_hot(a);
  }
  // dense stack: ReLU after every layer (DLRM bottom MLP)
  if (m.has_dense_fc) {
    int64_t in = a->dense_in;
    for (int l = 0; l < m.dense_fc.n; ++l) {
      a->dense_layers.push_back(make_layer(a, in, m.dense_fc.dims[l], 1, 1, dense_wid, dense_bid, l));
      in = m.dense_fc.dims[l];
      a->max_dense_w = std::max(a->max_dense_w, round_up(in, 4));
    }
  }
  // predict stacks: ReLU on hidden layers, identity on the last (logits)
  {
    int64_t in = a->p_in;
    for (int l = 0; l < m.predict_fc.n; ++l) {
      const int relu = l + 1 < m.predict_fc.n ? 1 : 0;
      a->pred_layers.push_back(make_layer(a, in, m.predict_fc.dims[l], relu, (int)a->stacks,
                                          pred_wid, pred_bid, l));
      in = m.predict_fc.dims[l];
      a->max_pred_w = std::max(a->max_pred_w, round_up(in, 4));
    }
  }
  if (m.pooling == RS_POOL_ATTENTION_FC && a->T > 0) {
    std::vector<float> w;
    for (int64_t t = 0; t < a->T; ++t) {
      auto v = fill_param(a->init.seed, id_att_w(t), a->D * a->D, fan_bound(a->D));
      w.insert(w.end(), v.begin(), v.end());
    }
    a->att_w = static_cast<float*>(dmalloc(a, a->allocs, w.size() * 4, false));
    upload(a->att_w, w);
    a->weight_bytes += (int64_t)w.size() * 4;
  }
  if (m.pooling == RS_POOL_ATTENTION_RNN && a->T > 0) {
    const int64_t H3 = 3 * a->H;
    std::vector<float> wih, whh, bih, bhh, watt;
    for (int64_t t = 0; t < a->T; ++t) {
      auto p0 = fill_param(a->init.seed, id_gru(t, 0), H3 * a->D, fan_bound(a->H));
      auto p1 = fill_param(a->init.seed, id_gru(t, 1), H3 * a->H, fan_bound(a->H));
      auto p2 = fill_param(a->init.seed, id_gru(t, 2), H3, fan_bound(a->H));
      auto p3 = fill_param(a->init.seed, id_gru(t, 3), H3, fan_bound(a->H));
      auto p4 = fill_param(a->init.seed, id_gru(t, 4), a->D * a->D, fan_bound(a->D));
      wih.insert(wih.end(), p0.begin(), p0.end());
      whh.insert(whh.end(), p1.begin(), p1.end());
      bih.insert(bih.end(), p2.begin(), p2.end());
      bhh.insert(bhh.end(), p3.begin(), p3.end());
      watt.insert(watt.end(), p4.begin(), p4.end());
    }
    auto put = [&](float*& dst, const std::vector<float>& v) {
      dst = static_cast<float*>(dmalloc(a, a->allocs, v.size() * 4, false));
      upload(dst, v);
      a->weight_bytes += (int64_t)v.size() * 4;
    };
    put(a->gru_wih, wih); put(a->gru_whh, whh); put(a->gru_bih, bih);
    put(a->gru_bhh, bhh); put(a->gru_watt, watt);
    GruArgs g{};
    g.T = (int)a->T; g.L = (int)a->L; g.D = (int)a->D; g.H = (int)a->H;
    prepare_gru(g);
    RS_CUDA(cudaGetLastError());
  }
  if (m.pooling == RS_POOL_SUM && a->T > 0) {
    const size_t smem = interaction_smem((int)a->T, (int)a->D);
    if (smem > 200 * 1024) raise(RS_E_INVALID, "too many tables for the interaction kernel");
  }
  RS_CUDA(cudaStreamSynchronize(a->own));
}

GruArgs gru_args(rs_accel* a, Slot* s, float* out, int64_t ld, int64_t off) {
  GruArgs g{};
  g.tables = a->tables; g.rows = a->init.rows_per_table;
  g.T = (int)a->T; g.L = (int)a->L; g.D = (int)a->D; g.H = (int)a->H;
  g.w_ih = a->gru_wih; g.w_hh = a->gru_whh; g.b_ih = a->gru_bih; g.b_hh = a->gru_bhh;
  g.w_att = a->gru_watt; g.augru = a->init.rnn_cell == RS_RNN_AUGRU ? 1 : 0;
  g.out = out; g.ld_out = ld; g.col_off = off; g.err = s->d_err;
  return g;
}

// Enqueue the pooling stage writing into out[item*ld + off ...].
void enqueue_pooling(rs_accel* a, Slot* s, float* out, int64_t ld, int64_t off, bool tc,
                     cudaStream_t st) {
  const rs_model_desc& m = a->m;
  const int64_t maxS = a->init.max_query_size;
  const int64_t rows = a->init.rows_per_table;
  if (a->T == 0) return;
  switch (m.pooling) {
    case RS_POOL_SUM:
      launch_sls_sum(s->d_q, a->tables, rows, (int)a->T, (int)a->L, (int)a->D, out + off, ld,
                     s->d_err, maxS, s->emb_sms, st, a->hot, a->hot_rows);
      break;
    case RS_POOL_CONCAT:
      launch_gather_concat(s->d_q, a->tables, rows, (int)a->T, (int)a->L, (int)a->D, out, ld,
                           off, s->d_err, maxS, s->emb_sms, st);
      break;
    case RS_POOL_ATTENTION_FC:
      launch_din_pool(s->d_q, a->tables, rows, (int)a->T, (int)a->L, (int)a->D, a->att_w, out,
                      ld, off, s->d_err, maxS, s->emb_sms, st);
      break;
    case RS_POOL_ATTENTION_RNN: {
      GruArgs g = gru_args(a, s, out, ld, off);
      // tensor-core recurrence in the tcgen05 graph, FFMA recurrence otherwise
      if (!(tc && launch_gru_tc(s->d_q, g, maxS, st))) launch_gru(s->d_q, g, maxS, s->emb_sms, st);
      break;
    }
  }
}

// One FC stack: layer l reads `in` and writes the next buffer; the last layer
// writes `final_out`.
// RS_FUSE_LAST=0 keeps the narrow final layer as its own kernel.
bool fuse_enabled() {
  const char* v = getenv("RS_FUSE_LAST");
  return !v || atoi(v) != 0;
}

// RS_DISCARD (default 1): dead intermediates are dropped from L2 with
// discard.global.L2 instead of being written back to DRAM (pooled sums after
// the interaction, FC activations after their only reader): in the pipelined
// queue those write-backs turn the gather's read stream around
// (tools/range_traffic.py: 1.25 -> 0.58 GB written per 256 queries)
bool discard_enabled() {
  const char* v = getenv("RS_DISCARD");
  return !v || atoi(v) != 0;
}

// a layer of the wide graph planned on CTA pairs (fc_tc2_kernel)
void note_pair(Slot* s, const TcPlan& p, const FcArgs& args) {
  if (p.cfg != 5) return;
  ++s->pair_layers;
  if (args.batch == 1) s->pair_single = true;
}

int enqueue_stack(rs_accel* a, Slot* s, const std::vector<FcLayer>& layers, const float* in0,
                  int64_t ld_in0, int64_t in0_rows, float* const* tmp, int64_t ld_tmp,
                  float* final_out, int64_t ld_final, int64_t final_sCz, bool allow_tc,
                  cudaStream_t st, bool final_to_desc = false, bool in0_discardable = false) {
  const int64_t maxS = a->init.max_query_size;
  // The whole stack as one tcgen05 kernel when every layer fits (activations
  // stay in shared memory between layers): one launch instead of one per layer.
  if (allow_tc && !layers.empty() && (int)layers.size() <= kChainMaxLayers + 1) {
    FcArgs ly[kChainMaxLayers + 1];
    for (size_t l = 0; l < layers.size(); ++l) {
      const FcLayer& f = layers[l];
      FcArgs& x = ly[l];
      x = FcArgs{};
      x.A = l == 0 ? in0 : nullptr; x.lda = ld_in0;
      x.W = f.W; x.ldw = f.ldk; x.sWz = f.out * f.ldk;
      x.bias = f.b; x.sbz = f.out;
      x.N = (int)f.out; x.K = (int)f.in; x.relu = f.relu; x.batch = f.batch;
    }
    FcArgs& fin = ly[layers.size() - 1];
    fin.C = final_out; fin.ldc = ld_final; fin.sCz = final_sCz;
    fin.c_desc = final_to_desc ? 1 : 0;
    TcChainPlan cp;
    if (tc_chain_plan(&cp, ly, (int)layers.size(), maxS, in0_rows)) {
      launch_fc_chain(s->d_q, cp, st);
      return (int)layers.size();
    }
  }
  int tc_count = 0;
  const float* in = in0;
  int64_t lda = ld_in0, sAz = 0, a_rows = in0_rows;
  for (size_t l = 0; l < layers.size(); ++l) {
    const FcLayer& f = layers[l];
    const bool last = l + 1 == layers.size();
    FcArgs args{};
    args.A = in; args.lda = lda; args.sAz = sAz;
    args.W = f.W; args.ldw = f.ldk; args.sWz = f.out * f.ldk;
    args.bias = f.b; args.sbz = f.out;
    if (last) {
      args.C = final_out; args.ldc = ld_final; args.sCz = final_sCz;
      args.c_desc = final_to_desc ? 1 : 0;
    } else {
      args.C = tmp[l & 1]; args.ldc = ld_tmp; args.sCz = maxS * ld_tmp;
    }
    args.N = (int)f.out; args.K = (int)f.in; args.relu = f.relu; args.batch = f.batch;
    args.smem_cap_kb = a->fc_smem_kb;
    args.pair_ok = s->pairs ? 1 : (a->pairs_all ? 2 : 0);
    args.pair_capped = a->pair_capped;
    bool used_tc = false;
    if (allow_tc) {
      // A narrow final layer (<= 4 outputs: the DLRM / DIN / DIEN logits)
      // after a single-N-tile layer is fused into that layer's epilogue: one
      // kernel fewer per query and no round trip of the hidden activations.
      const bool fuse = l + 2 == layers.size() && layers[l + 1].out <= kFuseMaxN2 &&
                        f.out <= 128 && fuse_enabled();
      if (fuse) {
        const FcLayer& g = layers[l + 1];
        args.single_n_tile = 1;
        args.W2 = g.W; args.ldw2 = g.ldk; args.sW2z = g.out * g.ldk;
        args.b2 = g.b; args.sb2z = g.out;
        args.C2 = final_out; args.ldc2 = ld_final; args.sC2z = final_sCz;
        args.N2 = (int)g.out; args.relu2 = g.relu; args.c2_desc = final_to_desc ? 1 : 0;
        args.skip_c = 1;
      }
      TcPlan p;
      if (tc_plan(&p, args, maxS, a_rows, &s->splitk) && (!fuse || p.n_tiles == 1)) {
        // dead-data discard (RS_DISCARD): a single-N-tile layer is the only
        // reader of its input rows (the previous layer's activations); the
        // second layer also drops the stack input, read by layer 0 only
        if (discard_enabled() && f.batch == 1 && p.n_tiles == 1 && p.splits <= 1 && l >= 1) {
          args.discard_a = 1;
          if (l == 1 && in0_discardable) {
            args.dz = in0;
            args.dz_ld = ld_in0 * 4;
          }
        }
        launch_fc_tc(s->d_q, p, args, st);
        note_pair(s, p, args);
        used_tc = true;
        ++tc_count;
        if (fuse) {
          ++tc_count;
          break;  // the final layer ran in this epilogue
        }
      } else if (fuse) {
        args.single_n_tile = 0; args.N2 = 0; args.skip_c = 0; args.W2 = nullptr;
        args.b2 = nullptr; args.C2 = nullptr;
        if (tc_plan(&p, args, maxS, a_rows, &s->splitk)) {
          launch_fc_tc(s->d_q, p, args, st);
          note_pair(s, p, args);
          used_tc = true;
          ++tc_count;
        }
      }
    }
    if (!used_tc) launch_fc_ffma(s->d_q, args, maxS, st);
    in = args.C; lda = args.ldc; sAz = args.sCz; a_rows = maxS;
  }
  return tc_count;
}

// RS_FC_BF16: the stack on tcgen05 kind::f16 layers with bf16 operands. The
// fp32 stack input (src, cols wide) is converted once into in16; layer l
// writes bf16 activations for layer l+1 whenever that layer also plans as a
// bf16 tcgen05 layer, fp32 otherwise (the logits, a fused narrow last layer's
// input stays in registers, or an FFMA successor). Returns the number of
// tcgen05 layers, or -1 (nothing enqueued) when layer 0 cannot run on bf16
// tcgen05 — the caller then uses the fp32/tf32 stack.
int enqueue_stack_bf16(rs_accel* a, Slot* s, const std::vector<FcLayer>& layers,
                       const float* src, int64_t ld_src, int64_t cols, uint16_t* in16,
                       int64_t ld_in16, uint16_t* const* tmp16, int64_t ld_tmp16,
                       float* const* tmp, int64_t ld_tmp, float* final_out, int64_t ld_final,
                       int64_t final_sCz, cudaStream_t st, bool final_to_desc, int sms) {
  const int64_t maxS = a->init.max_query_size;
  if (layers.empty() || !tc_available()) return -1;
  auto args16 = [&](const FcLayer& f, const uint16_t* A, int64_t lda, int64_t sAz) {
    FcArgs x{};
    x.A = reinterpret_cast<const float*>(A); x.lda = lda; x.sAz = sAz;
    x.W = reinterpret_cast<const float*>(f.W16); x.ldw = f.ldk16; x.sWz = f.out * f.ldk16;
    x.bias = f.b; x.sbz = f.out;
    x.N = (int)f.out; x.K = (int)f.in; x.relu = f.relu; x.batch = f.batch;
    x.ab16 = 1;
    x.smem_cap_kb = a->fc_smem_kb;
    x.pair_ok = s->pairs ? 1 : (a->pairs_all ? 2 : 0);
    x.pair_capped = a->pair_capped;
    return x;
  };
  // can layer l run as a bf16 tcgen05 layer reading A (dry-run plan)?
  auto can16 = [&](size_t l, const uint16_t* A, int64_t lda, int64_t sAz, int64_t rows) {
    if (!layers[l].W16) return false;
    FcArgs x = args16(layers[l], A, lda, sAz);
    x.C = tmp[0]; x.ldc = ld_tmp; x.sCz = maxS * ld_tmp;
    TcPlan p;
    return tc_plan(&p, x, maxS, rows, nullptr);
  };
  if (!can16(0, in16, ld_in16, 0, maxS)) return -1;
  launch_to_bf16(s->d_q, src, ld_src, in16, ld_in16, cols, maxS, sms, st);
  int tc_count = 0;
  const uint16_t* cur16 = in16;
  const float* cur32 = nullptr;
  int64_t lda = ld_in16, sAz = 0;
  for (size_t l = 0; l < layers.size(); ++l) {
    const FcLayer& f = layers[l];
    const bool last = l + 1 == layers.size();
    FcArgs args{};
    if (cur16) {
      args = args16(f, cur16, lda, sAz);
    } else {
      args.A = cur32; args.lda = lda; args.sAz = sAz;
      args.W = f.W; args.ldw = f.ldk; args.sWz = f.out * f.ldk;
      args.bias = f.b; args.sbz = f.out;
      args.N = (int)f.out; args.K = (int)f.in; args.relu = f.relu; args.batch = f.batch;
      args.smem_cap_kb = a->fc_smem_kb;
      args.pair_ok = s->pairs ? 1 : (a->pairs_all ? 2 : 0);
      args.pair_capped = a->pair_capped;
    }
    const bool fuse = l + 2 == layers.size() && layers[l + 1].out <= kFuseMaxN2 &&
                      f.out <= 128 && fuse_enabled();
    auto set_output = [&](bool fused) {
      args.c16 = 0;
      if (fused) {
        const FcLayer& g = layers[l + 1];
        args.single_n_tile = 1;
        args.W2 = g.W; args.ldw2 = g.ldk; args.sW2z = g.out * g.ldk;
        args.b2 = g.b; args.sb2z = g.out;
        args.C2 = final_out; args.ldc2 = ld_final; args.sC2z = final_sCz;
        args.N2 = (int)g.out; args.relu2 = g.relu; args.c2_desc = final_to_desc ? 1 : 0;
        args.skip_c = 1;
        args.C = tmp[l & 1]; args.ldc = ld_tmp; args.sCz = maxS * ld_tmp;
      } else if (last) {
        args.C = final_out; args.ldc = ld_final; args.sCz = final_sCz;
        args.c_desc = final_to_desc ? 1 : 0;
      } else if (can16(l + 1, tmp16[l & 1], ld_tmp16, maxS * ld_tmp16, maxS)) {
        args.C = reinterpret_cast<float*>(tmp16[l & 1]); args.ldc = ld_tmp16;
        args.sCz = maxS * ld_tmp16; args.c16 = 1;
      } else {
        args.C = tmp[l & 1]; args.ldc = ld_tmp; args.sCz = maxS * ld_tmp;
      }
    };
    set_output(fuse);
    TcPlan p;
    bool ok = tc_plan(&p, args, maxS, cur16 == in16 || cur32 == nullptr ? maxS : maxS,
                      &s->splitk) && (!fuse || p.n_tiles == 1);
    bool fused = fuse && ok;
    if (fuse && !ok) {
      args.single_n_tile = 0; args.N2 = 0; args.skip_c = 0; args.W2 = nullptr;
      args.b2 = nullptr; args.C2 = nullptr;
      set_output(false);
      ok = tc_plan(&p, args, maxS, maxS, &s->splitk);
    }
    if (ok) {
      launch_fc_tc(s->d_q, p, args, st);
      note_pair(s, p, args);
      tc_count += fused ? 2 : 1;
    } else {
      if (cur16) raise(RS_E_CUDA, "bf16 FC layer failed to plan after a bf16 producer");
      launch_fc_ffma(s->d_q, args, maxS, st);
    }
    if (fused) break;
    if (args.c16) {
      cur16 = reinterpret_cast<const uint16_t*>(args.C);
      cur32 = nullptr;
    } else {
      cur16 = nullptr;
      cur32 = args.C;
    }
    lda = args.ldc;
    sAz = args.sCz;
  }
  return tc_count;
}

// Graph kinds per slot: the embedding stage alone (rs_pooled), the whole
// forward with FFMA FC layers (small batches / fp32 parity) and the whole
// forward with tcgen05 FC layers wherever the layer shape fills a tile.
// kGraphPoolTimed: the pool graph with event-record nodes around the
// embedding kernel (rs_pooled with timing; the untimed graph stays lean)
// kGraphWide: the tcgen05 forward with the layers of >= 256 outputs on CTA
// pairs (fc_tc2_kernel, 256-row tiles), for queries that fill whole pairs.
enum GraphKind {
  kGraphPool = 0, kGraphSmall = 1, kGraphLarge = 2, kGraphPoolTimed = 3, kGraphStageTimed = 4,
  kGraphWide = 5, kGraphWideStageTimed = 6, kNumGraphs = 7
};
static_assert(kNumGraphs == sizeof(Slot::graph) / sizeof(Slot::graph[0]), "Slot::graph size");

cudaGraphExec_t capture(rs_accel* a, Slot* s, int kind, int* kernels, int* tc_layers) {
  // the queue's lane slots capture lane graphs (common.cuh capture_lane:
  // no PDL edges, one wave of gather CTAs); single-query slots keep both
  struct LaneScope {
    explicit LaneScope(bool lane) { capture_lane() = lane ? 1 : 0; }
    ~LaneScope() { capture_lane() = -1; }
  } lane_scope(s->lane);
  // A partitioned slot captures the gathers on the gather partition's stream
  // and everything else on the dense partition's; each kernel node keeps the
  // green context of the stream it was captured on, so one graph spans both.
  const bool part = s->gcap_d != nullptr;
  cudaStream_t st = part ? s->gcap_d : s->cap;
  // graphs of one slot never run concurrently (one lane stream): each capture
  // carves its split-K workspaces from the start of the slot's pool
  s->splitk.ws_used = 0;
  s->splitk.cnt_used = 0;
  cudaGraph_t g = nullptr;
  RS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const rs_model_desc& m = a->m;
  const int64_t maxS = a->init.max_query_size;
  // kGraphStageTimed: the forward graph of the handle's FC path with
  // event-record nodes around the embedding stage and around the predict
  // stack (RS_OPT_STAGE_TIMING; rs_timing.embed_ms / fc_ms)
  const bool stage_stamp = kind == kGraphStageTimed || kind == kGraphWideStageTimed;
  const bool tc = kind == kGraphLarge || kind == kGraphWide ||
                  (stage_stamp && a->init.fc_mode != RS_FC_FP32 && tc_available());
  const bool h16 = tc && a->init.fc_mode == RS_FC_BF16;  // bf16 FC stacks
  int ntc = 0;
  if (kind == kGraphPool || kind == kGraphPoolTimed) {
    // timestamps of the embedding kernel alone (rs_timing.embed_ms): external
    // event-record nodes on the kernel's own stream, right around it
    const bool stamp = kind == kGraphPoolTimed;
    auto pool = [&](cudaStream_t ps) {
      if (stamp) RS_CUDA(cudaEventRecordWithFlags(s->kev[0], ps, cudaEventRecordExternal));
      enqueue_pooling(a, s, s->pooled, a->pooled_dim, 0, a->init.fc_mode != RS_FC_FP32, ps);
      if (stamp) RS_CUDA(cudaEventRecordWithFlags(s->kev[1], ps, cudaEventRecordExternal));
    };
    if (part && a->T > 0) {
      RS_CUDA(cudaEventRecord(s->fork, st));
      RS_CUDA(cudaStreamWaitEvent(s->gcap_e, s->fork, 0));
      pool(s->gcap_e);
      RS_CUDA(cudaEventRecord(s->join, s->gcap_e));
      RS_CUDA(cudaStreamWaitEvent(st, s->join, 0));
    } else {
      pool(st);
    }
  } else {
    // diagnostic only (tools/pipe_micro.py): RS_DIAG_SKIP bit 1 drops the
    // bottom MLP, 2 the interaction, 4 the predict stack, 8 the embedding
    // stage (outputs invalid)
    const char* dsk = getenv("RS_DIAG_SKIP");
    const int skip = dsk ? atoi(dsk) : 0;
    // The dense branch (stage_dense + bottom MLP) and the embedding stage
    // are independent (they write disjoint columns of X): capture them as
    // parallel graph branches. Unpartitioned: the gather on the main stream,
    // the dense branch forked; partitioned: the gather forked onto the
    // gather partition, the dense branch on the main (dense) stream.
    const bool dense = a->dense_in > 0;
    // RS_DIAG_SERIAL=1 (diagnostic): the dense branch ahead of the gather on one stream
    const char* dser = getenv("RS_DIAG_SERIAL");
    const bool serial = dser && atoi(dser) && !part;
    const bool fork = !serial && (part ? a->T > 0 : (dense && a->T > 0));
    cudaStream_t bs = st, es = st;
    if (fork) {
      RS_CUDA(cudaEventRecord(s->fork, st));
      cudaStream_t other = part ? s->gcap_e : s->cap2;
      RS_CUDA(cudaStreamWaitEvent(other, s->fork, 0));
      if (part) es = other;
      else bs = other;
    }
    if (dense) {
      if (m.has_dense_fc) {
        launch_stage_dense(s->d_q, a->dense_in, s->dense_stage, a->ld_dense, maxS, s->dense_sms,
                           bs);
        if (!(skip & 1)) {
          const int u = h16 ? enqueue_stack_bf16(
                                  a, s, a->dense_layers, s->dense_stage, a->ld_dense, a->dense_in,
                                  s->dense16, a->ld_dense16, s->act16,
                                  round_up(std::max<int64_t>(a->max_dense_w, 8), 8), s->act,
                                  a->max_dense_w, s->X, a->ld_x, 0, bs, false, s->dense_sms)
                            : -1;
          ntc += u >= 0 ? u
                        : enqueue_stack(a, s, a->dense_layers, s->dense_stage, a->ld_dense, maxS,
                                        s->act, a->max_dense_w, s->X, a->ld_x, 0, tc, bs,
                                        false, /*in0_discardable=*/true);
        }
      } else {
        launch_stage_dense(s->d_q, a->dense_in, s->X, a->ld_x, maxS, s->dense_sms, bs);
      }
    }
    if (fork && !part) RS_CUDA(cudaEventRecord(s->join, bs));
    if (stage_stamp) RS_CUDA(cudaEventRecordWithFlags(s->kev[0], es, cudaEventRecordExternal));
    if (skip & 8) {
    } else if (m.pooling == RS_POOL_SUM) {
      if (a->T > 0) enqueue_pooling(a, s, s->pooled, a->T * a->D, 0, tc, es);
    } else {
      enqueue_pooling(a, s, s->X, a->ld_x, a->dense_out, tc, es);
    }
    if (stage_stamp) RS_CUDA(cudaEventRecordWithFlags(s->kev[1], es, cudaEventRecordExternal));
    if (fork && part) RS_CUDA(cudaEventRecord(s->join, es));
    if (fork) RS_CUDA(cudaStreamWaitEvent(st, s->join, 0));
    if (m.pooling == RS_POOL_SUM && a->T > 0 && !(skip & 2))
      launch_interaction(s->d_q, s->pooled, a->T * a->D, (int)a->T, (int)a->D, s->X, a->ld_x,
                         a->dense_out, a->dense_out + a->D, m.has_dense_fc ? 1 : 0, maxS,
                         s->dense_sms, st, tc, a->inter_threads);
    if (const char* de = getenv("RS_DIAG_EMPTY")) {
      const char* dc = getenv("RS_DIAG_EMPTY_CTAS");
      launch_diag_empty(atoi(de), dc ? atoi(dc) : 1, st);
    }
    if (stage_stamp) RS_CUDA(cudaEventRecordWithFlags(s->kev[2], st, cudaEventRecordExternal));
    if (!(skip & 4)) {
      const int u = h16 ? enqueue_stack_bf16(a, s, a->pred_layers, s->X, a->ld_x, a->p_in, s->X16,
                                             a->ld_x16, s->pact16,
                                             round_up(std::max<int64_t>(a->max_pred_w, 8), 8),
                                             s->pact, a->max_pred_w, s->out, a->out_w, a->out_dim,
                                             st, true, s->dense_sms)
                        : -1;
      ntc += u >= 0 ? u
                    : enqueue_stack(a, s, a->pred_layers, s->X, a->ld_x, maxS, s->pact,
                                    a->max_pred_w, s->out, a->out_w, a->out_dim, tc, st,
                                    /*final_to_desc=*/true, /*in0_discardable=*/true);
    }
    if (stage_stamp) RS_CUDA(cudaEventRecordWithFlags(s->kev[3], st, cudaEventRecordExternal));
  }
  cudaError_t le = cudaGetLastError();
  cudaError_t ce = cudaStreamEndCapture(st, &g);
  (void)cudaGetLastError();
  if ((le != cudaSuccess || ce != cudaSuccess) && g) cudaGraphDestroy(g);
  if (le != cudaSuccess) raise(RS_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(le));
  if (ce != cudaSuccess) raise(RS_E_CUDA, std::string("capture: ") + cudaGetErrorString(ce));
  size_t n = 0;
  RS_CUDA(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  RS_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
  int k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    RS_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeKernel) continue;
    ++k;
    if (a->hot) {  // the hot block's lines persist in L2 (setup_hot)
      cudaKernelNodeAttrValue v{};
      v.accessPolicyWindow.base_ptr = a->hot;
      v.accessPolicyWindow.num_bytes = a->hot_bytes;
      v.accessPolicyWindow.hitRatio = 1.0f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      RS_CUDA(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v));
    }
    if (a->carveout_pct > 0) {  // one shared-memory carveout for every kernel node
      cudaKernelNodeAttrValue v{};
      v.sharedMemCarveout = (unsigned)a->carveout_pct;
      RS_CUDA(cudaGraphKernelNodeSetAttribute(
          nd, cudaKernelNodeAttributePreferredSharedMemoryCarveout, &v));
    }
  }
  cudaGraphExec_t exec = nullptr;
  RS_CUDA(cudaGraphInstantiate(&exec, g,
                               prio_enabled() ? cudaGraphInstantiateFlagUseNodePriority : 0));
  RS_CUDA(cudaGraphDestroy(g));
  if (kernels) *kernels = k;
  if (tc_layers) *tc_layers = ntc;
  return exec;
}

#if RS_EXPERIMENTS  // green-context SM partitions: measured slower
// Green-context entry points (driver API, fetched at run time: no -lcuda).
struct GreenApi {
  CUresult (*get_res)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned,
                    unsigned) = nullptr;
  CUresult (*gen_desc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
  CUresult (*create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*destroy)(CUgreenCtx) = nullptr;
  CUresult (*stream)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
  bool ok = false;
};

const GreenApi& green_api() {
  static GreenApi g = [] {
    GreenApi r;
    auto get = [](const char* name) -> void* {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        return nullptr;
      return p;
    };
    r.get_res = reinterpret_cast<decltype(r.get_res)>(get("cuDeviceGetDevResource"));
    r.split = reinterpret_cast<decltype(r.split)>(get("cuDevSmResourceSplitByCount"));
    r.gen_desc = reinterpret_cast<decltype(r.gen_desc)>(get("cuDevResourceGenerateDesc"));
    r.create = reinterpret_cast<decltype(r.create)>(get("cuGreenCtxCreate"));
    r.destroy = reinterpret_cast<decltype(r.destroy)>(get("cuGreenCtxDestroy"));
    r.stream = reinterpret_cast<decltype(r.stream)>(get("cuGreenCtxStreamCreate"));
    r.ok = r.get_res && r.split && r.gen_desc && r.create && r.destroy && r.stream;
    return r;
  }();
  return g;
}

// Split the device for the pipelined queue: `dense_sms` SMs (a multiple of 8
// on sm_90+) for the latency-bound dense kernels, the rest for the gathers.
// Returns false (queue stays unpartitioned) if green contexts are unavailable.
bool make_partition(rs_accel* a, int dense_sms) {
  const GreenApi& ga = green_api();
  if (!ga.ok || dense_sms <= 0) return false;
  CUdevResource all, grp, rest;
  unsigned n = 1;
  if (ga.get_res((CUdevice)a->device, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return false;
  if (ga.split(&grp, &n, &all, &rest, 0, (unsigned)dense_sms) != CUDA_SUCCESS || n != 1)
    return false;
  CUdevResourceDesc dd, de;
  if (ga.gen_desc(&dd, &grp, 1) != CUDA_SUCCESS || ga.gen_desc(&de, &rest, 1) != CUDA_SUCCESS)
    return false;
  if (ga.create(&a->g_dense, dd, (CUdevice)a->device, CU_GREEN_CTX_DEFAULT_STREAM) !=
      CUDA_SUCCESS)
    return false;
  if (ga.create(&a->g_emb, de, (CUdevice)a->device, CU_GREEN_CTX_DEFAULT_STREAM) !=
      CUDA_SUCCESS) {
    ga.destroy(a->g_dense);
    a->g_dense = nullptr;
    return false;
  }
  a->part_dense_sms = (int)grp.sm.smCount;
  a->part_emb_sms = (int)rest.sm.smCount;
  return true;
}

#endif  // RS_EXPERIMENTS

std::unique_ptr<Slot> make_slot(rs_accel* a, bool partitioned = false) {
  RS_CUDA(cudaSetDevice(a->device));
  auto s = std::make_unique<Slot>();
  s->lane = partitioned;  // the pipelined queue's lane slots are the partitioned ones
  const int64_t maxS = a->init.max_query_size;
  RS_CUDA(cudaStreamCreateWithFlags(&s->cap, cudaStreamNonBlocking));
  s->emb_sms = s->dense_sms = a->sm_count;
#if RS_EXPERIMENTS
  if (partitioned && a->g_dense) {
    const GreenApi& ga = green_api();
    CUstream sd = nullptr, se = nullptr;
    if (ga.stream(&sd, a->g_dense, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
        ga.stream(&se, a->g_emb, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
      raise(RS_E_CUDA, "cuGreenCtxStreamCreate failed");
    s->gcap_d = reinterpret_cast<cudaStream_t>(sd);
    s->gcap_e = reinterpret_cast<cudaStream_t>(se);
    s->emb_sms = a->part_emb_sms;
    s->dense_sms = a->part_dense_sms;
  }
#else
  (void)partitioned;
#endif
  s->d_q = static_cast<QDesc*>(dmalloc(a, s->allocs, sizeof(QDesc)));
  RS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->h_q), sizeof(QDesc) * kDescRing,
                        cudaHostAllocPortable));
  RS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->h_err), sizeof(int), cudaHostAllocPortable));
  s->h_err[0] = 0;
  s->d_err = static_cast<int*>(dmalloc(a, s->allocs, sizeof(int)));
  s->dense_stage = static_cast<float*>(dmalloc(a, s->allocs, (size_t)(maxS * a->ld_dense * 4)));
  s->dense_raw = static_cast<float*>(
      dmalloc(a, s->allocs, (size_t)(maxS * std::max<int64_t>(a->dense_in, 1) * 4), false));
  s->idx_stage = static_cast<int64_t*>(
      dmalloc(a, s->allocs, (size_t)(maxS * std::max<int64_t>(a->T * a->L, 1) * 8)));
  s->idx32_stage = static_cast<int32_t*>(
      dmalloc(a, s->allocs, (size_t)(maxS * std::max<int64_t>(a->T * a->L, 1) * 4), false));
  s->landing = static_cast<uint8_t*>(
      dmalloc(a, s->allocs, (size_t)(maxS * (a->dense_in * 4 + a->T * a->L * 8) + 16), false));
  {
    // split-K scratch, sized for the long-K layers of this model (K >= 1024)
    size_t ws = 0, cnt = 0;
    auto need = [&](const std::vector<FcLayer>& ls) {
      for (const FcLayer& f : ls)
        if (f.in >= 1024) {
          const size_t tiles = (size_t)f.batch * ((maxS + 127) / 128) * ((f.out + 63) / 64);
          ws += 4 * tiles * 128 * 128;  // <= 4 splits of 128 x (BN <= 128... 256) partials
          cnt += tiles;
        }
    };
    need(a->dense_layers);
    need(a->pred_layers);
    if (ws) {
      s->splitk.ws = static_cast<float*>(dmalloc(a, s->allocs, ws * 4 * 2, false));
      s->splitk.ws_cap = ws * 2;
      s->splitk.cnt = static_cast<int*>(dmalloc(a, s->allocs, cnt * 4 * 2));
      s->splitk.cnt_cap = cnt * 2;
    }
  }
  for (int i = 0; i < 2; ++i) {
    s->act[i] = static_cast<float*>(
        dmalloc(a, s->allocs, (size_t)(maxS * std::max<int64_t>(a->max_dense_w, 4) * 4)));
    s->pact[i] = static_cast<float*>(dmalloc(
        a, s->allocs, (size_t)(a->stacks * maxS * std::max<int64_t>(a->max_pred_w, 4) * 4)));
  }
  s->pooled = static_cast<float*>(
      dmalloc(a, s->allocs, (size_t)(maxS * std::max<int64_t>(a->pooled_dim, 1) * 4)));
  s->X = static_cast<float*>(dmalloc(a, s->allocs, (size_t)(maxS * a->ld_x * 4)));
  if (a->init.fc_mode == RS_FC_BF16) {
    const int64_t wd = round_up(std::max<int64_t>(a->max_dense_w, 8), 8);
    const int64_t wp = round_up(std::max<int64_t>(a->max_pred_w, 8), 8);
    s->X16 = static_cast<uint16_t*>(dmalloc(a, s->allocs, (size_t)(maxS * a->ld_x16 * 2)));
    s->dense16 = static_cast<uint16_t*>(dmalloc(a, s->allocs, (size_t)(maxS * a->ld_dense16 * 2)));
    for (int i = 0; i < 2; ++i) {
      s->act16[i] = static_cast<uint16_t*>(dmalloc(a, s->allocs, (size_t)(maxS * wd * 2)));
      s->pact16[i] =
          static_cast<uint16_t*>(dmalloc(a, s->allocs, (size_t)(a->stacks * maxS * wp * 2)));
    }
  }
  s->out = static_cast<float*>(dmalloc(a, s->allocs, (size_t)(maxS * a->out_w * 4)));
  for (auto& e : s->ev) RS_CUDA(cudaEventCreate(&e));
  for (auto& e : s->kev) RS_CUDA(cudaEventCreate(&e));
  RS_CUDA(cudaEventCreateWithFlags(&s->ready, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&s->free, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&s->computed, cudaEventDisableTiming));
  RS_CUDA(cudaStreamCreateWithFlags(&s->cap2, cudaStreamNonBlocking));
  RS_CUDA(cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming));
  RS_CUDA(cudaDeviceSynchronize());
  s->graph[kGraphPool] = capture(a, s.get(), kGraphPool, nullptr, nullptr);
  s->graph[kGraphPoolTimed] = capture(a, s.get(), kGraphPoolTimed, nullptr, nullptr);
  // FC_AUTO routes every query size to the tcgen05 graph (measured faster
  // than the FFMA graph at every size, alone and pipelined: DESIGN.md §2);
  // the FFMA graph serves FC_FP32 and devices without tcgen05
  if (a->init.fc_mode == RS_FC_FP32 || !tc_available())
    s->graph[kGraphSmall] = capture(a, s.get(), kGraphSmall, &s->kernels[kGraphSmall], nullptr);
  if (a->init.fc_mode != RS_FC_FP32 && tc_available())
    s->graph[kGraphLarge] =
        capture(a, s.get(), kGraphLarge, &s->kernels[kGraphLarge], &s->tc_layers);
  return s;
}

Slot* get_slot(rs_accel* a, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(a->mu);
  auto it = a->slots.find(st);
  if (it != a->slots.end()) return it->second.get();
  auto s = make_slot(a);
  Slot* raw = s.get();
  a->slots.emplace(st, std::move(s));
  return raw;
}

// The two slots of the pipelined host-input queue (rs_forward_many).
Slot* get_pipe_slot(rs_accel* a, int i) {
  std::lock_guard<std::mutex> lock(a->mu);
  if (!a->pipe[i]) a->pipe[i] = make_slot(a, /*partitioned=*/true);
  if (!a->copy) RS_CUDA(cudaStreamCreateWithFlags(&a->copy, cudaStreamNonBlocking));
  for (auto& c : a->copy_more)
    if (!c) RS_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k)
    if (!a->d2h[k]) {
      RS_CUDA(cudaStreamCreateWithFlags(&a->d2h[k], cudaStreamNonBlocking));
      RS_CUDA(cudaEventCreateWithFlags(&a->d2h_join[k], cudaEventDisableTiming));
    }
  if (!a->lane[i]) {
    RS_CUDA(cudaStreamCreateWithFlags(&a->lane[i], cudaStreamNonBlocking));
    RS_CUDA(cudaEventCreateWithFlags(&a->lane_join[i], cudaEventDisableTiming));
  }
  return a->pipe[i].get();
}

void free_slot(Slot* s) {
  for (auto g : s->graph) if (g) cudaGraphExecDestroy(g);
  for (auto e : s->ev) if (e) cudaEventDestroy(e);
  for (auto e : s->kev) if (e) cudaEventDestroy(e);
  if (s->ready) cudaEventDestroy(s->ready);
  if (s->free) cudaEventDestroy(s->free);
  if (s->computed) cudaEventDestroy(s->computed);
  for (void* p : s->allocs) cudaFree(p);
  if (s->h_err) cudaFreeHost(s->h_err);
  if (s->h_q) cudaFreeHost(s->h_q);
  for (auto e : s->q_ev)
    if (e) cudaEventDestroy(e);
  if (s->cap) cudaStreamDestroy(s->cap);
  if (s->cap2) cudaStreamDestroy(s->cap2);
  if (s->fork) cudaEventDestroy(s->fork);
  if (s->join) cudaEventDestroy(s->join);
  if (s->gcap_d) cudaStreamDestroy(s->gcap_d);
  if (s->gcap_e) cudaStreamDestroy(s->gcap_e);
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

void check_query(rs_accel* a, const rs_query* q) {
  if (!q) raise(RS_E_INVALID, "null query");
  if (q->size < 1) raise(RS_E_INVALID, "query_size < 1");
  if (q->size > a->init.max_query_size) raise(RS_E_CAPACITY, "query larger than max_query_size");
  if (q->location != RS_MEM_HOST && q->location != RS_MEM_DEVICE)
    raise(RS_E_INVALID, "bad memory location");
  if (a->T > 0 && !q->indices) raise(RS_E_INVALID, "null indices");
  if (q->index_type & ~(RS_INDEX_I32 | RS_DENSE_BF16)) raise(RS_E_INVALID, "bad index_type");
}

// Stage one query's inputs for slot s on stream st: dense features into the
// bottom-MLP staging buffer (or straight into X[:, 0:dense_in] when there is
// no dense stack), indices into the slot's staging buffer (host) or by
// pointer (device), then the 16-byte device descriptor.
// Descriptor update with value semantics: four 64-bit stream writes, or a
// 32-byte copy from a pinned ring entry that is reused only after its
// previous copy executed.
void write_desc(rs_accel* a, Slot* s, const QDesc& v, cudaStream_t st) {
  if (a->memops) {
    const uint64_t vals[5] = {(uint64_t)v.S, (uint64_t)reinterpret_cast<uintptr_t>(v.idx),
                              (uint64_t)reinterpret_cast<uintptr_t>(v.dense),
                              (uint64_t)reinterpret_cast<uintptr_t>(v.out), (uint64_t)v.flags};
    CUstreamBatchMemOpParams ops[5];
    std::memset(ops, 0, sizeof(ops));
    for (int k = 0; k < 5; ++k) {
      ops[k].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
      ops[k].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
      ops[k].writeValue.address = reinterpret_cast<CUdeviceptr>(s->d_q) + 8 * k;
      ops[k].writeValue.value64 = (cuuint64_t)vals[k];
    }
    if (a->memops(reinterpret_cast<CUstream>(st), 5, ops, 0) != CUDA_SUCCESS)
      raise(RS_E_CUDA, "cuStreamBatchMemOp failed");
    return;
  }
  // Pinned ring: an entry is rewritten only after the copy that last read it
  // has executed (its event), so the host may run any distance ahead.
  const int r = s->ring;
  s->ring = (s->ring + 1) % kDescRing;
  if (s->q_ev[r]) {
    RS_CUDA(cudaEventSynchronize(s->q_ev[r]));
  } else {
    RS_CUDA(cudaEventCreateWithFlags(&s->q_ev[r], cudaEventDisableTiming));
  }
  s->h_q[r] = v;
  RS_CUDA(cudaMemcpyAsync(s->d_q, &s->h_q[r], sizeof(QDesc), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaEventRecord(s->q_ev[r], st));
}

#if RS_EXPERIMENTS  // stream-memop descriptors: measured slower
// Descriptor writes: a copy from the slot's event-guarded pinned ring
// (default; measured faster for a lone query, equal in the pipelined queue),
// or with RS_DESC_MEMOP=1 stream memory writes, used only if a test write lands.
BatchMemOpFn probe_memops(rs_accel* a) {
  BatchMemOpFn fn = batch_memop_fn();
  const char* want = getenv("RS_DESC_MEMOP");
  if (!fn || !want || !atoi(want)) return nullptr;
  uint64_t* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return nullptr;
  CUstreamBatchMemOpParams op;
  std::memset(&op, 0, sizeof(op));
  op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
  op.writeValue.address = reinterpret_cast<CUdeviceptr>(d);
  op.writeValue.value64 = 0x5eed5eed12345678ull;
  op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
  uint64_t h = 0;
  const bool ok = cudaMemsetAsync(d, 0, 8, a->own) == cudaSuccess &&
                  fn(reinterpret_cast<CUstream>(a->own), 1, &op, 0) == CUDA_SUCCESS &&
                  cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, a->own) == cudaSuccess &&
                  cudaStreamSynchronize(a->own) == cudaSuccess && h == 0x5eed5eed12345678ull;
  cudaFree(d);
  (void)cudaGetLastError();
  return ok ? fn : nullptr;
}

#endif  // RS_EXPERIMENTS

// Inputs of one query onto the slot: host buffers are copied (one contiguous
// H2D each) into the slot's landing zones; device buffers are used in place.
// The descriptor carries the item count and the dense / index / output
// pointers; the graph's stage_dense kernel places the dense rows, and for a
// device output buffer the final FC layer writes the logits straight into it.
// RS_INDEX_I32: widen the slot's int32 indices (landing zone, or the caller's
// device buffer) into the int64 staging buffer on stream st.
void widen_indices(rs_accel* a, Slot* s, const rs_query* q, cudaStream_t st) {
  if (a->T == 0 || !(q->index_type & RS_INDEX_I32)) return;
  const int64_t n = q->size * a->T * a->L;
  const int32_t* src = q->location == RS_MEM_HOST ? s->idx32_src
                                                  : reinterpret_cast<const int32_t*>(q->indices);
  launch_widen_idx(src, s->idx_stage, n, a->sm_count, st);
}

// `widen_later`: the caller launches widen_indices itself on its compute
// stream (the pipelined queue keeps kernels off the copy stream, where one
// would wait for SM slots and stall the next query's transfer).
void stage_inputs(rs_accel* a, Slot* s, const rs_query* q, bool full, cudaStream_t st,
                  float* out = nullptr, bool widen_later = false) {
  const int64_t S = q->size;
  const bool host = q->location == RS_MEM_HOST;
  QDesc v{};
  v.S = S;
  const bool bf16 = (q->index_type & RS_DENSE_BF16) != 0;
  const int64_t dense_bytes = S * a->dense_in * (bf16 ? 2 : 4);
  const bool i32 = (q->index_type & RS_INDEX_I32) != 0;
  v.flags = bf16 ? kDescDenseBf16 : 0;
  s->idx32_src = s->idx32_stage;
  if (host && full && a->dense_in > 0 && a->T > 0 && q->dense && dense_bytes % 8 == 0 &&
      reinterpret_cast<const uint8_t*>(q->indices) ==
          reinterpret_cast<const uint8_t*>(q->dense) + dense_bytes) {
    // packed host query [dense | indices] in one buffer: ONE transfer (same
    // bytes as the reference byte model, one DMA op's fixed cost instead of
    // two). Two separate pinned allocations that merely touch are rejected by
    // the copy (invalid argument, not sticky): then the two-copy path runs.
    const cudaError_t e = cudaMemcpyAsync(
        s->landing, q->dense, (size_t)(dense_bytes + S * a->T * a->L * (i32 ? 4 : 8)),
        cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      v.dense = reinterpret_cast<const float*>(s->landing);
      if (i32) {
        s->idx32_src = reinterpret_cast<const int32_t*>(s->landing + dense_bytes);
        if (!widen_later) widen_indices(a, s, q, st);
        v.idx = s->idx_stage;
      } else {
        v.idx = reinterpret_cast<const int64_t*>(s->landing + dense_bytes);
      }
      write_desc(a, s, v, st);
      return;
    }
    if (e != cudaErrorInvalidValue) RS_CUDA(e);
    (void)cudaGetLastError();
  }
  if (full && a->dense_in > 0) {
    if (!q->dense) raise(RS_E_INVALID, "null dense features");
    if (host) {
      RS_CUDA(cudaMemcpyAsync(s->dense_raw, q->dense, (size_t)dense_bytes,
                              cudaMemcpyHostToDevice, st));
      v.dense = s->dense_raw;
    } else {
      v.dense = q->dense;
    }
  }
  if (full && !host) v.out = out;
  const int64_t* idx = nullptr;
  if (a->T > 0) {
    const int64_t n = S * a->T * a->L;
    if (i32) {
      // labelled variant: int32 over the link (or in place), widened on device
      if (host)
        RS_CUDA(cudaMemcpyAsync(s->idx32_stage, q->indices, (size_t)(n * 4),
                                cudaMemcpyHostToDevice, st));
      if (!widen_later) widen_indices(a, s, q, st);
      idx = s->idx_stage;
    } else if (host) {
      RS_CUDA(cudaMemcpyAsync(s->idx_stage, q->indices, (size_t)(n * 8), cudaMemcpyHostToDevice,
                              st));
      idx = s->idx_stage;
    } else {
      idx = q->indices;
    }
  }
  v.idx = idx;
  write_desc(a, s, v, st);
}

// The wide graph (RS_OPT_CTA_PAIRS): the layers of >= 256 outputs on 256-row
// CTA-pair tiles (fc_tc2_kernel: half the weight bytes per flop of the
// one-CTA tile), captured on first use. Pairs only pay when the query fills
// them — an odd 128-row tile count leaves half a pair idle (MT-WND 640 items:
// 29.5 -> 32.7 us/query) — and, for single stacks whose 128-wide tiles would
// halve in number, only at large queries (WND 400 items -13%, 700 +6%, 1000
// +20%; batched MT-WND +6% from 400 items). In a queue of MIXED sizes the
// pair grids cost their neighbours about what they gain (MT-WND / WND
// log-normal streams +0.8% / +1.7% us/query at 16 lanes: a pair needs both
// SMs of a TPC while the other lanes' one-CTA tiles hold single SMs), so the
// option is for uniform-size queues (the configs[3] batch sweep).
// tools/env_sweep.py, profiles/r2_tc2/.
void ensure_wide(rs_accel* a, Slot* s) {
  if (s->wide_tried) return;
  s->wide_tried = true;
  const char* off = getenv("RS_TC2");  // RS_TC2=0: never (A/B runs)
  if (off && atoi(off) == 0) return;
  if (!s->graph[kGraphLarge] || a->init.max_query_size < 256) return;
  s->pairs = true;
  s->pair_layers = 0;
  s->pair_single = false;
  int wide_tc = 0;
  cudaGraphExec_t w = capture(a, s, kGraphWide, &s->kernels[kGraphWide], &wide_tc);
  s->pairs = false;
  if (s->pair_layers == 0) {
    cudaGraphExecDestroy(w);
    return;
  }
  s->graph[kGraphWide] = w;
  s->pair_min = s->pair_single ? 640 : 256;
  if (const char* pm = getenv("RS_TC2_MIN")) s->pair_min = atoll(pm);
}

cudaGraphExec_t pick_graph(rs_accel* a, Slot* s, int64_t S, bool full, bool timed = false) {
  if (!full) return s->graph[timed ? kGraphPoolTimed : kGraphPool];
  bool wide = false;
  if (a->cta_pairs && S >= 256 && ((S + 127) / 128) % 2 == 0) {
    ensure_wide(a, s);
    wide = s->graph[kGraphWide] && S >= s->pair_min;
  }
  if (timed && a->stage_timing) {
    // the stage-timed copy of the graph this query would run
    const int k = wide ? kGraphWideStageTimed : kGraphStageTimed;
    if (!s->graph[k]) {
      s->pairs = wide;
      s->graph[k] = capture(a, s, k, nullptr, nullptr);
      s->pairs = false;
    }
    return s->graph[k];
  }
  if (wide) return s->graph[kGraphWide];
  cudaGraphExec_t small = s->graph[kGraphSmall], large = s->graph[kGraphLarge];
  return large ? large : small;
}

void launch_stage(rs_accel* a, Slot* s, const rs_query* q, float* out, bool full,
                  cudaStream_t st) {
  const int64_t S = q->size;
  RS_CUDA(cudaGraphLaunch(pick_graph(a, s, S, full), st));
  if (full && q->location != RS_MEM_HOST) return;  // written in place by the final layer
  const int64_t w = full ? a->out_w : a->pooled_dim;
  const float* src = full ? s->out : s->pooled;
  RS_CUDA(cudaMemcpyAsync(out, src, (size_t)(S * w * 4),
                          q->location == RS_MEM_HOST ? cudaMemcpyDeviceToHost
                                                     : cudaMemcpyDeviceToDevice,
                          st));
}

// Errors are sticky per slot: kernels OR bits into d_err; a synchronising
// call reads, clears and reports them.
void collect_errors(Slot* s, cudaStream_t st) {
  RS_CUDA(cudaMemcpyAsync(s->h_err, s->d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  if (s->h_err[0]) {
    s->h_err[0] = 0;
    RS_CUDA(cudaMemsetAsync(s->d_err, 0, sizeof(int), st));
    RS_CUDA(cudaStreamSynchronize(st));
    raise(RS_E_INDEX, "embedding index outside [0, rows_per_table)");
  }
}

int run(rs_accel* a, const rs_query* q, float* out, void* stream, rs_timing* timing,
        bool full) {
  return guarded([&] {
    if (!a || !out) raise(RS_E_INVALID, "null argument");
    check_query(a, q);
    RS_CUDA(cudaSetDevice(a->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : a->own;
    Slot* s = get_slot(a, st);
    if (timing) RS_CUDA(cudaEventRecord(s->ev[0], st));
    stage_inputs(a, s, q, full, st, out);
    if (timing) RS_CUDA(cudaEventRecord(s->ev[1], st));
    RS_CUDA(cudaGraphLaunch(pick_graph(a, s, q->size, full, timing != nullptr), st));
    if (timing) RS_CUDA(cudaEventRecord(s->ev[2], st));
    const int64_t w = full ? a->out_w : a->pooled_dim;
    if (!full || q->location == RS_MEM_HOST)
      RS_CUDA(cudaMemcpyAsync(out, full ? s->out : s->pooled, (size_t)(q->size * w * 4),
                              q->location == RS_MEM_HOST ? cudaMemcpyDeviceToHost
                                                         : cudaMemcpyDeviceToDevice,
                              st));
    if (timing) {
      RS_CUDA(cudaEventRecord(s->ev[3], st));
      RS_CUDA(cudaEventSynchronize(s->ev[3]));
      timing->h2d_ms = elapsed(s->ev[0], s->ev[1]);
      timing->compute_ms = elapsed(s->ev[1], s->ev[2]);
      timing->d2h_ms = elapsed(s->ev[2], s->ev[3]);
      timing->total_ms = elapsed(s->ev[0], s->ev[3]);
      const bool staged = full && a->stage_timing;
      timing->embed_ms = a->T == 0 || (full && !staged) ? 0.0 : elapsed(s->kev[0], s->kev[1]);
      timing->fc_ms = staged ? elapsed(s->kev[2], s->kev[3]) : 0.0;
      collect_errors(s, st);
    }
  });
}

// RS_OPT_MERGE_QUERIES (labelled scheduler extension): stage m
// consecutive queries back to back in one slot (item offsets in arrival
// order) so one graph launch serves all of them; returns the total items.
int64_t stage_group(rs_accel* a, Slot* s, const rs_query* qs, int64_t m, cudaStream_t st) {
  const bool host = qs[0].location == RS_MEM_HOST;
  const cudaMemcpyKind kind = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const bool i32 = (qs[0].index_type & RS_INDEX_I32) != 0;
  if (qs[0].index_type & RS_DENSE_BF16)
    raise(RS_E_INVALID, "query merging does not take bf16 dense features");
  const int64_t TL = a->T * a->L;
  int64_t off = 0;
  if (!host) {
    // device-resident: one gather kernel for the whole group (no copy-engine
    // work queued behind the other lanes); int32 indices widened on the way
    GroupGather g{};
    g.m = (int)m;
    g.idx32 = i32 ? 1 : 0;
    for (int64_t k = 0; k < m; ++k) {
      if (a->dense_in > 0 && !qs[k].dense) raise(RS_E_INVALID, "null dense features");
      g.dense[k] = qs[k].dense;
      g.idx[k] = qs[k].indices;
      g.size[k] = qs[k].size;
      g.off[k] = off;
      off += qs[k].size;
    }
    launch_group_gather(g, a->dense_in, TL, s->dense_raw, s->idx_stage, a->sm_count, st);
    QDesc v{};
    v.S = off;
    v.dense = a->dense_in > 0 ? s->dense_raw : nullptr;
    v.idx = a->T > 0 ? s->idx_stage : nullptr;
    write_desc(a, s, v, st);
    return off;
  }
  for (int64_t k = 0; k < m; ++k) {
    const int64_t S = qs[k].size;
    if (a->dense_in > 0) {
      if (!qs[k].dense) raise(RS_E_INVALID, "null dense features");
      RS_CUDA(cudaMemcpyAsync(s->dense_raw + off * a->dense_in, qs[k].dense,
                              (size_t)(S * a->dense_in * 4), kind, st));
    }
    if (a->T > 0) {
      if (i32)
        RS_CUDA(cudaMemcpyAsync(s->idx32_stage + off * TL, qs[k].indices, (size_t)(S * TL * 4),
                                kind, st));
      else
        RS_CUDA(cudaMemcpyAsync(s->idx_stage + off * TL, qs[k].indices, (size_t)(S * TL * 8),
                                kind, st));
    }
    off += S;
  }
  QDesc v{};
  v.S = off;
  v.dense = a->dense_in > 0 ? s->dense_raw : nullptr;
  v.idx = a->T > 0 ? s->idx_stage : nullptr;
  v.out = nullptr;  // logits land in the slot and are split per query
  write_desc(a, s, v, st);
  return off;
}

int run_many(rs_accel* a, int64_t n, const rs_query* qs, float* const* outs, void* stream,
             double* service_ms, double* latency_ms, void* done_event = nullptr) {
  return guarded([&] {
    if (!a || !qs || !outs) raise(RS_E_INVALID, "null argument");
    if (n < 1) raise(RS_E_INVALID, "n < 1");
    const int loc = qs[0].location;
    for (int64_t i = 0; i < n; ++i) {
      check_query(a, &qs[i]);
      if (qs[i].location != loc) raise(RS_E_INVALID, "mixed memory locations in one batch");
      if (!outs[i]) raise(RS_E_INVALID, "null output");
    }
    RS_CUDA(cudaSetDevice(a->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : a->own;
    std::lock_guard<std::mutex> many_lock(a->many_mu);
    if (latency_ms && !service_ms) raise(RS_E_INVALID, "latency_ms needs service_ms");
    // Per-query completion (and staging-start) events live in a fixed ring:
    // when the ring wraps, the host harvests the oldest query's timestamps
    // (it completed long ago unless the GPU is kEvRing queries behind), so no
    // event is created inside a serving call after the first one.
    constexpr int64_t kEvRing = 4096;
    std::vector<double> t_done, t_start;
    if (service_ms) {
      auto fill = [](std::vector<cudaEvent_t>& pool, int64_t need) {
        while ((int64_t)pool.size() < need) {
          cudaEvent_t e;
          RS_CUDA(cudaEventCreate(&e));
          pool.push_back(e);
        }
      };
      fill(a->evpool, kEvRing + 1);
      if (latency_ms) fill(a->evstart, kEvRing);
      t_done.resize(n);
      if (latency_ms) t_start.resize(n);
      RS_CUDA(cudaEventRecord(a->evpool[0], st));
    }
    auto harvest = [&](int64_t j) {
      cudaEvent_t e = a->evpool[1 + j % kEvRing];
      RS_CUDA(cudaEventSynchronize(e));
      t_done[j] = elapsed(a->evpool[0], e);
      if (latency_ms) t_start[j] = elapsed(a->evpool[0], a->evstart[j % kEvRing]);
    };
    // Queries are dispatched in FIFO order round-robin over `depth` lanes
    // (compute stream + scratch slot each), so query i+1's embedding gather
    // overlaps query i's latency-bound FC tail. Host inputs are staged by one
    // copy stream that runs ahead of compute (a lane's next H2D waits only for
    // that lane's previous query to release its staging buffers).
    const int depth = a->depth;
    Slot* p[rs_accel::kMaxLanes] = {};
    for (int d = 0; d < depth; ++d) p[d] = get_pipe_slot(a, d);
    RS_CUDA(cudaEventRecord(a->copy_gate, st));
    for (int d = 0; d < depth; ++d) RS_CUDA(cudaStreamWaitEvent(a->lane[d], a->copy_gate, 0));
    // host inputs: one copy stream, or two alternating so one query's
    // per-transfer fixed costs overlap the other's transfer
    const char* cs = getenv("RS_COPY_STREAMS");
    const int ncopy = cs ? std::min(4, std::max(1, atoi(cs))) : 2;
    cudaStream_t copies[4] = {a->copy, a->copy_more[0], a->copy_more[1], a->copy_more[2]};
    if (loc == RS_MEM_HOST)
      for (int c = 0; c < ncopy; ++c) RS_CUDA(cudaStreamWaitEvent(copies[c], a->copy_gate, 0));
    // diagnostic (tools): RS_MANY_POOL_ONLY=1 runs only the embedding-stage
    // graph per query (outputs are the pooled rows), to separate the
    // gather's pipelined throughput from the FC tail's
    const char* po = getenv("RS_MANY_POOL_ONLY");
    const bool pool_only = po && atoi(po);
    // host results: copied back on separate streams (alternating), so a
    // lane's next query does not queue its kernels behind the copy and the
    // link carries both directions at once (RS_D2H_STREAMS=0: on the lane)
    const char* dse = getenv("RS_D2H_STREAMS");
    const int nd2h = loc == RS_MEM_HOST ? (dse ? std::min(2, std::max(0, atoi(dse))) : 2) : 0;
    if (nd2h)
      for (int c = 0; c < nd2h; ++c) RS_CUDA(cudaStreamWaitEvent(a->d2h[c], a->copy_gate, 0));
    const auto host_t0 = std::chrono::steady_clock::now();
    const int64_t maxS = a->init.max_query_size;
    int64_t group = 0;
    for (int64_t i = 0; i < n;) {
      // group [i, j): one query, or up to merge_queries consecutive ones of
      // the same index type whose items fit one slot
      int64_t j = i + 1, items = qs[i].size;
      while (!pool_only && j < n && j - i < a->merge_queries &&
             !(qs[i].index_type & RS_DENSE_BF16) &&
             items + qs[j].size <= maxS && qs[j].index_type == qs[i].index_type)
        items += qs[j++].size;
      const int d = (int)(group % depth);
      Slot* s = p[d];
      cudaStream_t ls = a->lane[d];
      for (int64_t k = i; k < j; ++k)
        if (service_ms && k >= kEvRing) harvest(k - kEvRing);
      cudaStream_t sst = ls;  // staging stream
      cudaStream_t ost = ls;  // stream the query's result lands on
      if (loc == RS_MEM_HOST) {
        sst = copies[group % ncopy];
        RS_CUDA(cudaStreamWaitEvent(sst, s->free, 0));
      }
      if (latency_ms)
        for (int64_t k = i; k < j; ++k) RS_CUDA(cudaEventRecord(a->evstart[k % kEvRing], sst));
      if (j - i == 1) {
        if (loc == RS_MEM_HOST) {
          stage_inputs(a, s, &qs[i], true, sst, nullptr, /*widen_later=*/true);
          RS_CUDA(cudaEventRecord(s->ready, sst));
          RS_CUDA(cudaStreamWaitEvent(ls, s->ready, 0));
          widen_indices(a, s, &qs[i], ls);
        } else {
          stage_inputs(a, s, &qs[i], true, ls, outs[i]);
        }
        if (nd2h) {
          const bool full = !pool_only;
          RS_CUDA(cudaGraphLaunch(pick_graph(a, s, qs[i].size, full), ls));
          RS_CUDA(cudaEventRecord(s->computed, ls));
          ost = a->d2h[group % nd2h];
          RS_CUDA(cudaStreamWaitEvent(ost, s->computed, 0));
          RS_CUDA(cudaMemcpyAsync(outs[i], full ? s->out : s->pooled,
                                  (size_t)(qs[i].size * (full ? a->out_w : a->pooled_dim) * 4),
                                  cudaMemcpyDeviceToHost, ost));
        } else {
          launch_stage(a, s, &qs[i], outs[i], !pool_only, ls);
        }
      } else {
        const int64_t S = stage_group(a, s, qs + i, j - i, sst);
        if (loc == RS_MEM_HOST) {
          RS_CUDA(cudaEventRecord(s->ready, sst));
          RS_CUDA(cudaStreamWaitEvent(ls, s->ready, 0));
        }
        if (loc == RS_MEM_HOST && a->T > 0 && (qs[i].index_type & RS_INDEX_I32))
          launch_widen_idx(s->idx32_stage, s->idx_stage, S * a->T * a->L, a->sm_count, ls);
        RS_CUDA(cudaGraphLaunch(pick_graph(a, s, S, true), ls));
        int64_t off = 0;
        for (int64_t k = i; k < j; ++k) {
          RS_CUDA(cudaMemcpyAsync(outs[k], s->out + off * a->out_w,
                                  (size_t)(qs[k].size * a->out_w * 4),
                                  loc == RS_MEM_HOST ? cudaMemcpyDeviceToHost
                                                     : cudaMemcpyDeviceToDevice,
                                  ls));
          off += qs[k].size;
        }
      }
      RS_CUDA(cudaEventRecord(s->free, ost));
      if (service_ms)
        for (int64_t k = i; k < j; ++k) RS_CUDA(cudaEventRecord(a->evpool[1 + k % kEvRing], ost));
      ++group;
      i = j;
    }
    for (int d = 0; d < depth; ++d) {
      RS_CUDA(cudaEventRecord(a->lane_join[d], a->lane[d]));
      RS_CUDA(cudaStreamWaitEvent(st, a->lane_join[d], 0));
    }
    for (int c = 0; c < nd2h; ++c) {
      RS_CUDA(cudaEventRecord(a->d2h_join[c], a->d2h[c]));
      RS_CUDA(cudaStreamWaitEvent(st, a->d2h_join[c], 0));
    }
    // the caller's completion stamp: recorded once every query finished, so
    // it excludes the host's timestamp harvest below
    if (done_event) RS_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(done_event), st));
    if (const char* tr = getenv("RS_TRACE_ENQUEUE")) {
      if (atoi(tr))
        fprintf(stderr, "rs_forward_many: n=%lld enqueue %.3f ms (%.2f us/query)\n",
                (long long)n,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                          host_t0).count(),
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() -
                                                          host_t0).count() / (double)n);
    }
    if (service_ms) {
      RS_CUDA(cudaStreamSynchronize(st));
      for (int64_t j = std::max<int64_t>(0, n - kEvRing); j < n; ++j) harvest(j);
      // Deliveries are in FIFO order: query i is delivered when it and every
      // earlier query completed; service = gap between deliveries.
      double prev = 0;
      for (int64_t i = 0; i < n; ++i) {
        const double done = std::max(prev, t_done[i]);
        service_ms[i] = done - prev;
        prev = done;
        // residence in the accelerator: input staging start -> completion
        if (latency_ms) latency_ms[i] = t_done[i] - t_start[i];
      }
      for (int d = 0; d < depth; ++d) collect_errors(p[d], st);
    }
  });
}

}  // namespace
}  // namespace rs

using namespace rs;

extern "C" int rs_accel_set_option(rs_accel* a, int32_t option, int64_t value) {
  return guarded([&] {
    if (!a) raise(RS_E_INVALID, "null handle");
    switch (option) {
      case RS_OPT_MERGE_QUERIES:
        if (value < 1 || value > kMaxGroup)
          raise(RS_E_INVALID, "merge_queries must be in [1, 64]");
        a->merge_queries = value;
        break;
      case RS_OPT_STAGE_TIMING:
        if (value != 0 && value != 1) raise(RS_E_INVALID, "stage_timing must be 0 or 1");
        a->stage_timing = (int)value;
        break;
      case RS_OPT_CTA_PAIRS:
        if (value != 0 && value != 1) raise(RS_E_INVALID, "cta_pairs must be 0 or 1");
        a->cta_pairs = (int)value;
        break;
      default:
        raise(RS_E_INVALID, "unknown option");
    }
  });
}

extern "C" int rs_device_count(int* out) {
  return guarded([&] {
    if (!out) raise(RS_E_INVALID, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    *out = n;
  });
}

extern "C" int rs_alloc_pinned(size_t bytes, void** out) {
  return guarded([&] {
    if (!out) raise(RS_E_INVALID, "null argument");
    RS_CUDA(cudaHostAlloc(out, std::max<size_t>(bytes, 16), cudaHostAllocPortable));
  });
}

extern "C" int rs_alloc_pinned_flags(size_t bytes, uint32_t flags, void** out) {
  return guarded([&] {
    if (!out) raise(RS_E_INVALID, "null argument");
    unsigned f = cudaHostAllocPortable;
    if (flags & RS_PINNED_WRITE_COMBINED) f |= cudaHostAllocWriteCombined;
    RS_CUDA(cudaHostAlloc(out, std::max<size_t>(bytes, 16), f));
  });
}

extern "C" int rs_free_pinned(void* p) {
  return guarded([&] {
    if (p) RS_CUDA(cudaFreeHost(p));
  });
}

extern "C" int rs_accel_create(const rs_model_desc* model, const rs_init_desc* init, int device,
                               rs_accel** out) {
  rs_accel* a = nullptr;
  int rc = guarded([&] {
    if (!model || !init || !out) raise(RS_E_INVALID, "null argument");
    *out = nullptr;
    validate_model(*model);
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      raise(RS_E_NO_DEVICE, "no CUDA device visible");
    if (device < 0 || device >= n) raise(RS_E_NO_DEVICE, "device ordinal out of range");
    cudaDeviceProp prop;
    RS_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      raise(RS_E_NO_DEVICE, "this library is built for sm_100a (B200) only");
    if (init->max_query_size < 1) raise(RS_E_INVALID, "max_query_size < 1");
    if (init->fc_mode < RS_FC_FP32 || init->fc_mode > RS_FC_BF16)
      raise(RS_E_INVALID, "bad fc_mode");
    RS_CUDA(cudaSetDevice(device));
    (void)cudaGetLastError();  // drop a stale non-sticky error from an earlier call
    a = new rs_accel();
    a->m = *model;
    a->init = *init;
    a->depth = init->queue_depth > 0 ? std::min<int>(init->queue_depth, rs_accel::kMaxLanes) : 4;
    {
      // carveout policy (tools/env_sweep.py, profiles/r2_carveout/): models
      // whose embedding stage bounds the queue (Sum / AttentionFC pooling with
      // more gather than FC time, and the AttentionRNN recurrence) get the
      // uniform carveout and the shallow FC tiles — cfg3 RMC2 -6%, zoo RMC2
      // -9%, DIN -4%, DIEN -5%; FC-bound models keep the deep tiles (MT-WND
      // +45%, WND +3.5% with the carveout). RS_CARVEOUT=<pct> overrides, 0 = off
      // "gather-bound": the embedding stage's HBM time at ~6.5 TB/s exceeds the
      // FC stacks' time at ~300 TF/s (the pipelined tcgen05 rate), per item
      // from work() — zoo RMC3 (2560-wide bottom MLP, 27 KB gathered per item)
      // is FC-bound and keeps the deep tiles (73.9K vs 86.9K QPS with them)
      const rs_work_breakdown wb = work(*model, 1);
      const double gather_s =
          (wb.bytes[RS_OP_EMBEDDING_LOOKUP] + wb.bytes[RS_OP_POOLING]) / 6.5e12;
      const double fc_s = (wb.flops[RS_OP_DENSE_FC] + wb.flops[RS_OP_PREDICT_FC]) / 3.0e14;
      const bool gather_bound =
          model->num_tables > 0 &&
          (model->pooling == RS_POOL_ATTENTION_RNN ||
           (model->pooling != RS_POOL_CONCAT && gather_s >= fc_s));
      const char* cv = getenv("RS_CARVEOUT");
      a->carveout_pct = cv ? std::max(0, std::min(100, atoi(cv))) : (gather_bound ? 50 : 0);
      a->fc_smem_kb = a->carveout_pct > 0 ? 110 : 0;
      // the interaction on 2-warp CTAs that fit beside the gathers when the
      // gather time is >= 4x the FC time (cfg3 / zoo RMC2; not cfg3 RMC3)
      a->inter_threads = gather_bound && gather_s >= 4.0 * fc_s ? 64 : 256;
      // CTA-pair FC tiles inside the capped shared memory when the FC stacks
      // are a substantial part of the work (cfg3 RMC3: FC ~60% of the gather
      // time, -8.5% us/query; RMC1/RMC2 shapes neutral)
      a->pair_capped = gather_bound && fc_s >= 0.25 * gather_s ? 1 : 0;
      // CTA pairs in every tcgen05 graph when EVERY FC layer is >= 256 wide
      // (a narrow final layer fused into the previous epilogue aside), one
      // stack, not gather-bound: no query then mixes pair and one-CTA kernels
      // (WND 7.84 -> 7.42 us/query at 4 stages; MT-WND's batched stacks and
      // RMC3's mixed-width bottom MLP lose with pairs: DESIGN.md §2b)
      bool all_wide = !gather_bound && model->num_parallel_predict_stacks <= 1 &&
                      model->predict_fc.n > 0;
      for (int l = 0; all_wide && l < model->predict_fc.n; ++l) {
        const int64_t w = model->predict_fc.dims[l];
        const bool fused_last = l == model->predict_fc.n - 1 && w <= kFuseMaxN2;
        if (w < 256 && !fused_last) all_wide = false;
      }
      if (model->has_dense_fc)
        for (int l = 0; all_wide && l < model->dense_fc.n; ++l)
          if (model->dense_fc.dims[l] < 256) all_wide = false;
      // Off by default: the bench's queue (device-resident WND, 16 lanes)
      // measured 90.1K-110.8K QPS@SLA with it vs 120.9K without, although the
      // env_sweep queue favoured it (7.64 vs 7.87 us/query): the pair grids'
      // cluster scheduling makes the lane graphs' timing erratic.
      // RS_TC2_ALL=1 turns it on for the shapes that qualify.
      const char* pae = getenv("RS_TC2_ALL");
      a->pairs_all = pae && atoi(pae) != 0 && all_wide;
    }
    a->device = device;
    a->sm_count = prop.multiProcessorCount;
    a->l2_bytes = prop.l2CacheSize;
    RS_CUDA(cudaStreamCreateWithFlags(&a->own, cudaStreamNonBlocking));
    RS_CUDA(cudaEventCreateWithFlags(&a->copy_gate, cudaEventDisableTiming));
    build_model(a);
#if RS_EXPERIMENTS
    a->memops = probe_memops(a);
    if (const char* ds = getenv("RS_DENSE_SMS")) make_partition(a, atoi(ds));
#endif
    *out = a;
  });
  if (rc != RS_OK && a) {
    for (void* p : a->allocs) cudaFree(p);
    if (a->own) cudaStreamDestroy(a->own);
    delete a;
  }
  return rc;
}

extern "C" int rs_accel_destroy(rs_accel* a) {
  return guarded([&] {
    if (!a) return;
    cudaSetDevice(a->device);
    cudaDeviceSynchronize();
    for (auto& kv : a->slots) free_slot(kv.second.get());
    a->slots.clear();
    for (auto& p : a->pipe)
      if (p) free_slot(p.get());
    for (auto e : a->evpool) cudaEventDestroy(e);
    for (auto e : a->evstart) cudaEventDestroy(e);
    if (a->copy_gate) cudaEventDestroy(a->copy_gate);
    if (a->copy) cudaStreamDestroy(a->copy);
    for (auto c : a->copy_more)
      if (c) cudaStreamDestroy(c);
    for (int k = 0; k < 2; ++k) {
      if (a->d2h[k]) cudaStreamDestroy(a->d2h[k]);
      if (a->d2h_join[k]) cudaEventDestroy(a->d2h_join[k]);
    }
    for (int d = 0; d < rs_accel::kMaxLanes; ++d) {
      if (a->lane[d]) cudaStreamDestroy(a->lane[d]);
      if (a->lane_join[d]) cudaEventDestroy(a->lane_join[d]);
    }
    if (a->hot) release_hot(a);
    for (void* p : a->allocs) cudaFree(p);
    if (a->own) cudaStreamDestroy(a->own);
#if RS_EXPERIMENTS
    if (a->g_dense) green_api().destroy(a->g_dense);
    if (a->g_emb) green_api().destroy(a->g_emb);
#endif
    delete a;
  });
}

extern "C" int rs_accel_info_get(const rs_accel* ca, rs_accel_info* out) {
  return guarded([&] {
    if (!ca || !out) raise(RS_E_INVALID, "null argument");
    rs_accel* a = const_cast<rs_accel*>(ca);
    Slot* s = get_slot(a, a->own);
    rs_accel_info i{};
    i.device = a->device;
    i.sm_count = a->sm_count;
    i.kernels_per_forward = s->kernels[kGraphLarge] ? s->kernels[kGraphLarge] : s->kernels[kGraphSmall];
    i.kernels_per_forward_small = s->kernels[kGraphSmall];
    i.fc_layers_tcgen05 = s->tc_layers;
    i.predict_input_dim = a->p_in;
    i.output_dim = a->out_w;
    i.pooled_dim = a->pooled_dim;
    i.table_bytes = a->table_bytes;
    i.weight_bytes = a->weight_bytes;
    i.l2_bytes = a->l2_bytes;
    i.hot_rows = a->hot_rows;
    *out = i;
  });
}

extern "C" int rs_forward(rs_accel* a, const rs_query* q, float* out, void* stream,
                          rs_timing* timing) {
  return run(a, q, out, stream, timing, true);
}

extern "C" int rs_forward_many(rs_accel* a, int64_t n, const rs_query* queries,
                               float* const* outs, void* stream, double* service_ms,
                               double* latency_ms) {
  return run_many(a, n, queries, outs, stream, service_ms, latency_ms);
}

extern "C" int rs_forward_many_ev(rs_accel* a, int64_t n, const rs_query* queries,
                                  float* const* outs, void* stream, double* service_ms,
                                  double* latency_ms, void* done_event) {
  return run_many(a, n, queries, outs, stream, service_ms, latency_ms, done_event);
}

// Real-time executors. The reference's single FIFO accelerator
// server (accel_busy + accel_fifo, proj/src/sim.cpp:95-97, 126-136) becomes a
// K-replica pool: the releasing thread routes each offloaded query to the
// replica with the least outstanding items (ties to the lowest index, SURVEY
// §8e); one dispatcher thread per replica stages, launches and retires that
// replica's queries on its lanes exactly as rs_forward_many does, so host
// dispatch cost scales with the replica count. Outstanding item counts are
// atomics: the releaser adds on assignment, the replica's dispatcher subtracts
// when the query's completion event has fired. GPU completion times are CUDA
// events relative to a start event recorded (and waited for) just before the
// host clock's t0.
namespace rs {
namespace {

struct ServeRep {
  rs_accel* a = nullptr;
  Slot* p[rs_accel::kMaxLanes] = {};
  std::atomic<int64_t> outstanding{0};
  // assignment ring (releaser -> dispatcher), single producer/consumer
  std::vector<int64_t> queue;
  std::atomic<int64_t> head{0};
  int64_t tail = 0;
  std::deque<std::pair<int64_t, int64_t>> inflight;  // (query, replica-local seq)
  int64_t issued = 0;
  int64_t dispatched = 0;
};

constexpr int64_t kServeRing = 4096;

struct ServeShared {
  const rs_query* qs = nullptr;
  float* const* outs = nullptr;
  int loc = RS_MEM_HOST;
  std::vector<double> done_ms;          // per query, device clock since t0
  std::atomic<bool> released_all{false};
  std::atomic<int> failed{0};
  std::mutex err_mu;
  Error first_err{RS_OK, ""};
  void record(const Error& e) {
    std::lock_guard<std::mutex> g(err_mu);
    if (!failed.exchange(1)) first_err = e;
  }
};

// Replica pool of one serving call: lanes, event rings, t0 events.
struct ServePool {
  std::vector<std::unique_ptr<ServeRep>> R;
  std::vector<std::thread> th;

  void setup(rs_accel* const* reps, int32_t k, int64_t n) {
    for (int r = 0; r < k; ++r) {
      auto rp = std::make_unique<ServeRep>();
      rs_accel* a = reps[r];
      RS_CUDA(cudaSetDevice(a->device));
      rp->a = a;
      for (int d = 0; d < a->depth; ++d) rp->p[d] = get_pipe_slot(a, d);
      while ((int64_t)a->evpool.size() < kServeRing + 1) {
        cudaEvent_t e;
        RS_CUDA(cudaEventCreate(&e));
        a->evpool.push_back(e);
      }
      rp->queue.assign((size_t)n, -1);
      R.push_back(std::move(rp));
    }
  }
  // t0 on every replica (a start event each; the lanes and copy stream wait
  // for it), returned only once the events have fired
  void start_clock() {
    for (auto& rp : R) {
      rs_accel* a = rp->a;
      RS_CUDA(cudaSetDevice(a->device));
      RS_CUDA(cudaEventRecord(a->evpool[0], a->own));
      RS_CUDA(cudaEventRecord(a->copy_gate, a->own));
      for (int d = 0; d < a->depth; ++d) RS_CUDA(cudaStreamWaitEvent(a->lane[d], a->copy_gate, 0));
      RS_CUDA(cudaStreamWaitEvent(a->copy, a->copy_gate, 0));
      RS_CUDA(cudaStreamSynchronize(a->own));
    }
  }
  void launch(ServeShared& sh) {
    th.reserve(R.size());
    for (auto& rp : R) th.emplace_back([&sh, p = rp.get()] { dispatch_loop(p, sh); });
  }
  // least outstanding items, ties to the lowest index
  void route(int64_t i, const ServeShared& sh) {
    int best = 0;
    int64_t best_out = R[0]->outstanding.load(std::memory_order_relaxed);
    for (int r = 1; r < (int)R.size(); ++r) {
      const int64_t o = R[r]->outstanding.load(std::memory_order_relaxed);
      if (o < best_out) { best = r; best_out = o; }
    }
    ServeRep* rp = R[best].get();
    rp->outstanding.fetch_add(sh.qs[i].size, std::memory_order_relaxed);
    rp->queue[(size_t)rp->tail++] = i;
    rp->head.store(rp->tail, std::memory_order_release);
  }
  void join() {
    for (auto& t : th) t.join();
    th.clear();
  }

  static void dispatch_loop(ServeRep* rp, ServeShared& sh) {
    try {
      rs_accel* a = rp->a;
      RS_CUDA(cudaSetDevice(a->device));
      auto retire = [&](bool block) {
        while (!rp->inflight.empty()) {
          const auto [qi, seq] = rp->inflight.front();
          cudaEvent_t e = a->evpool[1 + seq % kServeRing];
          if (block) {
            RS_CUDA(cudaEventSynchronize(e));
          } else {
            const cudaError_t st = cudaEventQuery(e);
            if (st == cudaErrorNotReady) break;
            if (st != cudaSuccess) RS_CUDA(st);
          }
          sh.done_ms[(size_t)qi] = elapsed(a->evpool[0], e);
          rp->outstanding.fetch_sub(sh.qs[qi].size, std::memory_order_relaxed);
          rp->inflight.pop_front();
        }
      };
      for (;;) {
        if (sh.failed.load(std::memory_order_relaxed)) return;
        const int64_t h = rp->head.load(std::memory_order_acquire);
        if (rp->dispatched == h) {
          retire(false);
          if (sh.released_all.load(std::memory_order_acquire) &&
              rp->dispatched == rp->head.load(std::memory_order_acquire))
            break;
          std::this_thread::yield();
          continue;
        }
        const int64_t i = rp->queue[(size_t)rp->dispatched++];
        const int64_t seq = rp->issued++;
        if (seq >= kServeRing)  // event-ring reuse: that query must have retired
          while (!rp->inflight.empty() && rp->inflight.front().second <= seq - kServeRing)
            retire(true);
        const int d = (int)(seq % a->depth);
        Slot* sl = rp->p[d];
        cudaStream_t ls = a->lane[d];
        if (sh.loc == RS_MEM_HOST) {
          RS_CUDA(cudaStreamWaitEvent(a->copy, sl->free, 0));
          stage_inputs(a, sl, &sh.qs[i], true, a->copy, nullptr, /*widen_later=*/true);
          RS_CUDA(cudaEventRecord(sl->ready, a->copy));
          RS_CUDA(cudaStreamWaitEvent(ls, sl->ready, 0));
          widen_indices(a, sl, &sh.qs[i], ls);
        } else {
          stage_inputs(a, sl, &sh.qs[i], true, ls, sh.outs[i]);
        }
        launch_stage(a, sl, &sh.qs[i], sh.outs[i], true, ls);
        RS_CUDA(cudaEventRecord(sl->free, ls));
        RS_CUDA(cudaEventRecord(a->evpool[1 + seq % kServeRing], ls));
        rp->inflight.emplace_back(i, seq);
        retire(false);
      }
      retire(true);
      for (int d = 0; d < a->depth; ++d) collect_errors(rp->p[d], a->lane[d]);
    } catch (const Error& e) {
      sh.record(e);
    } catch (const std::exception& e) {
      sh.record(Error{RS_E_INVALID, e.what()});
    }
  }
};

// host-clock wait until t0 + seconds
void wait_until(std::chrono::steady_clock::time_point t0, double seconds) {
  const auto due = t0 + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                            std::chrono::duration<double>(seconds));
  for (;;) {
    const auto now = std::chrono::steady_clock::now();
    if (now >= due) break;
    if (due - now > std::chrono::microseconds(200))
      std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

void check_serve_args(rs_accel* const* reps, int32_t k, int64_t n, const rs_query* qs,
                      const double* arrival_s, float* const* outs, double* latency_ms,
                      std::vector<std::unique_lock<std::mutex>>& locks) {
  if (!qs || !arrival_s || !outs || !latency_ms) raise(RS_E_INVALID, "null argument");
  if (k < 0 || n < 1 || (k > 0 && !reps)) raise(RS_E_INVALID, "k < 0 or n < 1");
  const int loc = qs[0].location;
  for (int r = 0; r < k; ++r)
    if (!reps[r]) raise(RS_E_INVALID, "null replica");
  for (int64_t i = 0; i < n; ++i) {
    for (int r = 0; r < k; ++r) check_query(reps[r], &qs[i]);
    if (qs[i].location != loc) raise(RS_E_INVALID, "mixed memory locations");
    if (!outs[i]) raise(RS_E_INVALID, "null output");
    if (!(arrival_s[i] >= 0) || (i && arrival_s[i] < arrival_s[i - 1]))
      raise(RS_E_INVALID, "arrival times must be non-negative and non-decreasing");
  }
  // queue locks in address order (two concurrent callers can never deadlock)
  std::vector<rs_accel*> order(reps, reps + k);
  std::sort(order.begin(), order.end());
  order.erase(std::unique(order.begin(), order.end()), order.end());
  if ((int)order.size() != k) raise(RS_E_INVALID, "a replica appears twice");
  for (rs_accel* a : order) locks.emplace_back(a->many_mu);
}

}  // namespace
}  // namespace rs

extern "C" int rs_serve(rs_accel* const* reps, int32_t k, int64_t n, const rs_query* qs,
                        const double* arrival_s, float* const* outs, double* latency_ms) {
  std::vector<std::unique_lock<std::mutex>> locks;
  return guarded([&] {
    if (k < 1) raise(RS_E_INVALID, "k < 1");
    check_serve_args(reps, k, n, qs, arrival_s, outs, latency_ms, locks);
    ServeShared sh;
    sh.qs = qs;
    sh.outs = outs;
    sh.loc = qs[0].location;
    sh.done_ms.assign((size_t)n, -1.0);
    ServePool pool;
    pool.setup(reps, k, n);
    pool.start_clock();
    pool.launch(sh);
    const auto t0 = std::chrono::steady_clock::now();
    for (int64_t i = 0; i < n && !sh.failed.load(std::memory_order_relaxed); ++i) {
      wait_until(t0, arrival_s[i]);
      pool.route(i, sh);
    }
    sh.released_all.store(true, std::memory_order_release);
    pool.join();
    if (sh.failed.load()) raise(sh.first_err.code, sh.first_err.msg);
    for (int64_t i = 0; i < n; ++i) latency_ms[i] = sh.done_ms[(size_t)i] - arrival_s[i] * 1e3;
  });
}

// DeepRecSched in real time: the routing decision of
// simulate() (proj/src/sim.cpp:173-191) executed — offloaded queries to the
// replica pool above, the rest split into requests of `batch` items on a FIFO
// served by `cores` host worker threads (the C-core pool, sim.cpp:114-124),
// each request run whole by rs_host_forward on its thread. A query completes
// when its last request (or its offloaded run) does.
extern "C" int rs_serve_hybrid(rs_host_model* cpu, int32_t cores, int64_t batch,
                               int64_t threshold, rs_accel* const* reps, int32_t k, int64_t n,
                               const rs_query* qs, const double* arrival_s, float* const* outs,
                               double* latency_ms, int32_t* offloaded) {
  std::vector<std::unique_lock<std::mutex>> locks;
  return guarded([&] {
    if (!cpu) raise(RS_E_INVALID, "null host model");
    if (cores < 1 || batch < 1) raise(RS_E_INVALID, "cores < 1 or batch < 1");
    check_serve_args(reps, k, n, qs, arrival_s, outs, latency_ms, locks);
    for (int64_t i = 0; i < n; ++i)
      if (qs[i].location != RS_MEM_HOST || qs[i].index_type != 0)
        raise(RS_E_INVALID, "hybrid serving takes host queries in the reference byte model");
    const bool use_gpu = k > 0 && threshold > 0;
    ServeShared sh;
    sh.qs = qs;
    sh.outs = outs;
    sh.loc = RS_MEM_HOST;
    sh.done_ms.assign((size_t)n, -1.0);
    ServePool pool;
    if (use_gpu) {
      pool.setup(reps, k, n);
      pool.start_clock();
      pool.launch(sh);
    }
    // CPU side: request FIFO + worker pool
    struct Req { int64_t q, off, cnt; };
    std::deque<Req> fifo;
    std::mutex fmu;
    std::condition_variable fcv;
    bool closed = false;
    std::vector<std::atomic<int64_t>> remaining((size_t)n);
    std::vector<double> cpu_done((size_t)n, -1.0);
    std::chrono::steady_clock::time_point t0;
    auto worker = [&] {
      try {
        for (;;) {
          Req r;
          {
            std::unique_lock<std::mutex> g(fmu);
            fcv.wait(g, [&] { return closed || !fifo.empty(); });
            if (fifo.empty()) return;
            r = fifo.front();
            fifo.pop_front();
          }
          if (sh.failed.load(std::memory_order_relaxed)) continue;
          const rs_query& q = qs[r.q];
          const int64_t bad = host_forward_rows(cpu, q.dense, q.indices, outs[r.q], r.off,
                                                r.off + r.cnt);
          if (bad >= 0) raise(RS_E_INDEX, "embedding index outside [0, rows_per_table)");
          if (remaining[(size_t)r.q].fetch_sub(1) == 1)
            cpu_done[(size_t)r.q] =
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count();
        }
      } catch (const Error& e) {
        sh.record(e);
      } catch (const std::exception& e) {
        sh.record(Error{RS_E_INVALID, e.what()});
      }
    };
    t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> workers;
    for (int c = 0; c < cores; ++c) workers.emplace_back(worker);
    for (int64_t i = 0; i < n && !sh.failed.load(std::memory_order_relaxed); ++i) {
      wait_until(t0, arrival_s[i]);
      const int64_t S = qs[i].size;
      const bool off = use_gpu && S > threshold;  // strictly greater (sim.cpp:178)
      if (offloaded) offloaded[i] = off ? 1 : 0;
      if (off) {
        pool.route(i, sh);
        continue;
      }
      const int64_t full = S / batch, rem = S % batch;
      remaining[(size_t)i].store(full + (rem > 0 ? 1 : 0));
      {
        std::lock_guard<std::mutex> g(fmu);
        for (int64_t j = 0; j < full; ++j) fifo.push_back({i, j * batch, batch});
        if (rem > 0) fifo.push_back({i, full * batch, rem});
      }
      fcv.notify_all();
    }
    {
      std::lock_guard<std::mutex> g(fmu);
      closed = true;
    }
    fcv.notify_all();
    sh.released_all.store(true, std::memory_order_release);
    for (auto& w : workers) w.join();
    if (use_gpu) pool.join();
    if (sh.failed.load()) raise(sh.first_err.code, sh.first_err.msg);
    for (int64_t i = 0; i < n; ++i) {
      const bool off = use_gpu && qs[i].size > threshold;
      latency_ms[i] = (off ? sh.done_ms[(size_t)i] : cpu_done[(size_t)i]) - arrival_s[i] * 1e3;
    }
  });
}

extern "C" int rs_sync(rs_accel* a, void* stream) {
  return guarded([&] {
    if (!a) raise(RS_E_INVALID, "null handle");
    RS_CUDA(cudaSetDevice(a->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : a->own;
    RS_CUDA(cudaStreamSynchronize(st));
    Slot* s = get_slot(a, st);
    collect_errors(s, st);
    for (auto& p : a->pipe)
      if (p) collect_errors(p.get(), st);
  });
}

extern "C" int rs_pooled(rs_accel* a, const rs_query* q, float* out, void* stream,
                         rs_timing* timing) {
  return run(a, q, out, stream, timing, false);
}

extern "C" int rs_service_time(rs_accel* a, int64_t query_size, double* seconds) {
  return guarded([&] {
    if (!a || !seconds) raise(RS_E_INVALID, "null argument");
    if (query_size < 1) raise(RS_E_INVALID, "query_size < 1");
    {
      std::lock_guard<std::mutex> lock(a->mu);
      auto it = a->service_memo.find(query_size);
      if (it != a->service_memo.end()) {
        *seconds = it->second;
        return;
      }
    }
    const int64_t S = query_size;
    // one pinned buffer [dense | indices] (a packed query: one transfer when the
    // dense block is a multiple of 8 bytes, as for every zoo shape)
    const size_t dense_b = (size_t)(S * a->dense_in * 4 + 15) / 16 * 16;
    const size_t idx_b = (size_t)(S * a->T * a->L * 8);
    void *in = nullptr, *out = nullptr;
    RS_CUDA(cudaHostAlloc(&in, std::max<size_t>(dense_b + idx_b, 16), 0));
    RS_CUDA(cudaHostAlloc(&out, (size_t)(S * a->out_w * 4), 0));
    void* dense = in;
    void* idx = static_cast<uint8_t*>(in) + dense_b;
    std::vector<double> t;
    int rc = rs_fill_query(&a->m, a->init.rows_per_table, a->init.seed ^ 0x5E41CEull, 0, S,
                           static_cast<float*>(dense), static_cast<int64_t*>(idx));
    for (int i = 0; rc == RS_OK && i < 6; ++i) {
      rs_query q{S, static_cast<float*>(dense), static_cast<int64_t*>(idx), RS_MEM_HOST, 0};
      rs_timing tm{};
      rc = rs_forward(a, &q, static_cast<float*>(out), nullptr, &tm);
      if (i > 0) t.push_back(tm.total_ms * 1e-3);
    }
    cudaFreeHost(in); cudaFreeHost(out);
    if (rc != RS_OK) raise(rc, rs_last_error());
    std::sort(t.begin(), t.end());
    const double med = t[t.size() / 2];
    std::lock_guard<std::mutex> lock(a->mu);
    a->service_memo[query_size] = med;
    *seconds = med;
  });
}

// Measured ServiceTime breakdown (recsim::ServiceTime, platform.hpp:60-68):
// total and transfer (H2D + D2H) from the timed whole-query call, and the
// compute part split over the operator categories the way the reference
// apportions its roofline (platform.cpp:121-134) — but from MEASURED stage
// times: the embedding stage (EmbeddingLookup / Pooling / Attention /
// Recurrent), the predict stack (PredictFC), and the rest of the compute
// (DenseFC / Interaction, what is not hidden under the gather); inside a
// stage by the categories' B200 roofline weights from work().
extern "C" int rs_service_breakdown(rs_accel* a, int64_t query_size, double* total,
                                    double* transfer, double* per_category) {
  return guarded([&] {
    if (!a || !total || !transfer || !per_category) raise(RS_E_INVALID, "null argument");
    if (query_size < 1) raise(RS_E_INVALID, "query_size < 1");
    const int64_t S = query_size;
    const size_t dense_b = (size_t)(S * a->dense_in * 4 + 15) / 16 * 16;
    const size_t idx_b = (size_t)(S * a->T * a->L * 8);
    void *in = nullptr, *out = nullptr;
    RS_CUDA(cudaHostAlloc(&in, std::max<size_t>(dense_b + idx_b, 16), 0));
    RS_CUDA(cudaHostAlloc(&out, (size_t)(S * a->out_w * 4), 0));
    void* dense = in;
    void* idx = static_cast<uint8_t*>(in) + dense_b;
    std::vector<double> tt, tx, te, tf;
    int rc = rs_fill_query(&a->m, a->init.rows_per_table, a->init.seed ^ 0x5E41CEull, 0, S,
                           static_cast<float*>(dense), static_cast<int64_t*>(idx));
    const int saved = a->stage_timing;
    for (int pass = 0; rc == RS_OK && pass < 2; ++pass) {
      // pass 0: the lean graph (total, transfer); pass 1: the stage-timed copy
      a->stage_timing = pass;
      for (int i = 0; rc == RS_OK && i < 6; ++i) {
        rs_query q{S, static_cast<float*>(dense), static_cast<int64_t*>(idx), RS_MEM_HOST, 0};
        rs_timing tm{};
        rc = rs_forward(a, &q, static_cast<float*>(out), nullptr, &tm);
        if (i == 0) continue;
        if (pass == 0) {
          tt.push_back(tm.total_ms * 1e-3);
          tx.push_back((tm.h2d_ms + tm.d2h_ms) * 1e-3);
        } else {
          te.push_back(tm.embed_ms * 1e-3);
          tf.push_back(tm.fc_ms * 1e-3);
        }
      }
    }
    a->stage_timing = saved;
    cudaFreeHost(in);
    cudaFreeHost(out);
    if (rc != RS_OK) raise(rc, rs_last_error());
    auto med = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v[v.size() / 2];
    };
    const double T = med(tt), X = std::min(med(tx), T), E = med(te), F = med(tf);
    const double compute = T - X;
    const rs_work_breakdown wb = work(a->m, S);
    // B200 roofline weight of a category: max(flops / tf32 rate, bytes / HBM)
    auto weight = [&](int c) { return std::max(wb.flops[c] / 854e12, wb.bytes[c] / 6.5e12); };
    double stage[3] = {E, F, std::max(0.0, compute - E - F)};
    const int cats[3][4] = {{RS_OP_EMBEDDING_LOOKUP, RS_OP_POOLING, RS_OP_ATTENTION, RS_OP_RECURRENT},
                            {RS_OP_PREDICT_FC, -1, -1, -1},
                            {RS_OP_DENSE_FC, RS_OP_INTERACTION, -1, -1}};
    double pc[RS_NUM_OP_CATEGORIES] = {};
    double sum = 0;
    for (int g = 0; g < 3; ++g) {
      double wsum = 0;
      for (int c : cats[g]) if (c >= 0) wsum += weight(c);
      for (int c : cats[g])
        if (c >= 0 && wsum > 0) pc[c] = stage[g] * weight(c) / wsum;
    }
    for (double v : pc) sum += v;
    for (int c = 0; c < RS_NUM_OP_CATEGORIES; ++c)
      per_category[c] = sum > 0 ? pc[c] * compute / sum : 0.0;  // sums to the compute time
    *total = T;
    *transfer = X;
  });
}

extern "C" int rs_build_flags(void) { return RS_EXPERIMENTS ? RS_BUILD_EXPERIMENTS : 0; }
