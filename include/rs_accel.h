/*
 * rs_accel.h — C-ABI of the B200-native accelerator path for DeepRecSched
 * (DeepRecSys, arXiv 2001.02772).
 *
 * The reference (`/root/reference/proj`, library `recsim`) models the
 * accelerator as a pure cost function; this header is the drop-in boundary
 * that replaces that model with real execution on a B200. Every entry point
 * names the reference interface it replaces or mirrors (file:line under
 * /root/reference/). Plain C types only: no torch, no C++ across the ABI,
 * no exceptions.
 *
 * Error convention: every function returns RS_OK (0) or a negative RS_E_*
 * code; rs_last_error() returns a thread-local message for the last failure
 * on the calling thread.
 */
#ifndef RS_ACCEL_H
#define RS_ACCEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 3

/* ---- error codes -------------------------------------------------------- */
enum {
  RS_OK = 0,
  RS_E_INVALID = -1,        /* std::invalid_argument in the reference        */
  RS_E_UNKNOWN_MODEL = -2,  /* recsim::UnknownModel (model_zoo.hpp:15-18)    */
  RS_E_CONFIG = -3,         /* recsim::ConfigError (sim.hpp:15-17)           */
  RS_E_DISTRIBUTION = -4,   /* recsim::InvalidDistribution (loadgen.hpp:12)  */
  RS_E_CUDA = -5,           /* CUDA runtime / driver failure                 */
  RS_E_OOM = -6,            /* device or pinned allocation failed            */
  RS_E_INDEX = -7,          /* embedding index outside [0, rows_per_table)   */
  RS_E_NO_DEVICE = -8,      /* no sm_100 device / extension cannot run       */
  RS_E_CAPACITY = -9,       /* query larger than the handle's max_query_size */
  RS_E_EMPTY = -10          /* recsim::EmptyResult (sim.hpp:19-21)           */
};

/* ---- operator API: mirror of recsim::ModelSpec -------------------------- */
/* Pooling — recsim::Pooling (proj/include/recsim/model_zoo.hpp:20).        */
enum {
  RS_POOL_SUM = 0,
  RS_POOL_CONCAT = 1,
  RS_POOL_ATTENTION_FC = 2,
  RS_POOL_ATTENTION_RNN = 3
};

/* OpCategory — recsim::OpCategory (model_zoo.hpp:22-31), same ordinals.    */
enum {
  RS_OP_DENSE_FC = 0,
  RS_OP_PREDICT_FC = 1,
  RS_OP_EMBEDDING_LOOKUP = 2,
  RS_OP_POOLING = 3,
  RS_OP_ATTENTION = 4,
  RS_OP_RECURRENT = 5,
  RS_OP_INTERACTION = 6,
  RS_NUM_OP_CATEGORIES = 7
};

#define RS_MAX_LAYERS 8
#define RS_NAME_LEN 32

/* recsim::LayerStack (model_zoo.hpp:39-44): ordered output widths.         */
typedef struct rs_layer_stack {
  int32_t n;                      /* number of layers (0 = absent stack)     */
  int64_t dims[RS_MAX_LAYERS];
} rs_layer_stack;

/* recsim::ModelSpec (model_zoo.hpp:54-65) + EmbeddingConfig (:46-52).
 * `has_dense_fc` encodes std::optional<LayerStack> dense_fc;
 * `recurrent_hidden_dim` = 0 encodes an empty std::optional.              */
typedef struct rs_model_desc {
  char name[RS_NAME_LEN];
  int32_t has_dense_fc;
  rs_layer_stack dense_fc;
  rs_layer_stack predict_fc;
  int64_t num_parallel_predict_stacks;
  int64_t num_tables;
  int64_t lookups_per_table;
  int64_t embedding_dim;
  int32_t pooling;                /* RS_POOL_*                               */
  int64_t dense_input_dim;
  int64_t recurrent_hidden_dim;   /* 0 = absent                              */
} rs_model_desc;

/* recsim::OpWork / WorkBreakdown (model_zoo.hpp:67-84).                    */
typedef struct rs_work_breakdown {
  double flops[RS_NUM_OP_CATEGORIES];
  double bytes[RS_NUM_OP_CATEGORIES];
  double gather_stream;
} rs_work_breakdown;

/* Host-only mirrors of the reference's model/operator API (no GPU needed). */

/* builtin_model() — proj/src/model_zoo.cpp:141-170. RS_E_UNKNOWN_MODEL.    */
int rs_model_builtin(const char* name, rs_model_desc* out);
/* zoo_names() — model_zoo.cpp:172-175. Writes up to `cap` names.           */
int rs_zoo_names(const char** names, int cap, int* count);
/* ModelSpec::validate() — model_zoo.cpp:41-59. RS_E_INVALID.               */
int rs_model_validate(const rs_model_desc* m);
/* work(m, batch) — model_zoo.cpp:177-245. RS_E_INVALID for batch < 1.      */
int rs_work(const rs_model_desc* m, int64_t batch, rs_work_breakdown* out);
/* predict_input_dim(m) — model_zoo.cpp:113-137 (anonymous in reference).   */
int rs_predict_input_dim(const rs_model_desc* m, int64_t* out);
/* accel_input_bytes(m, S) — proj/src/platform.cpp:105-111.                 */
int rs_accel_input_bytes(const rs_model_desc* m, int64_t query_size, double* out);
/* sla_target(name, level) — proj/src/autotune.cpp:73-88 (seconds).        */
int rs_sla_target(const char* model_name, const char* level, double* out);

/* ---- scheduler interface (host-only) ------------------------------------ */
/* Routing of one arriving query — the decision in simulate()
 * (proj/src/sim.cpp:178-188): offload iff threshold > 0 && S > threshold
 * (strictly greater); otherwise floor(S/B) requests of B items then one of
 * S mod B. `threshold` <= 0 encodes an absent std::optional. On return
 * *offload is 0/1; when 0, requests[0..*n_requests) hold the request sizes
 * in FIFO push order. RS_E_CAPACITY if more than `cap` requests.           */
int rs_route(int64_t query_size, int64_t batch_size, int64_t threshold,
             int32_t* offload, int64_t* requests, int64_t cap,
             int64_t* n_requests);

/* Query streams — gen_trace() (proj/src/loadgen.cpp:106-125) with the
 * SizeDistribution kinds of loadgen.hpp:23-45; bit-identical to the
 * reference for identical (seed, parameters) (mt19937_64, rng.hpp:14-48).  */
enum {
  RS_DIST_FIXED = 0,
  RS_DIST_NORMAL = 1,
  RS_DIST_LOGNORMAL = 2,
  RS_DIST_PRODUCTION_HEAVY_TAIL = 3
};
typedef struct rs_size_dist {
  int32_t kind;      /* RS_DIST_*                                           */
  double p0, p1, p2, p3;
  int64_t max_size;
} rs_size_dist;
/* SizeDistribution::production_heavy_tail() (loadgen.cpp:15-23).           */
int rs_dist_production(rs_size_dist* out);
int rs_gen_trace(uint64_t seed, double lambda, const rs_size_dist* dist,
                 int64_t n, double* arrival_times, int64_t* sizes);

/* QPS under a p95 SLA for a FIFO server pool fed by a trace whose per-query
 * service times are given (measured on the device). Mirrors the search of
 * max_qps_under_sla (proj/src/sim.cpp:246-290): evaluate lambda=1, then
 * `hi`, then geometric bisection to 1%; p95 is the exact order statistic
 * of summarize() (sim.cpp:217-235) over post-warmup queries.
 * `service_s[i]` is the service time of query i of the *base* trace; each
 * evaluation re-times the same size sequence with Poisson gaps at the new
 * rate (seed base_seed + eval index, as sim.cpp:253). `servers` FIFO
 * replicas; dispatch = least outstanding work, ties to lowest index.
 * `extra_s` (may be NULL): per-query time a query spends in a pipelined
 * accelerator beyond its service gap (residence - service, clamped at 0);
 * it is added to that query's latency so pipelining never hides latency.   */
typedef struct rs_qps_result {
  double qps;        /* achieved QPS of the accepted evaluation            */
  double at_lambda;  /* offered rate that met the SLA (0 if none)           */
  double p95;        /* seconds                                             */
  double p50;
  int32_t evaluations;
} rs_qps_result;
int rs_qps_under_sla(const double* service_s, const double* extra_s, int64_t n,
                     int32_t servers, double sla_s, double warmup_fraction,
                     uint64_t base_seed, double lambda_hi, rs_qps_result* out);

/* ---- the accelerator (B200) --------------------------------------------- */
typedef struct rs_accel rs_accel;

enum {
  RS_FC_FP32 = 0,  /* FFMA fp32 path (tight parity)                        */
  RS_FC_TF32 = 1,  /* tcgen05 kind::tf32 (fp32 operands, fp32 accumulate)   */
  RS_FC_AUTO = 2,  /* the measured-fastest path: today the tcgen05 graph at
                      every query size (= RS_FC_TF32)                   */
  RS_FC_BF16 = 3   /* tcgen05 kind::f16 with bf16 weights and activations,
                      fp32 accumulate (LABELLED lower-precision variant:
                      its own tolerance, tests/parity_rule.py)           */
};
enum { RS_RNN_GRU = 0, RS_RNN_AUGRU = 1 };

/* Deterministic initialisation and capacity. `rows_per_table` is kept
 * OUTSIDE the model descriptor because recsim::ModelSpec has no row count
 * (SURVEY.md §0.3 D1).                                                      */
typedef struct rs_init_desc {
  uint64_t seed;
  int64_t rows_per_table;
  int64_t max_query_size;   /* scratch capacity, items (reference max 1000) */
  int32_t fc_mode;          /* RS_FC_*                                       */
  int32_t rnn_cell;         /* RS_RNN_* (AttentionRNN only)                  */
  int32_t l2_persist_mb;    /* >0: hot-row block of up to this many MiB (rows
                               [0, R) of every table) kept in the L2
                               persisting set-aside; capped by the device's
                               persisting/window limits. Sum pooling only.  */
  int32_t queue_depth;      /* rs_forward_many lanes in flight (0 = 4, <= 16) */
} rs_init_desc;

/* One query: S items. dense f32[S * dense_input_dim] and indices
 * i64[S * num_tables * lookups_per_table] (item-major, then table, then
 * lookup) — the byte model of accel_input_bytes (platform.cpp:105-111).
 * location RS_MEM_HOST: pointers are host memory (pinned for async copy);
 * RS_MEM_DEVICE: pointers are device memory on the handle's GPU.
 * index_type holds LABELLED input-format flags; 0 = the
 * reference byte model. RS_INDEX_I32: `indices` points at int32 values (half
 * the index bytes), widened on the device — bit-identical to the int64
 * query. RS_DENSE_BF16: `dense` points at bfloat16 values (half the dense
 * bytes), widened on the device — identical to the fp32 query whose dense
 * features are those bf16 values.                                           */
enum { RS_MEM_HOST = 0, RS_MEM_DEVICE = 1 };
enum { RS_INDEX_I64 = 0, RS_INDEX_I32 = 1, RS_DENSE_BF16 = 2 };
typedef struct rs_query {
  int64_t size;
  const float* dense;
  const int64_t* indices;   /* int32_t* when index_type == RS_INDEX_I32 */
  int32_t location;
  int32_t index_type;       /* RS_INDEX_I32 | RS_DENSE_BF16 flags (0 = reference) */
} rs_query;

/* Per-call timing (CUDA events on the call's stream), milliseconds.        */
typedef struct rs_timing {
  double h2d_ms;
  double compute_ms;   /* the forward (or embedding-stage) graph             */
  double d2h_ms;
  double total_ms;
  double embed_ms;     /* rs_pooled: the embedding kernel alone, between
                          event-record nodes captured around it in the
                          graph; rs_forward: the embedding stage when
                          RS_OPT_STAGE_TIMING is on, else 0              */
  double fc_ms;        /* rs_forward with RS_OPT_STAGE_TIMING: the predict
                          stack (PredictFC kernels) alone; else 0         */
} rs_timing;

typedef struct rs_accel_info {
  int32_t device;
  int32_t sm_count;
  int32_t kernels_per_forward;     /* kernel nodes of the graph a query runs */
  int32_t kernels_per_forward_small; /* kernel nodes, FFMA graph (0 if none) */
  int32_t fc_layers_tcgen05;       /* FC layers routed to tcgen05          */
  int64_t predict_input_dim;
  int64_t output_dim;              /* per item: stacks * last predict dim  */
  int64_t pooled_dim;              /* per item: rs_pooled width            */
  int64_t table_bytes;
  int64_t weight_bytes;
  int64_t l2_bytes;
  int64_t hot_rows;                /* rows per table in the L2-persisting
                                      hot block (0 = off; l2_persist_mb)  */
} rs_accel_info;

/* Create one model replica on one GPU: allocate and initialise tables and
 * weights on the device (seeded). One handle = one model
 * on one device. Replaces the AcceleratorSpec value that the reference
 * passes around (platform.hpp:48-58).                                       */
int rs_accel_create(const rs_model_desc* model, const rs_init_desc* init,
                    int device, rs_accel** out);
int rs_accel_destroy(rs_accel* a);
int rs_accel_info_get(const rs_accel* a, rs_accel_info* out);

/* Whole-query forward: the real execution behind accel_service_time
 * (platform.cpp:113-136). Writes logits f32[S * stacks * out_dim] to `out`
 * (same location kind as the query). `stream` is a cudaStream_t (NULL =
 * the handle's own stream). When `timing` is non-NULL the call records
 * events, waits for completion and reports index errors; otherwise it is
 * asynchronous on `stream`, errors stay sticky until rs_sync, and the
 * caller owns synchronisation. Inputs and outputs must stay valid until the
 * stream reaches the end of this call.                                     */
int rs_forward(rs_accel* a, const rs_query* q, float* out, void* stream,
               rs_timing* timing);

/* Serve n whole queries on `stream` — the FIFO accelerator server of
 * simulate() (proj/src/sim.cpp:126-136), made a pipeline: queries are
 * dispatched in arrival order round-robin over `queue_depth` lanes (each a
 * compute stream with its own scratch slot), so query i+1's embedding gather
 * overlaps query i's latency-bound FC tail; results are delivered in FIFO
 * order. outs[i] receives query i's logits. Host-resident queries are staged
 * by an internal copy stream that runs ahead of compute. When service_ms is
 * non-NULL the call waits and returns per-query service times: gaps between
 * FIFO deliveries (ms; the first from the call's start). latency_ms
 * (optional, needs service_ms) returns each query's residence in the
 * accelerator: input staging start to completion. All queries must share
 * one memory location. Concurrent rs_forward_many calls on one handle are
 * serialised.                                                               */
int rs_forward_many(rs_accel* a, int64_t n, const rs_query* queries,
                    float* const* outs, void* stream, double* service_ms,
                    double* latency_ms);

/* rs_forward_many plus a completion stamp: `done_event` (a cudaEvent_t the
 * caller created; may be NULL) is recorded on `stream` once every query of
 * the call has completed on the device — before the host reads the
 * per-query timestamps — so a caller's CUDA-event bracket around the call
 * measures device time only.                                                */
int rs_forward_many_ev(rs_accel* a, int64_t n, const rs_query* queries,
                       float* const* outs, void* stream, double* service_ms,
                       double* latency_ms, void* done_event);

/* Real-time serving over K replicas (one handle per GPU, same model): query i
 * is released at host time t0 + arrival_s[i] (non-decreasing), dispatched to
 * the replica with the least outstanding items (ties to the lowest index; the
 * reference's FIFO accelerator generalised to a K-server pool) and served on
 * its lanes like rs_forward_many. latency_ms[i] = completion (CUDA events)
 * minus arrival: queueing + service. Synchronous; all queries one location. */
int rs_serve(rs_accel* const* replicas, int32_t k, int64_t n, const rs_query* queries,
             const double* arrival_s, float* const* outs, double* latency_ms);

/* Runtime options of a handle.
 * RS_OPT_MERGE_QUERIES (default 1 = off): rs_forward_many stages up to
 *   `value` (1..64) consecutive queries of one index type whose items fit
 *   max_query_size back to back in one slot and serves them with ONE graph
 *   launch; every merged query completes with the group. A LABELLED
 *   scheduler extension: the reference never merges distinct
 *   queries.
 * RS_OPT_STAGE_TIMING (default 0): 1 = a timed rs_forward runs a copy of the
 *   forward graph with event-record nodes around the embedding stage and the
 *   predict stack and reports them in rs_timing.embed_ms / fc_ms (the
 *   per-kernel roofline measurement; untimed calls are unaffected).
 * RS_OPT_CTA_PAIRS (default 0): 1 = queries whose 128-row tile count is even
 *   (and >= 256 items; >= 640 when a single FC stack has a layer of >= 256
 *   outputs) run a forward graph whose layers of >= 256 outputs use 256-row
 *   tiles on CTA pairs (tcgen05.mma.cta_group::2), captured on first use.
 *   For queues of uniform query size: faster there (MT-WND 1000 items -10%,
 *   WND -22% per query), slower in a mixed-size stream.   */
enum { RS_OPT_MERGE_QUERIES = 1, RS_OPT_STAGE_TIMING = 2, RS_OPT_CTA_PAIRS = 3 };
int rs_accel_set_option(rs_accel* a, int32_t option, int64_t value);

/* Wait for `stream` and report (then clear) errors that asynchronous calls
 * left in the handle's sticky error words (e.g. RS_E_INDEX).               */
int rs_sync(rs_accel* a, void* stream);

/* Embedding stage only (parity hook): writes the pooled sparse features
 * f32[S * pooled_dim] — [S,T,D] sums (Sum), [S,T*L*D] (Concat),
 * [S,T,D] attention-weighted sums (AttentionFC), [S,T,h] final GRU
 * states (AttentionRNN).                                                    */
int rs_pooled(rs_accel* a, const rs_query* q, float* out, void* stream,
              rs_timing* timing);

/* Measured whole-query service time for S items (seconds), memoised per S
 * like the accel_time cache of simulate() (proj/src/sim.cpp:81-88):
 * host-staged synthetic inputs, H2D + forward + D2H, median of 5 runs.     */
int rs_service_time(rs_accel* a, int64_t query_size, double* seconds);

/* Measured counterpart of the whole recsim::ServiceTime (platform.hpp:60-68)
 * for S items: *total (seconds, median of 5 timed host-staged queries),
 * *transfer (H2D + D2H of those queries) and per_category[RS_NUM_OP_CATEGORIES]
 * (the compute time total - transfer, split from measured stage times —
 * embedding stage, predict stack, remaining dense work — and within a stage
 * by the categories' B200 roofline weights from work(); sums to the compute
 * time, as the reference's apportioning does, platform.cpp:121-134).        */
int rs_service_breakdown(rs_accel* a, int64_t query_size, double* total,
                         double* transfer, double* per_category);

/* Synthetic query inputs: dense U(-1,1), indices uniform in
 * [0, rows_per_table), a pure function of (seed, query_id).                */
int rs_fill_query(const rs_model_desc* m, int64_t rows_per_table,
                  uint64_t seed, uint64_t query_id, int64_t size,
                  float* dense, int64_t* indices);

/* As rs_fill_query, but indices follow a bounded power law (Zipf-like,
 * exponent alpha > 0): index k in [0, rows) drawn with probability ~
 * (k+1)^-alpha by inverse transform of the continuous density on
 * [1, rows+1), so low indices are the hot rows (frequency-sorted ids).
 * SURVEY §8d's Zipf(1.05) variant for the L2-persistence run.             */
int rs_fill_query_zipf(const rs_model_desc* m, int64_t rows_per_table,
                       uint64_t seed, uint64_t query_id, int64_t size,
                       double alpha, float* dense, int64_t* indices);

/* SparseLengthsSum on the host cores for the CPU side of the split
 * (replaces the costed EmbeddingLookup/Sum work of
 * cpu_service_time, proj/src/platform.cpp:71-103, for sub-queries routed to
 * CPU by proj/src/sim.cpp:173-191). tables f32[T][rows][D] in host memory,
 * indices i64[S][T][L], pooled f32[S][T][D]. Bit-identical to rs_pooled's
 * Sum path (same canonical order). threads <= 0: all hardware threads.
 * RS_E_INDEX for an index outside [0, rows_per_table).                     */
int rs_host_sls(const float* tables, int64_t rows_per_table, int32_t num_tables,
                int32_t lookups, int32_t dim, int64_t query_size,
                const int64_t* indices, float* pooled, int32_t threads);

/* Fully connected layer on the host cores (the GEMM half of
 * the CPU side of the split; replaces the costed DenseFC/PredictFC flops of
 * cpu_service_time, proj/src/platform.cpp:71-103):
 * y[rows][out] = act(bias + x[rows][in] * weight^T), weight f32[out][ldw]
 * (row stride ldw >= in; 0 = in — the device layout pads rows to
 * round4(in), so device-layout weights pass as is), bias may be
 * NULL, relu != 0 applies ReLU. fp32 with FMA; DESIGN.md §4 tolerance, not
 * bit identity. threads <= 0: every core this process may run on.          */
int rs_host_fc(const float* x, int64_t rows, int32_t in_dim, const float* weight, int64_t ldw,
               const float* bias, int32_t out_dim, int32_t relu, float* y,
               int32_t threads);

/* ---- the CPU side of the split: whole model on the host cores ------------
 * DeepRecSched sends every query of size <= T to the CPU as floor(S/B)
 * requests of B items plus one of S mod B (proj/src/sim.cpp:184-188), each
 * served whole by one core (sim.cpp:114-124) and priced by cpu_service_time
 * (proj/src/platform.cpp:71-97). rs_host_model holds the same model as an
 * rs_accel (tables + weights from the same seeded init) in host
 * memory; rs_host_forward executes one request on the host cores: the same
 * operator order and widths as the device graph, logits within the fp32
 * tolerance rule of the oracle, SLS sums bit-identical to the device.       */
typedef struct rs_host_model rs_host_model;
/* threads <= 0: every core this process may run on (sched_getaffinity) for
 * the table fill at create.                                                  */
int rs_host_model_create(const rs_model_desc* model, const rs_init_desc* init,
                         int32_t threads, rs_host_model** out);
int rs_host_model_destroy(rs_host_model* h);
/* One request (host memory, index_type 0): logits f32[S * stacks * out_dim].
 * threads <= 1: the calling thread alone (the reference's one core per
 * request); > 1: the request's items dealt to that many threads.
 * RS_E_INDEX for an index outside [0, rows_per_table).                     */
int rs_host_forward(rs_host_model* h, const rs_query* q, float* out, int32_t threads);

/* Real-time DeepRecSched over this host's cores AND K accelerator replicas:
 * query i is released at t0 + arrival_s[i]; if threshold > 0 and S >
 * threshold it is offloaded whole to the least-loaded replica (as rs_serve),
 * else split into floor(S/B) requests of `batch` items plus one of S mod B
 * pushed to a FIFO served by `cores` worker threads, each request run by
 * rs_host_forward on one thread (proj/src/sim.cpp:173-191). latency_ms[i]:
 * completion (all of a query's requests, or its CUDA event) minus arrival;
 * offloaded[i] (may be NULL): 1 if the query went to a replica. Queries are
 * host memory; k = 0 serves CPU only (threshold ignored).                   */
int rs_serve_hybrid(rs_host_model* cpu, int32_t cores, int64_t batch, int64_t threshold,
                    rs_accel* const* replicas, int32_t k, int64_t n, const rs_query* queries,
                    const double* arrival_s, float* const* outs, double* latency_ms,
                    int32_t* offloaded);

/* Pinned host memory for rs_query buffers. rs_alloc_pinned_flags accepts
 * RS_PINNED_WRITE_COMBINED for input buffers the host only writes (faster
 * H2D over PCIe; host reads from it are very slow).                         */
enum { RS_PINNED_DEFAULT = 0, RS_PINNED_WRITE_COMBINED = 1 };
int rs_alloc_pinned(size_t bytes, void** out);
int rs_alloc_pinned_flags(size_t bytes, uint32_t flags, void** out);
int rs_free_pinned(void* p);

int rs_device_count(int* out);
/* Build flags of the loaded library: RS_BUILD_EXPERIMENTS = the measured-
 * slower alternatives (SLS variants 1/3/4, RS_FC_CHAIN, RS_SPLITK,
 * RS_DENSE_SMS, RS_DESC_MEMOP) are compiled in (make EXPERIMENTS=1); the
 * product build leaves them out and ignores those environment knobs.        */
enum { RS_BUILD_EXPERIMENTS = 1 };
int rs_build_flags(void);
const char* rs_last_error(void);
int rs_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RS_ACCEL_H */
