/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h for scope and parity
 * status). CPU restatement of the offloaded forward pass plus the frozen
 * initialisation spec of DESIGN.md §3, written independently of the product
 * sources so that agreement between the two is evidence, not tautology.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

/* ---- seeded parameter lattice -------------------------------- */
static uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t key_of(uint64_t seed, uint64_t id) { return sm64(seed ^ (id * 0xD1B54A32D192ED03ull)); }
static float lattice(uint64_t h) {
  int32_t q = (int32_t)(h >> 40) - 8388608; /* 24-bit signed */
  return (float)q * (1.0f / 8388608.0f);
}
static float pval(uint64_t key, uint64_t e, float bound) { return lattice(sm64(key + e)) * bound; }
static float fan(int64_t n) { return 1.0f / sqrtf((float)n); }

float or_table_value(uint64_t seed, int64_t t, int64_t r, int64_t c, int64_t D) {
  return pval(key_of(seed, 0x1000ull + (uint64_t)t), (uint64_t)(r * D + c), 0.05f);
}

void or_fill_query(const or_model* m, int64_t rows, uint64_t seed, uint64_t q, int64_t S,
                   float* dense, int64_t* idx) {
  const uint64_t nd = (uint64_t)(S * m->dense_in);
  if (dense) {
    const uint64_t k = key_of(seed, 0x70000000000ull + q);
    for (uint64_t i = 0; i < nd; ++i) dense[i] = lattice(sm64(k + i));
  }
  const uint64_t ni = (uint64_t)(S * m->T * m->L);
  if (idx) {
    const uint64_t k = key_of(seed, 0x80000000000ull + q);
    for (uint64_t i = 0; i < ni; ++i)
      idx[i] = (int64_t)(((unsigned __int128)sm64(k + i) * (unsigned __int128)(uint64_t)rows) >> 64);
  }
}

/* ---- state ---------------------------------------------------------------- */
struct or_state {
  or_model m;
  int64_t rows;
  uint64_t seed;
  int augru;
  int64_t dense_out, p_in, pooled_dim;
  uint64_t tkey[4096];
  float* tables; /* materialised, or NULL */
  float* dW[8];
  float* db[8];
  float* pW[8]; /* [stacks][out][in] */
  float* pb[8];
  float* att;
  float *wih, *whh, *bih, *bhh, *watt;
};

static float* gen(uint64_t seed, uint64_t id, int64_t n, float bound) {
  float* v = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  const uint64_t k = key_of(seed, id);
  for (int64_t i = 0; i < n; ++i) v[i] = pval(k, (uint64_t)i, bound);
  return v;
}

/* Row t,r of the tables: pointer into the materialised copy, or regenerated
 * into `buf` (D <= 256). NULL when r is out of range. */
static const float* or_row(const or_state* s, int64_t t, int64_t r, float* buf) {
  if (r < 0 || r >= s->rows) return NULL;
  const int64_t D = s->m.D;
  if (s->tables) return s->tables + (t * s->rows + r) * D;
  const uint64_t k = s->tkey[t];
  for (int64_t c = 0; c < D; ++c) buf[c] = pval(k, (uint64_t)(r * D + c), 0.05f);
  return buf;
}

/* Materialise every table element (tables of the 10M-row configs are 82 GB:
 * the fill runs on every core, chunks of rows per work item). */
typedef struct {
  or_state* s;
  atomic_llong next;
} fill_ctx;

static void* fill_worker(void* p) {
  fill_ctx* c = (fill_ctx*)p;
  or_state* s = c->s;
  const int64_t D = s->m.D, rows = s->rows, chunk = 1 << 16;
  const int64_t total = s->m.T * rows;
  for (;;) {
    const int64_t r0 = atomic_fetch_add(&c->next, chunk);
    if (r0 >= total) break;
    const int64_t r1 = r0 + chunk < total ? r0 + chunk : total;
    for (int64_t g = r0; g < r1; ++g) {
      const int64_t t = g / rows, r = g % rows;
      float* dst = s->tables + g * D;
      for (int64_t cc = 0; cc < D; ++cc) dst[cc] = pval(s->tkey[t], (uint64_t)(r * D + cc), 0.05f);
    }
  }
  return NULL;
}

static void fill_tables(or_state* s) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  if (n < 1) n = 1;
  fill_ctx c;
  c.s = s;
  atomic_init(&c.next, 0);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n);
  for (long i = 0; i < n; ++i) pthread_create(&th[i], NULL, fill_worker, &c);
  for (long i = 0; i < n; ++i) pthread_join(th[i], NULL);
  free(th);
}

or_state* or_create(const or_model* m, int64_t rows, uint64_t seed, int augru, int materialize) {
  if (m->T > 4096 || m->D > 256 || m->dense_fc.n > 8 || m->predict_fc.n > 8) return NULL;
  or_state* s = (or_state*)calloc(1, sizeof(or_state));
  s->m = *m;
  s->rows = rows;
  s->seed = seed;
  s->augru = augru;
  s->dense_out = m->has_dense_fc ? m->dense_fc.dims[m->dense_fc.n - 1] : m->dense_in;
  int64_t sparse = 0;
  switch (m->pooling) {
    case 0: sparse = m->D; break;
    case 1: sparse = m->T * m->L * m->D; break;
    case 2: sparse = m->T * m->D; break;
    case 3: sparse = m->T * m->hidden; break;
  }
  int64_t pairs = 0;
  if (m->pooling == 0 && m->has_dense_fc) pairs = (m->T + 1) * m->T / 2;
  s->p_in = s->dense_out + sparse + pairs;
  if (s->p_in < 1) s->p_in = 1;
  switch (m->pooling) {
    case 0: s->pooled_dim = m->T * m->D; break;
    case 1: s->pooled_dim = m->T * m->L * m->D; break;
    case 2: s->pooled_dim = m->T * m->D; break;
    case 3: s->pooled_dim = m->T * m->hidden; break;
  }
  for (int64_t t = 0; t < m->T; ++t) s->tkey[t] = key_of(seed, 0x1000ull + (uint64_t)t);
  if (materialize && m->T > 0) {
    s->tables = (float*)malloc(sizeof(float) * (size_t)(m->T * rows * m->D));
    if (!s->tables) { free(s); return NULL; }
    fill_tables(s);
  }
  if (m->has_dense_fc) {
    int64_t in = m->dense_in;
    for (int l = 0; l < m->dense_fc.n; ++l) {
      const int64_t o = m->dense_fc.dims[l];
      s->dW[l] = gen(seed, 0x2000ull + 2ull * (uint64_t)l, o * in, fan(in));
      s->db[l] = gen(seed, 0x2001ull + 2ull * (uint64_t)l, o, fan(in));
      in = o;
    }
  }
  {
    int64_t in = s->p_in;
    for (int l = 0; l < m->predict_fc.n; ++l) {
      const int64_t o = m->predict_fc.dims[l];
      s->pW[l] = (float*)malloc(sizeof(float) * (size_t)(m->stacks * o * in));
      s->pb[l] = (float*)malloc(sizeof(float) * (size_t)(m->stacks * o));
      for (int64_t z = 0; z < m->stacks; ++z) {
        const uint64_t wid = 0x3000ull + 64ull * (uint64_t)z + 2ull * (uint64_t)l;
        float* w = gen(seed, wid, o * in, fan(in));
        float* b = gen(seed, wid + 1, o, fan(in));
        memcpy(s->pW[l] + z * o * in, w, sizeof(float) * (size_t)(o * in));
        memcpy(s->pb[l] + z * o, b, sizeof(float) * (size_t)o);
        free(w); free(b);
      }
      in = o;
    }
  }
  const int64_t T = m->T, D = m->D, H = m->hidden;
  if (m->pooling == 2 && T > 0) {
    s->att = (float*)malloc(sizeof(float) * (size_t)(T * D * D));
    for (int64_t t = 0; t < T; ++t) {
      float* w = gen(seed, 0x4000ull + (uint64_t)t, D * D, fan(D));
      memcpy(s->att + t * D * D, w, sizeof(float) * (size_t)(D * D));
      free(w);
    }
  }
  if (m->pooling == 3 && T > 0) {
    const int64_t H3 = 3 * H;
    s->wih = (float*)malloc(sizeof(float) * (size_t)(T * H3 * D));
    s->whh = (float*)malloc(sizeof(float) * (size_t)(T * H3 * H));
    s->bih = (float*)malloc(sizeof(float) * (size_t)(T * H3));
    s->bhh = (float*)malloc(sizeof(float) * (size_t)(T * H3));
    s->watt = (float*)malloc(sizeof(float) * (size_t)(T * D * D));
    for (int64_t t = 0; t < T; ++t) {
      const uint64_t base = 0x5000ull + 8ull * (uint64_t)t;
      float* a0 = gen(seed, base + 0, H3 * D, fan(H));
      float* a1 = gen(seed, base + 1, H3 * H, fan(H));
      float* a2 = gen(seed, base + 2, H3, fan(H));
      float* a3 = gen(seed, base + 3, H3, fan(H));
      float* a4 = gen(seed, base + 4, D * D, fan(D));
      memcpy(s->wih + t * H3 * D, a0, sizeof(float) * (size_t)(H3 * D));
      memcpy(s->whh + t * H3 * H, a1, sizeof(float) * (size_t)(H3 * H));
      memcpy(s->bih + t * H3, a2, sizeof(float) * (size_t)H3);
      memcpy(s->bhh + t * H3, a3, sizeof(float) * (size_t)H3);
      memcpy(s->watt + t * D * D, a4, sizeof(float) * (size_t)(D * D));
      free(a0); free(a1); free(a2); free(a3); free(a4);
    }
  }
  return s;
}

void or_destroy(or_state* s) {
  if (!s) return;
  free(s->tables);
  for (int l = 0; l < 8; ++l) { free(s->dW[l]); free(s->db[l]); free(s->pW[l]); free(s->pb[l]); }
  free(s->att); free(s->wih); free(s->whh); free(s->bih); free(s->bhh); free(s->watt);
  free(s);
}

int64_t or_predict_input_dim(const or_state* s) { return s->p_in; }
int64_t or_output_dim(const or_state* s) {
  return s->m.stacks * s->m.predict_fc.dims[s->m.predict_fc.n - 1];
}
int64_t or_pooled_dim(const or_state* s) { return s->pooled_dim; }

/* ---- the two precisions ---------------------------------------------------- */
#define REAL double
#define FN(x) x##_f64
#include "forward_impl.h"
#undef REAL
#undef FN
#define REAL float
#define FN(x) x##_f32
#define FAST_FC 1
#include "forward_impl.h"
#undef FAST_FC
#undef REAL
#undef FN

int or_forward64(const or_state* s, int64_t S, const float* dense, const int64_t* idx,
                 double* out, double* mag, double* pooled, double* pooled_mag) {
  if (!s || S < 1 || !out) return -1;
  return forward_f64(s, S, dense, idx, out, mag, pooled, pooled_mag);
}

/* Items are independent: the fp64 forward over item chunks on `threads`
 * pthreads (test-time speed only; each item's arithmetic is unchanged). */
typedef struct {
  const or_state* s;
  int64_t S, chunk;
  const float* dense;
  const int64_t* idx;
  double *out, *mag, *pooled, *pmag;
  atomic_llong next;
  atomic_int rc;
} f64_ctx;

static void* f64_worker(void* p) {
  f64_ctx* c = (f64_ctx*)p;
  const or_state* s = c->s;
  const int64_t ow = or_output_dim(s), pd = s->pooled_dim, TL = s->m.T * s->m.L;
  for (;;) {
    const int64_t i0 = atomic_fetch_add(&c->next, c->chunk);
    if (i0 >= c->S) break;
    const int64_t n = c->S - i0 < c->chunk ? c->S - i0 : c->chunk;
    const int rc = forward_f64(s, n, c->dense ? c->dense + i0 * s->m.dense_in : NULL,
                               c->idx ? c->idx + i0 * TL : NULL, c->out + i0 * ow,
                               c->mag ? c->mag + i0 * ow : NULL,
                               c->pooled ? c->pooled + i0 * pd : NULL,
                               c->pmag ? c->pmag + i0 * pd : NULL);
    if (rc) atomic_store(&c->rc, rc);
  }
  return NULL;
}

int or_forward64_mt(const or_state* s, int64_t S, const float* dense, const int64_t* idx,
                    double* out, double* mag, double* pooled, double* pooled_mag, int threads) {
  if (!s || S < 1 || !out) return -1;
  if (threads < 1) threads = 1;
  f64_ctx c;
  c.s = s; c.S = S; c.chunk = 16;
  c.dense = dense; c.idx = idx; c.out = out; c.mag = mag; c.pooled = pooled; c.pmag = pooled_mag;
  atomic_init(&c.next, 0);
  atomic_init(&c.rc, 0);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, f64_worker, &c);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
  return atomic_load(&c.rc);
}

int or_forward32(const or_state* s, int64_t S, const float* dense, const int64_t* idx,
                 float* out) {
  if (!s || S < 1 || !out) return -1;
  return forward_f32(s, S, dense, idx, out, NULL, NULL, NULL);
}

int or_sls_canonical(const or_state* s, int64_t S, const int64_t* idx, float* pooled) {
  const int64_t T = s->m.T, L = s->m.L, D = s->m.D;
  int R = 1;
  if (D == 8 || D == 16 || D == 32 || D == 64 || D == 128 || D == 256) {
    const int64_t lpr = D / 4 < 32 ? D / 4 : 32;
    R = (int)(32 / lpr);
  }
  /* R-interleaved partials over the whole bag, pairwise tree (R = 1: one
   * sequential sum). */
  const int64_t CH = L;
  float row[256];
  float part[32][256];
  float total[256];
  for (int64_t bag = 0; bag < S * T; ++bag) {
    const int64_t t = bag % T;
    for (int64_t l0 = 0; l0 < L; l0 += CH) {
      const int64_t n = L - l0 < CH ? L - l0 : CH;
      for (int g = 0; g < R; ++g)
        for (int64_t c = 0; c < D; ++c) part[g][c] = 0.0f;
      for (int64_t l = l0; l < l0 + n; ++l) {
        const float* e = or_row(s, t, idx[bag * L + l], row);
        if (!e) return -7;
        float* p = part[(l - l0) % R];
        for (int64_t c = 0; c < D; ++c) p[c] = p[c] + e[c];
      }
      for (int half = R / 2; half >= 1; half /= 2)
        for (int g = 0; g < half; ++g)
          for (int64_t c = 0; c < D; ++c) part[g][c] = part[g][c] + part[g + half][c];
      for (int64_t c = 0; c < D; ++c) total[c] = l0 == 0 ? part[0][c] : total[c] + part[0][c];
    }
    for (int64_t c = 0; c < D; ++c) pooled[bag * D + c] = total[c];
  }
  return 0;
}

/* ---- multi-threaded CPU throughput driver ----------------------------------- */
typedef struct {
  const or_state* s;
  int64_t nq;
  const int64_t* sizes;
  float** dense;
  int64_t** idx;
  atomic_llong next;
  atomic_int rc;
} bench_ctx;

static void* bench_worker(void* p) {
  bench_ctx* c = (bench_ctx*)p;
  const int64_t ow = or_output_dim(c->s);
  int64_t cap = 0;
  float* out = NULL;
  for (;;) {
    const int64_t q = atomic_fetch_add(&c->next, 1);
    if (q >= c->nq) break;
    const int64_t S = c->sizes[q];
    if (S > cap) { free(out); cap = S; out = (float*)malloc(sizeof(float) * (size_t)(S * ow)); }
    const int rc = or_forward32(c->s, S, c->dense[q], c->idx[q], out);
    if (rc) atomic_store(&c->rc, rc);
  }
  free(out);
  return NULL;
}

int or_bench_queries(const or_state* s, int64_t nq, const int64_t* sizes, int threads,
                     uint64_t seed, double* seconds) {
  if (!s || nq < 1 || threads < 1) return -1;
  bench_ctx c;
  c.s = s; c.nq = nq; c.sizes = sizes;
  c.dense = (float**)calloc((size_t)nq, sizeof(float*));
  c.idx = (int64_t**)calloc((size_t)nq, sizeof(int64_t*));
  for (int64_t q = 0; q < nq; ++q) {
    const int64_t S = sizes[q];
    c.dense[q] = (float*)malloc(sizeof(float) * (size_t)(S * s->m.dense_in + 1));
    c.idx[q] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S * s->m.T * s->m.L + 1));
    or_fill_query(&s->m, s->rows, seed, (uint64_t)q, S, c.dense[q], c.idx[q]);
  }
  atomic_init(&c.next, 0);
  atomic_init(&c.rc, 0);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, bench_worker, &c);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  for (int64_t q = 0; q < nq; ++q) { free(c.dense[q]); free(c.idx[q]); }
  free(c.dense); free(c.idx); free(th);
  return atomic_load(&c.rc);
}

/* ---- per-request service times on the host cores ------------------------------
 * `threads` workers each serve `per_thread` requests of `b` items (inputs
 * pre-generated), all starting together, so each measured time carries the
 * memory contention of `threads` active cores — the quantity the
 * reference's cpu_service_time models (proj/src/platform.cpp:71-97, active
 * cores sampled at dispatch, proj/src/sim.cpp:114-124). times[threads *
 * per_thread] receives each request's wall seconds. */
typedef struct {
  const or_state* s;
  int64_t b, per_thread;
  float** dense;
  int64_t** idx;
  double* times;
  atomic_int ready;
  int threads;
  atomic_int rc;
} req_ctx;

typedef struct {
  req_ctx* c;
  int id;
} req_arg;

static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

static void* req_worker(void* p) {
  req_arg* a = (req_arg*)p;
  req_ctx* c = a->c;
  const int64_t ow = or_output_dim(c->s);
  float* out = (float*)malloc(sizeof(float) * (size_t)(c->b * ow));
  atomic_fetch_add(&c->ready, 1);
  while (atomic_load(&c->ready) < c->threads) {
  }
  for (int64_t k = 0; k < c->per_thread; ++k) {
    const int64_t q = (int64_t)a->id * c->per_thread + k;
    const double t0 = now_s();
    const int rc = or_forward32(c->s, c->b, c->dense[q], c->idx[q], out);
    c->times[q] = now_s() - t0;
    if (rc) atomic_store(&c->rc, rc);
  }
  free(out);
  return NULL;
}

int or_time_requests(const or_state* s, int64_t b, int threads, int64_t per_thread, uint64_t seed,
                     double* times) {
  if (!s || b < 1 || threads < 1 || per_thread < 1 || !times) return -1;
  const int64_t nq = (int64_t)threads * per_thread;
  req_ctx c;
  c.s = s; c.b = b; c.per_thread = per_thread; c.times = times; c.threads = threads;
  c.dense = (float**)calloc((size_t)nq, sizeof(float*));
  c.idx = (int64_t**)calloc((size_t)nq, sizeof(int64_t*));
  for (int64_t q = 0; q < nq; ++q) {
    c.dense[q] = (float*)malloc(sizeof(float) * (size_t)(b * s->m.dense_in + 1));
    c.idx[q] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(b * s->m.T * s->m.L + 1));
    or_fill_query(&s->m, s->rows, seed, (uint64_t)q, b, c.dense[q], c.idx[q]);
  }
  atomic_init(&c.ready, 0);
  atomic_init(&c.rc, 0);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  req_arg* args = (req_arg*)malloc(sizeof(req_arg) * (size_t)threads);
  for (int i = 0; i < threads; ++i) {
    args[i].c = &c;
    args[i].id = i;
    pthread_create(&th[i], NULL, req_worker, &args[i]);
  }
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  for (int64_t q = 0; q < nq; ++q) { free(c.dense[q]); free(c.idx[q]); }
  free(c.dense); free(c.idx); free(th); free(args);
  return atomic_load(&c.rc);
}
