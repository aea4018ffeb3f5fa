/*
 * oracle.c — CPU restatement of the reference hot path. TEST INFRASTRUCTURE
 * ONLY (see oracle.h). Plain C, no FMA contraction (-ffp-contract=off), so
 * every floating-point operation rounds exactly where the reference's does.
 *
 * Reference: /root/reference/proj (qvserve, C++20). Citations are file:line.
 */
#include "oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>

static __thread char g_err[512];

const char* qvo_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, unsigned long long a, unsigned long long b) {
  snprintf(g_err, sizeof g_err, fmt, a, b);
  return code;
}

/* ---- rng.hpp:10-57 ------------------------------------------------------ */
#define GAMMA 0x9e3779b97f4a7c15ULL

uint64_t qvo_splitmix64(uint64_t x) { /* rng.hpp:12-18 */
  x += GAMMA;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t qvo_derive_state(uint64_t master, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:50-57 */
  uint64_t s = qvo_splitmix64(master ^ 0x6a09e667f3bcc909ULL);
  s = qvo_splitmix64(s ^ qvo_splitmix64(a ^ 0xbb67ae8584caa73bULL));
  s = qvo_splitmix64(s ^ qvo_splitmix64(b ^ 0x3c6ef372fe94f82bULL));
  s = qvo_splitmix64(s ^ qvo_splitmix64(c ^ 0xa54ff53a5f1d36f1ULL));
  return s;
}

static inline uint64_t rng_next(uint64_t* state) { /* rng.hpp:26-32 */
  *state += GAMMA;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline double rng_uniform(uint64_t* s) { /* rng.hpp:35 */
  return (double)(rng_next(s) >> 11) * 0x1.0p-53;
}
static inline uint64_t rng_below(uint64_t* s, uint64_t n) { /* rng.hpp:42-45 */
  return (uint64_t)(((unsigned __int128)rng_next(s) * n) >> 64);
}

/* ---- synthetic graph: tools/bench.cpp:22-34 ----------------------------- */
int qvo_synthetic_edges(uint64_t n, uint64_t e, uint64_t seed, int weighted, int transposed,
                        uint64_t* src, uint64_t* dst, double* w) {
  if (n == 0) return fail(QVB_ERR_VALIDATION, "empty graph: node count is zero%.0llu%.0llu", 0, 0);
  uint64_t st = qvo_derive_state(seed, 0xBE9C4ULL, 0, 0);
  for (uint64_t i = 0; i < e; ++i) {
    double u = rng_uniform(&st);
    uint64_t s = (uint64_t)(u * u * (double)n); /* bench.cpp:29 */
    uint64_t d = rng_below(&st, n);             /* bench.cpp:30 */
    double wt = 1.0 + rng_uniform(&st);         /* bench.cpp:31; draw consumed */
    if (s > n - 1) s = n - 1;
    if (transposed) { uint64_t t = s; s = d; d = t; }
    src[i] = s;
    dst[i] = d;
    w[i] = weighted ? wt : 1.0;
  }
  return 0;
}

/* build_csr (graph.cpp:16-47): counting sort by source, input order kept. */
int qvo_build_csr(uint64_t n, uint64_t e, const uint64_t* src, const uint64_t* dst,
                  const double* w, uint64_t* row_offsets, uint64_t* col, double* w_out) {
  if (n == 0) return fail(QVB_ERR_VALIDATION, "empty graph: node count is zero%.0llu%.0llu", 0, 0);
  memset(row_offsets, 0, (n + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < e; ++i) {
    if (src[i] >= n || dst[i] >= n)
      return fail(QVB_ERR_VALIDATION, "edge endpoint %llu out of range for node count %llu",
                  src[i] > dst[i] ? src[i] : dst[i], n);
    if (!(w[i] >= 0.0))
      return fail(QVB_ERR_VALIDATION, "negative or NaN edge weight on edge %llu -> %llu", src[i],
                  dst[i]);
    ++row_offsets[src[i] + 1];
  }
  for (uint64_t i = 0; i < n; ++i) row_offsets[i + 1] += row_offsets[i];
  uint64_t* cursor = (uint64_t*)malloc(n * sizeof(uint64_t));
  memcpy(cursor, row_offsets, n * sizeof(uint64_t));
  for (uint64_t i = 0; i < e; ++i) {
    uint64_t at = cursor[src[i]]++;
    col[at] = dst[i];
    w_out[at] = w[i];
  }
  free(cursor);
  return qvo_validate(n, e, row_offsets, col, w_out);
}

int qvo_synthetic_graph(uint64_t n, uint64_t e, uint64_t seed, int weighted, int transposed,
                        uint64_t* row_offsets, uint64_t* col, double* w) {
  uint64_t* s = (uint64_t*)malloc((e ? e : 1) * sizeof(uint64_t));
  uint64_t* d = (uint64_t*)malloc((e ? e : 1) * sizeof(uint64_t));
  double* ww = (double*)malloc((e ? e : 1) * sizeof(double));
  int rc = qvo_synthetic_edges(n, e, seed, weighted, transposed, s, d, ww);
  if (rc == 0) rc = qvo_build_csr(n, e, s, d, ww, row_offsets, col, w);
  free(s);
  free(d);
  free(ww);
  return rc;
}

/* The same graph (tools/bench.cpp:22-34 + build_csr, graph.cpp:16-47) built
 * by `threads` host threads, for papers-scale inputs (1.6B edges) that the
 * sequential generator takes minutes over. SplitMix64 is counter-based:
 * draw j of the stream is mix(state0 + (j+1)*GAMMA), so edge i's three draws
 * (3i, 3i+1, 3i+2) are computed directly. Threads own row ranges and scan
 * the edges in input order, which keeps build_csr's stable order inside a
 * row. Output identical to qvo_synthetic_graph (tests/test_oracle.py). */
static inline uint64_t mix_at(uint64_t st0, uint64_t j) {
  uint64_t z = st0 + (j + 1) * GAMMA;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

typedef struct {
  int phase;
  uint64_t n, e, st0, lo, hi; /* edge range (phase 0) or row range (1, 2) */
  int weighted, transposed;
  uint32_t* row_of;
  uint64_t* ro;     /* phase 1: counts at ro[r+1]; phase 2: cursors */
  uint64_t* col;
  double* w;
} gen_job;

static void* gen_worker(void* arg) {
  gen_job* j = (gen_job*)arg;
  if (j->phase == 0) {
    for (uint64_t i = j->lo; i < j->hi; ++i) {
      double u = (double)(mix_at(j->st0, 3 * i) >> 11) * 0x1.0p-53;
      uint64_t s = (uint64_t)(u * u * (double)j->n);
      if (s > j->n - 1) s = j->n - 1;
      uint64_t d = (uint64_t)(((unsigned __int128)mix_at(j->st0, 3 * i + 1) * j->n) >> 64);
      j->row_of[i] = (uint32_t)(j->transposed ? d : s);
    }
  } else if (j->phase == 1) {
    for (uint64_t i = 0; i < j->e; ++i) {
      uint64_t r = j->row_of[i];
      if (r >= j->lo && r < j->hi) ++j->ro[r + 1];
    }
  } else {
    for (uint64_t i = 0; i < j->e; ++i) {
      uint64_t r = j->row_of[i];
      if (r < j->lo || r >= j->hi) continue;
      uint64_t at = j->ro[r]++;
      uint64_t other;
      if (j->transposed) {
        double u = (double)(mix_at(j->st0, 3 * i) >> 11) * 0x1.0p-53;
        other = (uint64_t)(u * u * (double)j->n);
        if (other > j->n - 1) other = j->n - 1;
      } else {
        other = (uint64_t)(((unsigned __int128)mix_at(j->st0, 3 * i + 1) * j->n) >> 64);
      }
      j->col[at] = other;
      j->w[at] = j->weighted ? 1.0 + (double)(mix_at(j->st0, 3 * i + 2) >> 11) * 0x1.0p-53 : 1.0;
    }
  }
  return NULL;
}

static void run_jobs(gen_job* jobs, int threads) {
  pthread_t th[256];
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, gen_worker, &jobs[t]);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

int qvo_synthetic_graph_mt(uint64_t n, uint64_t e, uint64_t seed, int weighted, int transposed,
                           int threads, uint64_t* ro, uint64_t* col, double* w) {
  if (n == 0) return fail(QVB_ERR_VALIDATION, "empty graph: node count is zero%.0llu%.0llu", 0, 0);
  if (n > 0xFFFFFFFFull) return fail(QVB_ERR_VALIDATION, "threaded generator needs n < 2^32%.0llu%.0llu", 0, 0);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  uint64_t st0 = qvo_derive_state(seed, 0xBE9C4ULL, 0, 0);
  uint32_t* row_of = (uint32_t*)malloc((e ? e : 1) * sizeof(uint32_t));
  if (!row_of) return fail(QVB_ERR_GENERIC, "out of host memory%.0llu%.0llu", 0, 0);
  gen_job jobs[256];
  for (int t = 0; t < threads; ++t)
    jobs[t] = (gen_job){0, n, e, st0, e * t / threads, e * (t + 1) / threads, weighted, transposed,
                        row_of, ro, col, w};
  run_jobs(jobs, threads);
  memset(ro, 0, (n + 1) * sizeof(uint64_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t].phase = 1;
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
  }
  run_jobs(jobs, threads);
  for (uint64_t i = 0; i < n; ++i) ro[i + 1] += ro[i];
  /* phase 2 row ranges balanced by edge count; ro[r] serves as row r's
   * cursor and ends at ro[r+1], so shift it back afterwards */
  uint64_t r = 0;
  for (int t = 0; t < threads; ++t) {
    jobs[t].phase = 2;
    jobs[t].lo = r;
    uint64_t target = e * (uint64_t)(t + 1) / threads;
    while (r < n && ro[r] < target) ++r;
    if (t == threads - 1) r = n;
    jobs[t].hi = r;
  }
  run_jobs(jobs, threads);
  for (uint64_t i = n; i > 0; --i) ro[i] = ro[i - 1];
  ro[0] = 0;
  free(row_of);
  return 0;
}

typedef struct {
  uint64_t first, lo, hi;
  uint32_t dim;
  float* x;
} feat_job;

static void* feat_worker(void* arg) {
  feat_job* j = (feat_job*)arg;
  qvo_features(j->first + j->lo, j->hi - j->lo, j->dim, j->x + j->lo * j->dim);
  return NULL;
}

void qvo_features_mt(uint64_t first, uint64_t count, uint32_t dim, float* x, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  feat_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (feat_job){first, count * t / threads, count * (t + 1) / threads, dim, x};
    pthread_create(&th[t], NULL, feat_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* out[i] = X[ids[i]] straight from the feature generator,
 * without materialising X: the expected rows of a gather over a table too
 * big for host RAM checks (C4: 56.8 GB). */
typedef struct {
  const uint64_t* ids;
  uint32_t dim;
  float* out;
  uint64_t lo, hi;
} rows_job;

static void* rows_worker(void* arg) {
  rows_job* j = (rows_job*)arg;
  for (uint64_t i = j->lo; i < j->hi; ++i) qvo_features(j->ids[i], 1, j->dim, j->out + i * j->dim);
  return NULL;
}

void qvo_feature_rows(const uint64_t* ids, uint64_t b, uint32_t dim, float* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  rows_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (rows_job){ids, dim, out, b * t / threads, b * (t + 1) / threads};
    pthread_create(&th[t], NULL, rows_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* Graph::validate (graph.cpp:58-93) */
int qvo_validate(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                 const double* w) {
  if (n == 0) return fail(QVB_ERR_VALIDATION, "empty graph: node count is zero%.0llu%.0llu", 0, 0);
  if (ro[0] != 0 || ro[n] != e)
    return fail(QVB_ERR_VALIDATION, "row_offsets endpoints invalid%.0llu%.0llu", 0, 0);
  for (uint64_t i = 0; i < n; ++i)
    if (ro[i + 1] < ro[i])
      return fail(QVB_ERR_VALIDATION, "row_offsets not non-decreasing at node %llu%.0llu", i, 0);
  for (uint64_t i = 0; i < n; ++i) {
    int any_positive = ro[i + 1] == ro[i];
    for (uint64_t k = ro[i]; k < ro[i + 1]; ++k) {
      if (col[k] >= n)
        return fail(QVB_ERR_VALIDATION, "column index out of range at node %llu%.0llu", i, 0);
      double wk = w ? w[k] : 1.0;
      if (!(wk >= 0.0))
        return fail(QVB_ERR_VALIDATION, "negative or NaN edge weight at node %llu%.0llu", i, 0);
      if (wk > 0.0) any_positive = 1;
    }
    if (!any_positive)
      return fail(QVB_ERR_VALIDATION, "node %llu has out-edges but all weights are zero%.0llu", i,
                  0);
  }
  return 0;
}

/* in_adjacency (graph.cpp:260-281): counting sort by destination; iterating
 * rows in order keeps each transposed row sorted by source. */
int qvo_in_adjacency(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                     const double* w, uint64_t* tro, uint64_t* tcol, double* tw) {
  int rc = qvo_validate(n, e, ro, col, w);
  if (rc) return rc;
  memset(tro, 0, (n + 1) * sizeof(uint64_t));
  for (uint64_t k = 0; k < e; ++k) ++tro[col[k] + 1];
  for (uint64_t i = 0; i < n; ++i) tro[i + 1] += tro[i];
  uint64_t* cursor = (uint64_t*)malloc(n * sizeof(uint64_t));
  memcpy(cursor, tro, n * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t k = ro[i]; k < ro[i + 1]; ++k) {
      uint64_t at = cursor[col[k]]++;
      tcol[at] = i;
      tw[at] = w ? w[k] : 1.0;
    }
  }
  free(cursor);
  return 0;
}

/* transition_view row sums (graph.cpp:301-316): plain sequential sum. */
int qvo_row_sums(uint64_t n, const uint64_t* ro, const double* w, double* rs) {
  for (uint64_t i = 0; i < n; ++i) {
    double sum = 0.0;
    for (uint64_t k = ro[i]; k < ro[i + 1]; ++k) sum += w ? w[k] : 1.0;
    rs[i] = sum;
  }
  return 0;
}

/* One node of the sweep, metrics.cpp:152-169. */
static inline double sweep_node(uint64_t i, const uint64_t* tro, const uint64_t* tcol,
                                const double* tw, const double* rs, const double* prev) {
  double miss_all = 1.0;
  uint64_t k = tro[i];
  const uint64_t end = tro[i + 1];
  while (k < end) {
    uint64_t s = tcol[k];
    double wt = tw[k];
    ++k;
    while (k < end && tcol[k] == s) { /* coalesce parallel edges, :161-164 */
      wt += tw[k];
      ++k;
    }
    if (rs[s] > 0.0) miss_all *= 1.0 - prev[s] * (wt / rs[s]); /* :165-167 */
  }
  return prev[i] + (1.0 - prev[i]) * (1.0 - miss_all); /* :169 */
}

/* compute_access_prob_ie_impl<false> (metrics.cpp:134-173). */
int qvo_access_prob(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                    const double* w, uint32_t layers, double* out) {
  if (layers < 1)
    return fail(QVB_ERR_VALIDATION, "access probability needs layers >= 1%.0llu%.0llu", 0, 0);
  int rc = qvo_validate(n, e, ro, col, w); /* transition_view + in_adjacency validate */
  if (rc) return rc;
  for (uint64_t i = 0; i < n; ++i) out[i] = 1.0 / (double)n; /* :143 */
  if (layers == 1) return 0;
  uint64_t* tro = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint64_t* tcol = (uint64_t*)malloc((e ? e : 1) * sizeof(uint64_t));
  double* tw = (double*)malloc((e ? e : 1) * sizeof(double));
  double* rs = (double*)malloc(n * sizeof(double));
  double* prev = (double*)malloc(n * sizeof(double));
  qvo_row_sums(n, ro, w, rs);
  qvo_in_adjacency(n, e, ro, col, w, tro, tcol, tw); /* :145 */
  for (uint32_t j = 2; j <= layers; ++j) {
    memcpy(prev, out, n * sizeof(double)); /* :149 */
    for (uint64_t i = 0; i < n; ++i) out[i] = sweep_node(i, tro, tcol, tw, rs, prev);
  }
  free(tro);
  free(tcol);
  free(tw);
  free(rs);
  free(prev);
  return 0;
}

int qvo_access_prob_sweep_nodes(uint64_t n, const uint64_t* tro, const uint64_t* tcol,
                                const double* tw, const double* rs, const double* prev,
                                const uint64_t* nodes, uint64_t count, double* out) {
  for (uint64_t k = 0; k < count; ++k) {
    if (nodes[k] >= n) return fail(QVB_ERR_VALIDATION, "node %llu out of range %llu", nodes[k], n);
    out[k] = sweep_node(nodes[k], tro, tcol, tw, rs, prev);
  }
  return 0;
}

/* ---- compute_fap (metrics.cpp:95-132), distribution_step (:42-58) ------- */
static inline void neumaier_add(double* sum, double* comp, double v) { /* numeric.hpp:14-23 */
  double t = *sum + v;
  if (fabs(*sum) >= fabs(v)) *comp += (*sum - t) + v;
  else *comp += (v - t) + *sum;
  *sum = t;
}

int qvo_compute_fap(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                    const double* w, uint32_t hops, const double* seed, double* values) {
  int rc = qvo_validate(n, e, ro, col, w); /* transition_view validates */
  if (rc) return rc;
  double* p0 = (double*)malloc(n * sizeof(double));
  if (seed) { /* :100-112 */
    double sum = 0.0, comp = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      if (!(seed[i] >= 0.0)) {
        free(p0);
        return fail(QVB_ERR_VALIDATION, "seed distribution has negative mass%.0llu%.0llu", 0, 0);
      }
      neumaier_add(&sum, &comp, seed[i]);
    }
    if (fabs((sum + comp) - 1.0) > 1e-12) {
      free(p0);
      return fail(QVB_ERR_VALIDATION, "seed distribution does not sum to 1%.0llu%.0llu", 0, 0);
    }
    memcpy(p0, seed, n * sizeof(double));
  } else {
    for (uint64_t i = 0; i < n; ++i) p0[i] = 1.0 / (double)n;
  }
  memcpy(values, p0, n * sizeof(double)); /* hop-0 term */
  uint64_t* tro = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint64_t* tcol = (uint64_t*)malloc((e ? e : 1) * sizeof(uint64_t));
  double* tw = (double*)malloc((e ? e : 1) * sizeof(double));
  double* rs = (double*)malloc(n * sizeof(double));
  double* next = (double*)malloc(n * sizeof(double));
  qvo_row_sums(n, ro, w, rs);
  qvo_in_adjacency(n, e, ro, col, w, tro, tcol, tw);
  double* cur = p0;
  for (uint32_t k = 1; k <= hops; ++k) {
    for (uint64_t i = 0; i < n; ++i) {
      double sum = 0.0, comp = 0.0;
      for (uint64_t q = tro[i]; q < tro[i + 1]; ++q) {
        uint64_t j = tcol[q];
        if (rs[j] > 0.0) neumaier_add(&sum, &comp, cur[j] * tw[q] / rs[j]);
      }
      next[i] = sum + comp;
    }
    for (uint64_t i = 0; i < n; ++i) values[i] += next[i];
    double* t = cur;
    cur = next;
    next = t;
  }
  free(cur == p0 ? next : p0);
  free(cur);
  free(tro);
  free(tcol);
  free(tw);
  free(rs);
  return 0;
}

/* ---- sampler (sampler.cpp:21-149) ---------------------------------------- */
typedef struct {
  double key;
  uint64_t idx;
} keyidx_t;
static int cmp_keyidx(const void* a, const void* b) { /* std::pair<double,size_t> order */
  const keyidx_t *x = (const keyidx_t*)a, *y = (const keyidx_t*)b;
  if (x->key < y->key) return -1;
  if (y->key < x->key) return 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* One seed's k-hop sample (sample_khop, sampler.cpp:56-112). Appends the
 * frontier instances of hops 0..hops to nodes (seed first) and writes the
 * per-hop counts. Returns the number of instances appended, or -1 on error. */
static int64_t sample_khop(uint64_t n, const uint64_t* ro, const uint64_t* col, const double* w,
                           int parallel, uint64_t seed, const uint32_t* fanouts, uint32_t hops,
                           uint64_t rng_seed, uint64_t** nodes, uint64_t* cap, uint64_t at,
                           uint64_t* counts) {
  uint64_t start = at;
  if (at + 1 > *cap) {
    *cap = (*cap + 1) * 2;
    *nodes = (uint64_t*)realloc(*nodes, *cap * sizeof(uint64_t));
  }
  (*nodes)[at++] = seed;
  counts[0] = 1;
  uint64_t prev_lo = start, prev_hi = at;
  for (uint32_t k = 1; k <= hops; ++k) {
    for (uint64_t pi = prev_lo; pi < prev_hi; ++pi) {
      uint64_t p = (*nodes)[pi], idx = pi - prev_lo;
      uint64_t a = ro[p], b = ro[p + 1];
      /* candidates: coalesced in first-occurrence order when the graph has
       * parallel edges (sampler.cpp:75-90) */
      uint64_t L = 0;
      uint64_t* cn = (uint64_t*)malloc((b - a + 1) * sizeof(uint64_t));
      double* cw = (double*)malloc((b - a + 1) * sizeof(double));
      for (uint64_t q = a; q < b; ++q) {
        uint64_t j = col[q];
        int merged = 0;
        if (parallel)
          for (uint64_t t = 0; t < L; ++t)
            if (cn[t] == j) {
              cw[t] += w[q];
              merged = 1;
              break;
            }
        if (!merged) {
          cn[L] = j;
          cw[L] = w[q];
          ++L;
        }
      }
      uint64_t st = qvo_derive_state(rng_seed, k, idx, p); /* sampler.cpp:94 */
      uint64_t positive = 0;
      for (uint64_t t = 0; t < L; ++t) positive += cw[t] > 0.0;
      uint64_t m = positive < fanouts[k - 1] ? positive : fanouts[k - 1];
      if (at + m > *cap) {
        *cap = (at + m) * 2;
        *nodes = (uint64_t*)realloc(*nodes, *cap * sizeof(uint64_t));
      }
      if (m > 0 && m == positive) {
        for (uint64_t t = 0; t < L; ++t)
          if (cw[t] > 0.0) (*nodes)[at++] = cn[t];
      } else if (m > 0) {
        keyidx_t* keys = (keyidx_t*)malloc(L * sizeof(keyidx_t));
        uint64_t nk = 0;
        for (uint64_t t = 0; t < L; ++t) {
          double e = -log1p(-rng_uniform(&st)); /* rng.hpp:38: exponential() */
          if (cw[t] > 0.0) {
            keys[nk].key = e / cw[t];
            keys[nk].idx = t;
            ++nk;
          }
        }
        qsort(keys, nk, sizeof(keyidx_t), cmp_keyidx); /* == nth_element's m smallest */
        uint64_t* pick = (uint64_t*)malloc(m * sizeof(uint64_t));
        for (uint64_t t = 0; t < m; ++t) pick[t] = keys[t].idx;
        qsort(pick, m, sizeof(uint64_t), cmp_u64); /* candidate order */
        for (uint64_t t = 0; t < m; ++t) (*nodes)[at++] = cn[pick[t]];
        free(pick);
        free(keys);
      }
      free(cn);
      free(cw);
    }
    counts[k] = at - prev_hi;
    prev_lo = prev_hi;
    prev_hi = at;
  }
  (void)n;
  return (int64_t)(at - start);
}

/* batch_sample (sampler.cpp:114-149): per-seed frontiers flattened into
 * nodes_out (seed-major, hop-major, instance order) with counts_out[s*(hops+1)+k];
 * the sorted union of all sampled nodes in unique_out. Two-phase: call with
 * nodes_out == NULL to get *total and *unique_count. */
int qvo_batch_sample(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                     const double* w, const uint64_t* seeds, uint64_t nseeds,
                     const uint32_t* fanouts, uint32_t hops, uint64_t rng_seed,
                     uint64_t* total, uint64_t* unique_count, uint64_t* nodes_out,
                     uint64_t* counts_out, uint64_t* unique_out) {
  int rc = qvo_validate(n, e, ro, col, w);
  if (rc) return rc;
  if (hops == 0) return fail(QVB_ERR_VALIDATION, "sampling config needs >= 1 hop%.0llu%.0llu", 0, 0);
  for (uint32_t k = 0; k < hops; ++k)
    if (fanouts[k] < 1) return fail(QVB_ERR_VALIDATION, "fanouts must be >= 1%.0llu%.0llu", 0, 0);
  for (uint64_t i = 0; i < nseeds; ++i)
    if (seeds[i] >= n)
      return fail(QVB_ERR_VALIDATION, "batch seed at position %llu (node %llu) out of range", i,
                  seeds[i]);
  /* transition_view's has_parallel_edges (graph.cpp:299-313) */
  int parallel = 0;
  uint64_t* stamp = (uint64_t*)malloc(n * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) stamp[i] = ~0ull;
  for (uint64_t i = 0; i < n && !parallel; ++i)
    for (uint64_t q = ro[i]; q < ro[i + 1]; ++q) {
      if (stamp[col[q]] == i) {
        parallel = 1;
        break;
      }
      stamp[col[q]] = i;
    }
  free(stamp);
  uint64_t cap = 1024, at = 0;
  uint64_t* nodes = (uint64_t*)malloc(cap * sizeof(uint64_t));
  uint64_t* counts = (uint64_t*)malloc((hops + 1) * (nseeds ? nseeds : 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < nseeds; ++i) {
    uint64_t s = seeds[i];
    uint64_t rs = qvo_splitmix64(rng_seed ^ s * 0x9e3779b97f4a7c15ULL); /* sampler.cpp:136 */
    int64_t got = sample_khop(n, ro, col, w, parallel, s, fanouts, hops, rs, &nodes, &cap, at,
                              counts + i * (hops + 1));
    at += (uint64_t)got;
  }
  *total = at;
  uint64_t* u = (uint64_t*)malloc((at ? at : 1) * sizeof(uint64_t));
  memcpy(u, nodes, at * sizeof(uint64_t));
  qsort(u, at, sizeof(uint64_t), cmp_u64);
  uint64_t uc = 0;
  for (uint64_t i = 0; i < at; ++i)
    if (i == 0 || u[i] != u[i - 1]) u[uc++] = u[i];
  *unique_count = uc;
  if (nodes_out) {
    memcpy(nodes_out, nodes, at * sizeof(uint64_t));
    memcpy(counts_out, counts, nseeds * (hops + 1) * sizeof(uint64_t));
    memcpy(unique_out, u, uc * sizeof(uint64_t));
  }
  free(u);
  free(nodes);
  free(counts);
  return 0;
}

/* ---- fap_ranking (placement.cpp:79-87) ---------------------------------- */
static const double* g_rank_values;
static int rank_cmp(const void* pa, const void* pb) {
  uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
  double va = g_rank_values[a], vb = g_rank_values[b];
  if (va != vb) return va > vb ? -1 : 1; /* value descending */
  return a < b ? -1 : (a > b ? 1 : 0);  /* id ascending */
}
/* The comparator is a strict total order on non-NaN input, so qsort gives
 * exactly std::stable_sort's permutation. */
int qvo_rank_desc(const double* values, uint64_t n, uint64_t* ranks) {
  for (uint64_t i = 0; i < n; ++i) {
    if (values[i] != values[i]) return fail(QVB_ERR_VALIDATION, "NaN value at %llu%.0llu", i, 0);
    ranks[i] = i;
  }
  g_rank_values = values;
  qsort(ranks, n, sizeof(uint64_t), rank_cmp);
  return 0;
}

/* ---- topology helpers (topology.cpp:42-64, placement.cpp:25-51) --------- */
static int topo_validate(const qvb_topology* t) {
  if (t->servers < 1) return fail(QVB_ERR_VALIDATION, "topology: servers must be >= 1%.0llu%.0llu", 0, 0);
  if (t->numa_per_server < 1)
    return fail(QVB_ERR_VALIDATION, "topology: numa_per_server must be >= 1%.0llu%.0llu", 0, 0);
  if (t->gpus_per_server % t->numa_per_server != 0)
    return fail(QVB_ERR_VALIDATION,
                "topology: gpus_per_server must be divisible by numa_per_server%.0llu%.0llu", 0, 0);
  for (int i = 0; i < QVB_LINK_COUNT; ++i) {
    if (!(t->link_bandwidth_Bps[i] > 0.0))
      return fail(QVB_ERR_VALIDATION, "topology: non-positive bandwidth for link %llu%.0llu", i, 0);
    if (t->link_latency_s[i] < 0.0)
      return fail(QVB_ERR_VALIDATION, "topology: negative latency for link %llu%.0llu", i, 0);
  }
  if (t->tlb_miss_penalty_s < 0.0)
    return fail(QVB_ERR_VALIDATION, "topology: negative tlb_miss_penalty_s%.0llu%.0llu", 0, 0);
  if (t->gpu_replicated_capacity > t->gpu_feature_capacity)
    return fail(QVB_ERR_VALIDATION,
                "topology: gpu_replicated_capacity %llu exceeds gpu_feature_capacity %llu",
                t->gpu_replicated_capacity, t->gpu_feature_capacity);
  return 0;
}

static inline int64_t enc(const qvb_topology* t, uint32_t server, int tier, uint32_t dev) {
  int64_t stride = (int64_t)t->gpus_per_server + 2, base = (int64_t)server * stride;
  if (tier == QVB_TIER_GPU) return base + dev;
  if (tier == QVB_TIER_HOST) return base + t->gpus_per_server;
  return base + t->gpus_per_server + 1;
}

/* ---- plan_placement (placement.cpp:94-226) ------------------------------ */
typedef struct {
  uint32_t maxc;
  uint32_t* cnt;
  int64_t* ids;
} copies_t;

static void add_copy(copies_t* c, uint64_t f, int64_t id) {
  c->ids[f * c->maxc + c->cnt[f]++] = id;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* place_gpu_range (placement.cpp:94-123) with the replicated-prefix extension. */
static int place_gpu_range(const uint64_t* range, uint64_t len, const double* v,
                           const qvb_topology* t, uint32_t server, copies_t* c) {
  const uint32_t gpn = t->gpus_per_server / t->numa_per_server;
  if (len == 0 || t->gpus_per_server == 0) return 0;
  uint64_t rep = t->nvlink_within_numa ? t->gpu_replicated_capacity : 0;
  if (rep > len) rep = len;
  for (uint64_t i = 0; i < rep; ++i) /* extension: hottest rep on every GPU */
    for (uint32_t d = 0; d < t->gpus_per_server; ++d) add_copy(c, range[i], enc(t, server, 0, d));
  if (t->nvlink_within_numa) {
    const uint64_t cap = t->gpu_feature_capacity - t->gpu_replicated_capacity;
    double* load = (double*)calloc(gpn, sizeof(double));
    uint64_t* used = (uint64_t*)calloc(gpn, sizeof(uint64_t));
    for (uint64_t i = rep; i < len; ++i) { /* :103-115 */
      uint64_t f = range[i];
      uint32_t best = gpn;
      for (uint32_t s = 0; s < gpn; ++s) {
        if (used[s] >= cap) continue;
        if (best == gpn || load[s] < load[best]) best = s;
      }
      if (best == gpn) {
        free(load);
        free(used);
        return fail(QVB_ERR_GENERIC, "gpu range exceeds numa group capacity%.0llu%.0llu", 0, 0);
      }
      load[best] += v[f];
      ++used[best];
      for (uint32_t g = 0; g < t->numa_per_server; ++g) add_copy(c, f, enc(t, server, 0, g * gpn + best));
    }
    free(load);
    free(used);
  } else {
    for (uint64_t i = 0; i < len; ++i) /* :116-122 */
      for (uint32_t d = 0; d < t->gpus_per_server; ++d) add_copy(c, range[i], enc(t, server, 0, d));
  }
  return 0;
}

static int place_server_run(const uint64_t* run, uint64_t len, uint64_t gpu_range_size,
                            const double* v, const qvb_topology* t, uint32_t server, copies_t* c) {
  uint64_t g = len < gpu_range_size ? len : gpu_range_size; /* :158-169 */
  int rc = place_gpu_range(run, g, v, t, server, c);
  if (rc) return rc;
  uint64_t h = len - g < t->host_feature_capacity ? len - g : t->host_feature_capacity;
  for (uint64_t i = 0; i < h; ++i) add_copy(c, run[g + i], enc(t, server, QVB_TIER_HOST, 0));
  for (uint64_t i = g + h; i < len; ++i) add_copy(c, run[i], enc(t, server, QVB_TIER_DISK, 0));
  return 0;
}

int qvo_plan_placement(const double* v, uint64_t n, const qvb_topology* t, uint64_t* loc_offsets,
                       int64_t* loc_ids, uint64_t loc_capacity, uint64_t* copies_out) {
  int rc = topo_validate(t);
  if (rc) return rc;
  if (n == 0) return fail(QVB_ERR_VALIDATION, "placement needs at least one feature%.0llu%.0llu", 0, 0);
  uint64_t* ranks = (uint64_t*)malloc(n * sizeof(uint64_t));
  rc = qvo_rank_desc(v, n, ranks);
  if (rc) {
    free(ranks);
    return rc;
  }
  const uint64_t gpn = t->gpus_per_server / t->numa_per_server;
  const uint64_t rep = t->nvlink_within_numa ? t->gpu_replicated_capacity : 0;
  const uint64_t gpu_range_size =
      t->gpus_per_server == 0 ? 0
      : (t->nvlink_within_numa ? rep + gpn * (t->gpu_feature_capacity - rep)
                               : t->gpu_feature_capacity); /* :147-152 */
  copies_t c;
  c.maxc = t->servers * (t->gpus_per_server + 1);
  c.cnt = (uint32_t*)calloc(n, sizeof(uint32_t));
  c.ids = (int64_t*)malloc(n * (uint64_t)c.maxc * sizeof(int64_t));
  if (!t->infiniband) { /* :171-184 */
    uint64_t per_server = gpu_range_size + t->host_feature_capacity + t->disk_feature_capacity;
    if (n > per_server) {
      snprintf(g_err, sizeof g_err,
               "placement infeasible without infiniband: %llu features vs per-server capacity %llu "
               "(short by %llu)",
               (unsigned long long)n, (unsigned long long)per_server,
               (unsigned long long)(n - per_server));
      rc = QVB_ERR_PLACEMENT;
      goto done;
    }
    for (uint32_t s = 0; s < t->servers && !rc; ++s)
      rc = place_server_run(ranks, n, gpu_range_size, v, t, s, &c);
  } else { /* :185-221 */
    const uint64_t ns = gpu_range_size + t->host_feature_capacity;
    const uint64_t cap_all = (uint64_t)t->servers * ns;
    const uint64_t partitioned = n < cap_all ? n : cap_all;
    for (uint32_t s = 0; s < t->servers && !rc; ++s) {
      uint64_t lo = (uint64_t)s * ns, hi = (uint64_t)(s + 1) * ns;
      if (lo > partitioned) lo = partitioned;
      if (hi > partitioned) hi = partitioned;
      if (lo < hi) rc = place_server_run(ranks + lo, hi - lo, gpu_range_size, v, t, s, &c);
    }
    const uint64_t remainder = n - partitioned;
    if (!rc && remainder > 0) {
      uint64_t disk_total = (uint64_t)t->servers * t->disk_feature_capacity;
      if (remainder > disk_total) {
        snprintf(g_err, sizeof g_err,
                 "placement infeasible: remainder %llu features exceed total disk capacity %llu "
                 "(short by %llu)",
                 (unsigned long long)remainder, (unsigned long long)disk_total,
                 (unsigned long long)(remainder - disk_total));
        rc = QVB_ERR_PLACEMENT;
        goto done;
      }
      uint64_t base = remainder / t->servers, extra = remainder % t->servers, at = partitioned;
      for (uint32_t s = 0; s < t->servers; ++s) {
        uint64_t len = base + (s < extra ? 1 : 0);
        for (uint64_t i = 0; i < len; ++i) add_copy(&c, ranks[at + i], enc(t, s, QVB_TIER_DISK, 0));
        at += len;
      }
    }
  }
  if (rc) goto done;
  /* canonicalize (:125-134): ascending encoded id == (server, tier, device). */
  uint64_t total = 0;
  for (uint64_t f = 0; f < n; ++f) {
    if (c.cnt[f] == 0) {
      rc = fail(QVB_ERR_GENERIC, "feature %llu has no location%.0llu", f, 0);
      goto done;
    }
    qsort(c.ids + f * c.maxc, c.cnt[f], sizeof(int64_t), cmp_i64);
    total += c.cnt[f];
  }
  /* PlacementPlan::validate (:53-74) */
  {
    int64_t nloc = (int64_t)t->servers * (t->gpus_per_server + 2);
    uint64_t* counts = (uint64_t*)calloc((size_t)nloc, sizeof(uint64_t));
    for (uint64_t f = 0; f < n; ++f)
      for (uint32_t k = 0; k < c.cnt[f]; ++k) ++counts[c.ids[f * c.maxc + k]];
    for (int64_t id = 0; id < nloc && !rc; ++id) {
      int64_t slot = id % ((int64_t)t->gpus_per_server + 2);
      uint64_t cap = slot < t->gpus_per_server ? t->gpu_feature_capacity
                     : slot == t->gpus_per_server ? t->host_feature_capacity
                                                  : t->disk_feature_capacity;
      if (counts[id] > cap)
        rc = fail(QVB_ERR_GENERIC, "placement overfills location %llu: %llu", (unsigned long long)id,
                  counts[id]);
    }
    free(counts);
  }
  if (rc) goto done;
  *copies_out = total;
  if (total > loc_capacity) {
    rc = fail(QVB_ERR_VALIDATION, "loc_capacity %llu too small, need %llu", loc_capacity, total);
    goto done;
  }
  {
    uint64_t at = 0;
    for (uint64_t f = 0; f < n; ++f) {
      loc_offsets[f] = at;
      for (uint32_t k = 0; k < c.cnt[f]; ++k) loc_ids[at++] = c.ids[f * c.maxc + k];
    }
    loc_offsets[n] = at;
  }
done:
  free(ranks);
  free(c.cnt);
  free(c.ids);
  return rc;
}

/* ---- classify_link / nominal_read_cost (placement.cpp:228-302) ---------- */
/* Returns first link, *second = -1 if none. Reader is GPU reader_dev of
 * reader_server, or the host when the server has no GPUs (:292-295). */
static int classify(const qvb_topology* t, uint32_t rs, int reader_is_gpu, uint32_t rdev,
                    int64_t id, int* second) {
  int64_t stride = (int64_t)t->gpus_per_server + 2;
  uint32_t server = (uint32_t)(id / stride);
  int64_t slot = id % stride;
  int tier = slot < t->gpus_per_server ? QVB_TIER_GPU
             : slot == t->gpus_per_server ? QVB_TIER_HOST
                                          : QVB_TIER_DISK;
  uint32_t dev = tier == QVB_TIER_GPU ? (uint32_t)slot : 0;
  *second = -1;
  if (server == rs) {
    if (tier == QVB_TIER_GPU) {
      if (reader_is_gpu) {
        uint32_t gpn = t->gpus_per_server / t->numa_per_server;
        if (rdev == dev) return QVB_LINK_LOCAL;
        if (gpn > 0 && rdev / gpn == dev / gpn)
          return t->nvlink_within_numa ? QVB_LINK_NVLINK : QVB_LINK_PCIE;
        return QVB_LINK_UPI;
      }
      return QVB_LINK_PCIE;
    }
    if (tier == QVB_TIER_HOST) return reader_is_gpu ? QVB_LINK_PCIE : QVB_LINK_LOCAL;
    return QVB_LINK_DISK;
  }
  int net = t->infiniband ? QVB_LINK_INFINIBAND : QVB_LINK_ETHERNET;
  if (tier == QVB_TIER_DISK) {
    *second = net;
    return QVB_LINK_DISK;
  }
  return net;
}

static double nominal_cost(const qvb_topology* t, uint32_t rs, int reader_is_gpu, uint32_t rdev,
                           int64_t id) {
  int second;
  int first = classify(t, rs, reader_is_gpu, rdev, id, &second);
  double setup = t->link_latency_s[first];
  double bw = t->link_bandwidth_Bps[first];
  if (second >= 0) {
    setup += t->link_latency_s[second];
    if (t->link_bandwidth_Bps[second] < bw) bw = t->link_bandwidth_Bps[second];
  }
  return setup + 1048576.0 / bw;
}

/* build_lookup_table (placement.cpp:306-342). */
int qvo_build_lookup_table(const uint64_t* loc_offsets, const int64_t* loc_ids, uint64_t n,
                           const qvb_topology* t, uint32_t home, uint32_t reader_dev,
                           int64_t* location_ids, uint64_t* offsets) {
  if (home >= t->servers) return fail(QVB_ERR_VALIDATION, "home server out of range%.0llu%.0llu", 0, 0);
  int64_t nloc = (int64_t)t->servers * (t->gpus_per_server + 2);
  uint64_t* cursor = (uint64_t*)calloc((size_t)nloc, sizeof(uint64_t));
  int reader_is_gpu = t->gpus_per_server > 0;
  for (uint64_t f = 0; f < n; ++f) {
    int64_t best_id = -1;
    double best_cost = 0.0;
    uint64_t best_off = 0;
    for (uint64_t k = loc_offsets[f]; k < loc_offsets[f + 1]; ++k) {
      int64_t id = loc_ids[k];
      if (id < 0 || id >= nloc) {
        free(cursor);
        return fail(QVB_ERR_VALIDATION, "unknown location id %llu%.0llu", (unsigned long long)id, 0);
      }
      uint64_t off = cursor[id]++; /* :329 every copy consumes a slot */
      double cost = nominal_cost(t, home, reader_is_gpu, reader_dev, id);
      if (best_id < 0 || cost < best_cost || (cost == best_cost && id < best_id)) {
        best_id = id;
        best_cost = cost;
        best_off = off;
      }
    }
    location_ids[f] = best_id;
    offsets[f] = best_off;
  }
  free(cursor);
  return 0;
}

/* page_transitions (placement.cpp:344-353) */
int qvo_page_transitions(const uint64_t* o, uint64_t count, uint64_t page, uint64_t* out) {
  if (count == 0) {
    *out = 0;
    return 0;
  }
  if (page == 0) return fail(QVB_ERR_VALIDATION, "page size must be > 0%.0llu%.0llu", 0, 0);
  uint64_t tr = 1;
  for (uint64_t i = 1; i < count; ++i)
    if (o[i] / page != o[i - 1] / page) ++tr;
  *out = tr;
  return 0;
}

typedef struct {
  int64_t loc;
  uint64_t off;
} pair_t;
static int cmp_pair(const void* a, const void* b) {
  const pair_t *x = (const pair_t*)a, *y = (const pair_t*)b;
  if (x->loc != y->loc) return x->loc < y->loc ? -1 : 1;
  return x->off < y->off ? -1 : (x->off > y->off ? 1 : 0);
}

/* plan_reads (placement.cpp:355-380): std::map groups by ascending location,
 * each group's offsets sorted ascending (duplicates kept). */
int qvo_plan_reads(const int64_t* location_ids, const uint64_t* offsets, uint64_t table_n,
                   const uint64_t* ids, uint64_t b, uint64_t page, int64_t* group_loc,
                   uint64_t* group_count, uint64_t* group_transitions, uint64_t* n_groups,
                   uint64_t* offsets_out) {
  if (page == 0) return fail(QVB_ERR_VALIDATION, "page size must be > 0%.0llu%.0llu", 0, 0);
  pair_t* p = (pair_t*)malloc((b ? b : 1) * sizeof(pair_t));
  for (uint64_t i = 0; i < b; ++i) {
    if (ids[i] >= table_n) {
      free(p);
      return fail(QVB_ERR_VALIDATION, "feature id %llu outside lookup table%.0llu", ids[i], 0);
    }
    p[i].loc = location_ids[ids[i]];
    p[i].off = offsets[ids[i]];
  }
  qsort(p, b, sizeof(pair_t), cmp_pair);
  uint64_t g = 0;
  for (uint64_t i = 0; i < b; ++i) {
    offsets_out[i] = p[i].off;
    if (i == 0 || p[i].loc != p[i - 1].loc) {
      group_loc[g] = p[i].loc;
      group_count[g] = 0;
      group_transitions[g] = 1;
      ++g;
    } else if (p[i].off / page != p[i - 1].off / page) {
      ++group_transitions[g - 1];
    }
    ++group_count[g - 1];
  }
  *n_groups = g;
  free(p);
  return 0;
}

/* ---- synthetic features / requests ----------------------- */
void qvo_features(uint64_t first, uint64_t count, uint32_t dim, float* x) {
  for (uint64_t f = 0; f < count; ++f)
    for (uint32_t k = 0; k < dim; ++k)
      x[f * dim + k] =
          (float)(qvo_splitmix64((first + f) * dim + k) >> 40) * 0x1.0p-24f;
}

void qvo_request_ids(uint64_t seed, uint64_t batch, uint64_t n, uint64_t* ids, uint64_t b) {
  uint64_t st = qvo_derive_state(seed, 0x5EEDULL, batch, 0);
  for (uint64_t i = 0; i < b; ++i) ids[i] = rng_below(&st, n);
}

typedef struct {
  const float* x;
  uint32_t dim;
  const uint64_t* ids;
  float* out;
  uint64_t lo, hi;
} gather_job;

static void* gather_worker(void* arg) {
  gather_job* j = (gather_job*)arg;
  size_t row = (size_t)j->dim * sizeof(float);
  for (uint64_t i = j->lo; i < j->hi; ++i)
    memcpy(j->out + i * j->dim, j->x + j->ids[i] * j->dim, row);
  return NULL;
}

int qvo_gather(const float* x, uint64_t n, uint32_t dim, const uint64_t* ids, uint64_t b,
               float* out, int threads) {
  for (uint64_t i = 0; i < b; ++i)
    if (ids[i] >= n) return fail(QVB_ERR_VALIDATION, "feature id %llu outside table of %llu", ids[i], n);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  gather_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (gather_job){x, dim, ids, out, b * t / threads, b * (t + 1) / threads};
    if (threads > 1) pthread_create(&th[t], NULL, gather_worker, &jobs[t]);
  }
  if (threads == 1) gather_worker(&jobs[0]);
  else
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  return 0;
}
