/*
 * alsncg_oracle.c -- CPU ORACLE (test infrastructure only; see alsncg_oracle.h).
 *
 * Plain-C restatement of the reference hot path.  Every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Compile with -ffp-contract=off and no -ffast-math so that every double
 * operation is rounded exactly where the reference rounds it (the reference is
 * built for baseline x86-64 and emits no FMA).
 */
#include "alsncg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ rng --
 * rng.hpp:26-45 wraps std::mt19937_64; restated from the published
 * Matsumoto-Nishimura MT19937-64 algorithm (same constants as the C++ std). */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->mti >= MT_N) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_N - MT_M; ++i) {
      x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
      r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
    }
    for (; i < MT_N - 1; ++i) {
      x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
      r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
    }
    x = (r->mt[MT_N - 1] & MT_UM) | (r->mt[0] & MT_LM);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* rng.hpp:33 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.cpp:25-34 */
uint64_t orc_rng_uniform_below(orc_rng* r, uint64_t n) {
  if (n == 0) return 0;
  const uint64_t mx = UINT64_MAX;
  const uint64_t limit = mx - mx % n;
  uint64_t v;
  do { v = orc_rng_next(r); } while (v >= limit);
  return v % n;
}

/* rng.cpp:36-49 (Box-Muller with cached spare) */
double orc_rng_normal(orc_rng* r) {
  if (r->has_spare) { r->has_spare = 0; return r->spare; }
  const double u1 = 1.0 - orc_rng_uniform(r);
  const double u2 = orc_rng_uniform(r);
  const double mag = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.141592653589793 * u2;
  r->spare = mag * sin(ang);
  r->has_spare = 1;
  return mag * cos(ang);
}

/* rng.cpp:51-58: first index whose cumulative weight exceeds u*total. */
int orc_sample_cumulative(const double* cum, int n, double u) {
  const double target = u * cum[n - 1];
  int lo = 0, hi = n; /* upper_bound */
  while (lo < hi) {
    int mid = lo + (hi - lo) / 2;
    if (target < cum[mid]) hi = mid; else lo = mid + 1;
  }
  if (lo == n) --lo;
  return lo;
}

/* ------------------------------------------------------- parallel_for --
 * parallel.cpp:25-55: tasks claimed from a shared counter by n_workers
 * threads (callers write disjoint outputs, so results never depend on it). */
typedef void (*orc_task_fn)(int task, void* ctx);
typedef struct { int n_tasks; int next; pthread_mutex_t mu; orc_task_fn fn; void* ctx; } pf_state;

static void* pf_worker(void* arg) {
  pf_state* s = (pf_state*)arg;
  for (;;) {
    pthread_mutex_lock(&s->mu);
    const int t = s->next++;
    pthread_mutex_unlock(&s->mu);
    if (t >= s->n_tasks) break;
    s->fn(t, s->ctx);
  }
  return NULL;
}

static void orc_parallel_for(int n_tasks, int n_workers, orc_task_fn fn, void* ctx) {
  if (n_tasks <= 0) return;
  if (n_workers > n_tasks) n_workers = n_tasks;
  if (n_workers <= 1) { for (int t = 0; t < n_tasks; ++t) fn(t, ctx); return; }
  pf_state s;
  s.n_tasks = n_tasks; s.next = 0; s.fn = fn; s.ctx = ctx;
  pthread_mutex_init(&s.mu, NULL);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)(n_workers - 1));
  for (int w = 1; w < n_workers; ++w) pthread_create(&th[w - 1], NULL, pf_worker, &s);
  pf_worker(&s);
  for (int w = 1; w < n_workers; ++w) pthread_join(th[w - 1], NULL);
  free(th);
  pthread_mutex_destroy(&s.mu);
}

/* ------------------------------------------------------------- ratings --
 * ratings.cpp:28-89: validate, sort by (user,item), reject duplicates, CSR
 * straight copy, CSC by a stable counting pass (users ascend within an item). */
typedef struct { int u, i; double v; } orc_triple;

static int cmp_triple(const void* a, const void* b) {
  const orc_triple* x = (const orc_triple*)a;
  const orc_triple* y = (const orc_triple*)b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->i != y->i) return x->i < y->i ? -1 : 1;
  return 0;
}

int orc_build(int n_u, int n_m, int64_t nnz, const int* users, const int* items,
              const double* values, int single_precision,
              int64_t* uptr, int* uidx, double* uval,
              int64_t* iptr, int* iidx, double* ival, int* dup_user, int* dup_item) {
  if (n_u < 0 || n_m < 0) return 1;                                   /* :30-31 */
  for (int64_t t = 0; t < nnz; ++t) {                                  /* :32-42 */
    if (users[t] < 0 || users[t] >= n_u || items[t] < 0 || items[t] >= n_m) return 1;
    if (!isfinite(values[t])) return 2;
  }
  orc_triple* tr = (orc_triple*)malloc(sizeof(orc_triple) * (size_t)(nnz > 0 ? nnz : 1));
  for (int64_t t = 0; t < nnz; ++t) { tr[t].u = users[t]; tr[t].i = items[t]; tr[t].v = values[t]; }
  qsort(tr, (size_t)nnz, sizeof(orc_triple), cmp_triple);              /* :43-46 */
  for (int64_t t = 1; t < nnz; ++t)                                    /* :47-51 */
    if (tr[t].u == tr[t - 1].u && tr[t].i == tr[t - 1].i) {
      if (dup_user) *dup_user = tr[t].u;
      if (dup_item) *dup_item = tr[t].i;
      free(tr);
      return 3;
    }
  memset(uptr, 0, sizeof(int64_t) * ((size_t)n_u + 1));                /* :59-66 */
  memset(iptr, 0, sizeof(int64_t) * ((size_t)n_m + 1));
  for (int64_t t = 0; t < nnz; ++t) { ++uptr[tr[t].u + 1]; ++iptr[tr[t].i + 1]; }
  for (int i = 0; i < n_u; ++i) uptr[i + 1] += uptr[i];
  for (int j = 0; j < n_m; ++j) iptr[j + 1] += iptr[j];
  int64_t* icur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_m > 0 ? n_m : 1));
  for (int j = 0; j < n_m; ++j) icur[j] = iptr[j];
  for (int64_t t = 0; t < nnz; ++t) {                                  /* :76-87 */
    double v = tr[t].v;
    if (single_precision) v = (double)(float)v;
    uidx[t] = tr[t].i;
    uval[t] = v;
    const int64_t ip = icur[tr[t].i]++;
    iidx[ip] = tr[t].u;
    ival[ip] = v;
  }
  free(icur);
  free(tr);
  return 0;
}

/* ---------------------------------------------------- workload generator --
 * BASELINE.json configs (SURVEY.md 8(d) "Synthetic generator"): the reference
 * has no generator for these workloads, so this restates the recipe SURVEY.md
 * 8(d) fixes, on the reference's own Rng draws (rng.cpp:36-58):
 *   rank-10 truth u*, m* ~ sd*normal(), sd = 10^-1/4 (variance 1/sqrt(10));
 *   per-user counts min + round(extra * exp(normal() - 1/2)) clamped to
 *   [min, cap = max(min, n_m/2)], then +-1 passes in user order to hit nnz;
 *   items ~ Zipf(1) via sample_cumulative (rng.cpp:51-58), repeats of the same
 *   user redrawn (as data.cpp:250-264);
 *   r = clamp(round(2*(3.5 + u*.m* + 0.5*normal()))/2, 0.5, 5.0), round half
 *   away from zero (support.hpp:104).
 * The product's alsncg_synth_generate must produce the same triples bit for
 * bit (tests/test_golden.py); the bench's reference arm builds its input from
 * this function so that it never loads the product library.
 * Returns 0, or 1 on bad dimensions / unreachable nnz. */
int orc_synth_generate(int n_u, int n_m, int64_t nnz, int min_per_user, uint64_t seed,
                       int* users, int* items, double* values) {
  enum { RANK = 10 };
  if (n_u <= 0 || n_m <= 0 || min_per_user < 1 || min_per_user > n_m) return 1;
  const int cap = min_per_user > n_m / 2 ? min_per_user : n_m / 2;
  if (nnz < (int64_t)min_per_user * n_u || nnz > (int64_t)cap * n_u) return 1;
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  const double sd = pow(10.0, -0.25);
  double* ut = (double*)malloc(sizeof(double) * (size_t)n_u * RANK);
  double* mt = (double*)malloc(sizeof(double) * (size_t)n_m * RANK);
  int* cnt = (int*)malloc(sizeof(int) * (size_t)n_u);
  double* cum = (double*)malloc(sizeof(double) * (size_t)n_m);
  int* stamp = (int*)malloc(sizeof(int) * (size_t)n_m);
  for (int64_t k = 0; k < (int64_t)n_u * RANK; ++k) ut[k] = sd * orc_rng_normal(&rng);
  for (int64_t k = 0; k < (int64_t)n_m * RANK; ++k) mt[k] = sd * orc_rng_normal(&rng);
  const double extra = (double)nnz / n_u - min_per_user;
  for (int i = 0; i < n_u; ++i) {
    cnt[i] = min_per_user;
    if (extra > 0.0) {
      double c = min_per_user + round(extra * exp(orc_rng_normal(&rng) - 0.5));
      if (c < min_per_user) c = min_per_user;
      if (c > cap) c = cap;
      cnt[i] = (int)c;
    }
  }
  int64_t total = 0;
  for (int i = 0; i < n_u; ++i) total += cnt[i];
  int rc = 0;
  while (total != nnz) {
    int moved = 0;
    for (int i = 0; i < n_u && total != nnz; ++i) {
      if (total < nnz && cnt[i] < cap) { ++cnt[i]; ++total; moved = 1; }
      else if (total > nnz && cnt[i] > min_per_user) { --cnt[i]; --total; moved = 1; }
    }
    if (!moved) { rc = 1; break; }
  }
  if (rc == 0) {
    double run = 0.0;
    for (int j = 0; j < n_m; ++j) { run += 1.0 / (double)(j + 1); cum[j] = run; stamp[j] = -1; }
    int64_t pos = 0;
    for (int i = 0; i < n_u; ++i) {
      const double* u = ut + (size_t)i * RANK;
      for (int drawn = 0; drawn < cnt[i];) {
        const int j = orc_sample_cumulative(cum, n_m, orc_rng_uniform(&rng));
        if (stamp[j] == i) continue;
        stamp[j] = i;
        ++drawn;
        const double* m = mt + (size_t)j * RANK;
        double score = 0.0;
        for (int k = 0; k < RANK; ++k) score += u[k] * m[k];
        const double eps = 0.5 * orc_rng_normal(&rng);
        double r = round(2.0 * (3.5 + score + eps)) / 2.0;
        if (r < 0.5) r = 0.5;
        if (r > 5.0) r = 5.0;
        users[pos] = i;
        items[pos] = j;
        values[pos] = r;
        ++pos;
      }
    }
  }
  free(ut); free(mt); free(cnt); free(cum); free(stamp);
  return rc;
}

/* ------------------------------------------------------------- factors -- */
/* factors.cpp:24-32: items first, then users, U[0,1) * 1/sqrt(n_f). */
void orc_random_init(int n_f, int n_u, int n_m, uint64_t seed, double* user, double* item) {
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  const double scale = 1.0 / sqrt((double)n_f);
  for (int64_t k = 0; k < (int64_t)n_f * n_m; ++k) item[k] = orc_rng_uniform(&rng) * scale;
  for (int64_t k = 0; k < (int64_t)n_f * n_u; ++k) user[k] = orc_rng_uniform(&rng) * scale;
}

/* factors.cpp:80-93 */
void orc_axpby(int64_t nu, int64_t nm, double a, const double* xu, const double* xm,
               double b, const double* yu, const double* ym, double* ou, double* om) {
  for (int64_t k = 0; k < nu; ++k) ou[k] = a * xu[k] + b * yu[k];
  for (int64_t k = 0; k < nm; ++k) om[k] = a * xm[k] + b * ym[k];
}

/* factors.cpp:95-103: sequential, user part then item part. */
double orc_dot(int64_t nu, int64_t nm, const double* xu, const double* xm,
               const double* yu, const double* ym) {
  double acc = 0.0;
  for (int64_t k = 0; k < nu; ++k) acc += xu[k] * yu[k];
  for (int64_t k = 0; k < nm; ++k) acc += xm[k] * ym[k];
  return acc;
}

static inline double dot_nf(const double* a, const double* b, int n_f) { /* ncg.cpp:29-33 */
  double acc = 0.0;
  for (int k = 0; k < n_f; ++k) acc += a[k] * b[k];
  return acc;
}

/* ---------------------------------------------------------------- loss --
 * ncg.cpp:43-68: residuals user-major in sorted item order, then the two
 * weighted regularisation sums; returns early when lambda == 0. */
double orc_loss(const orc_ratings* r, int n_f, const double* xu, const double* xm, double lambda) {
  double sq = 0.0;
  for (int i = 0; i < r->n_u; ++i) {
    const double* u = xu + (size_t)i * n_f;
    for (int64_t t = r->uptr[i]; t < r->uptr[i + 1]; ++t) {
      const double e = r->uval[t] - dot_nf(u, xm + (size_t)r->uidx[t] * n_f, n_f);
      sq += e * e;
    }
  }
  if (lambda == 0.0) return sq;
  double reg_u = 0.0;
  for (int i = 0; i < r->n_u; ++i) {
    const double* u = xu + (size_t)i * n_f;
    reg_u += (int)(r->uptr[i + 1] - r->uptr[i]) * dot_nf(u, u, n_f);
  }
  double reg_m = 0.0;
  for (int j = 0; j < r->n_m; ++j) {
    const double* m = xm + (size_t)j * n_f;
    reg_m += (int)(r->iptr[j + 1] - r->iptr[j]) * dot_nf(m, m, n_f);
  }
  return sq + lambda * (reg_u + reg_m);
}

/* ------------------------------------------------------------ gradient --
 * ncg.cpp:70-116: user-major CSR pass then item-major CSC pass; each block
 * starts at 2*lambda*n*x and accumulates 2(x.y - r) y rating by rating. */
typedef struct {
  const orc_ratings* r; int n_f; const double* xu; const double* xm; double lambda;
  double* gu; double* gm; int chunks;
} grad_ctx;

static void grad_user_task(int c, void* p) {
  grad_ctx* g = (grad_ctx*)p;
  const int n_u = g->r->n_u, n_f = g->n_f;
  const int lo = (int)((int64_t)c * n_u / g->chunks);
  const int hi = (int)((int64_t)(c + 1) * n_u / g->chunks);
  for (int i = lo; i < hi; ++i) {
    const double* u = g->xu + (size_t)i * n_f;
    double* gu = g->gu + (size_t)i * n_f;
    const double w = 2.0 * g->lambda * (int)(g->r->uptr[i + 1] - g->r->uptr[i]);
    for (int k = 0; k < n_f; ++k) gu[k] = w * u[k];
    for (int64_t t = g->r->uptr[i]; t < g->r->uptr[i + 1]; ++t) {
      const double* m = g->xm + (size_t)g->r->uidx[t] * n_f;
      const double e2 = 2.0 * (dot_nf(u, m, n_f) - g->r->uval[t]);
      for (int k = 0; k < n_f; ++k) gu[k] += e2 * m[k];
    }
  }
}

static void grad_item_task(int c, void* p) {
  grad_ctx* g = (grad_ctx*)p;
  const int n_m = g->r->n_m, n_f = g->n_f;
  const int lo = (int)((int64_t)c * n_m / g->chunks);
  const int hi = (int)((int64_t)(c + 1) * n_m / g->chunks);
  for (int j = lo; j < hi; ++j) {
    const double* m = g->xm + (size_t)j * n_f;
    double* gm = g->gm + (size_t)j * n_f;
    const double w = 2.0 * g->lambda * (int)(g->r->iptr[j + 1] - g->r->iptr[j]);
    for (int k = 0; k < n_f; ++k) gm[k] = w * m[k];
    for (int64_t t = g->r->iptr[j]; t < g->r->iptr[j + 1]; ++t) {
      const double* u = g->xu + (size_t)g->r->iidx[t] * n_f;
      const double e2 = 2.0 * (dot_nf(u, m, n_f) - g->r->ival[t]);
      for (int k = 0; k < n_f; ++k) gm[k] += e2 * u[k];
    }
  }
}

static int imax(int a, int b) { return a > b ? a : b; }
static int imin(int a, int b) { return a < b ? a : b; }

void orc_gradient(const orc_ratings* r, int n_f, const double* xu, const double* xm,
                  double lambda, int n_workers, double* gu, double* gm) {
  if (n_workers < 1) n_workers = 1;
  grad_ctx g = {r, n_f, xu, xm, lambda, gu, gm, 0};
  g.chunks = imax(1, imin(r->n_u, n_workers * 4));                      /* :78 */
  orc_parallel_for(g.chunks, n_workers, grad_user_task, &g);
  g.chunks = imax(1, imin(r->n_m, n_workers * 4));                      /* :97 */
  orc_parallel_for(g.chunks, n_workers, grad_item_task, &g);
}

/* ncg.cpp:118-132 */
double orc_beta_bar(int64_t nu, int64_t nm, const double* gnu, const double* gnm,
                    const double* gpu, const double* gpm, const double* bnu,
                    const double* bnm, const double* bpu, const double* bpm) {
  const double den = orc_dot(nu, nm, bpu, bpm, gpu, gpm);
  if (fabs(den) < 1e-30) return 0.0;
  double num = 0.0;
  for (int64_t k = 0; k < nu; ++k) num += bnu[k] * (gnu[k] - gpu[k]);
  for (int64_t k = 0; k < nm; ++k) num += bnm[k] * (gnm[k] - gpm[k]);
  const double beta = num / den;
  return isfinite(beta) ? beta : 0.0;
}

/* ------------------------------------------------------------- quartic --
 * linesearch.cpp:26-111: Kahan5 per chunk, chunks merged in chunk order
 * using the sums only. */
typedef struct { double sum[5]; double comp[5]; } kahan5;

static inline void k5_add(kahan5* k, int n, double v) {               /* :30-35 */
  const double y = v - k->comp[n];
  const double t = k->sum[n] + y;
  k->comp[n] = (t - k->sum[n]) - y;
  k->sum[n] = t;
}

typedef struct {
  const orc_ratings* r; int n_f; const double *xu, *xm, *pu, *pm; double lambda;
  int n_chunks; kahan5* partial;
} quart_ctx;

static void quart_task(int c, void* p) {
  quart_ctx* q = (quart_ctx*)p;
  const orc_ratings* r = q->r;
  const int n_f = q->n_f, n_u = r->n_u, n_m = r->n_m;
  kahan5 acc;
  memset(&acc, 0, sizeof acc);
  const int ulo = (int)((int64_t)c * n_u / q->n_chunks);
  const int uhi = (int)((int64_t)(c + 1) * n_u / q->n_chunks);
  for (int i = ulo; i < uhi; ++i) {
    const double* xu = q->xu + (size_t)i * n_f;
    const double* pu = q->pu + (size_t)i * n_f;
    const int count = (int)(r->uptr[i + 1] - r->uptr[i]);
    if (q->lambda > 0.0 && count > 0) {                               /* :68-73 */
      const double w = q->lambda * count;
      k5_add(&acc, 0, w * dot_nf(xu, xu, n_f));
      k5_add(&acc, 1, 2.0 * w * dot_nf(xu, pu, n_f));
      k5_add(&acc, 2, w * dot_nf(pu, pu, n_f));
    }
    for (int64_t t = r->uptr[i]; t < r->uptr[i + 1]; ++t) {           /* :76-88 */
      const double* xm = q->xm + (size_t)r->uidx[t] * n_f;
      const double* pm = q->pm + (size_t)r->uidx[t] * n_f;
      const double a = r->uval[t] - dot_nf(xu, xm, n_f);
      const double b = dot_nf(xu, pm, n_f) + dot_nf(pu, xm, n_f);
      const double d = dot_nf(pu, pm, n_f);
      k5_add(&acc, 0, a * a);
      k5_add(&acc, 1, -2.0 * a * b);
      k5_add(&acc, 2, b * b - 2.0 * a * d);
      k5_add(&acc, 3, 2.0 * b * d);
      k5_add(&acc, 4, d * d);
    }
  }
  if (q->lambda > 0.0) {                                              /* :90-103 */
    const int mlo = (int)((int64_t)c * n_m / q->n_chunks);
    const int mhi = (int)((int64_t)(c + 1) * n_m / q->n_chunks);
    for (int j = mlo; j < mhi; ++j) {
      const int count = (int)(r->iptr[j + 1] - r->iptr[j]);
      if (count == 0) continue;
      const double* xm = q->xm + (size_t)j * n_f;
      const double* pm = q->pm + (size_t)j * n_f;
      const double w = q->lambda * count;
      k5_add(&acc, 0, w * dot_nf(xm, xm, n_f));
      k5_add(&acc, 1, 2.0 * w * dot_nf(xm, pm, n_f));
      k5_add(&acc, 2, w * dot_nf(pm, pm, n_f));
    }
  }
  q->partial[c] = acc;
}

void orc_quartic(const orc_ratings* r, int n_f, const double* xu, const double* xm,
                 const double* pu, const double* pm, double lambda, int n_chunks,
                 int n_workers, double c[5]) {
  if (n_chunks < 1) n_chunks = 1;
  quart_ctx q = {r, n_f, xu, xm, pu, pm, lambda, n_chunks, NULL};
  q.partial = (kahan5*)calloc((size_t)n_chunks, sizeof(kahan5));
  orc_parallel_for(n_chunks, n_workers < 1 ? 1 : n_workers, quart_task, &q);
  for (int n = 0; n < 5; ++n) c[n] = 0.0;
  for (int ch = 0; ch < n_chunks; ++ch)                               /* :107-110 */
    for (int n = 0; n < 5; ++n) c[n] += q.partial[ch].sum[n];
  free(q.partial);
}

/* config.hpp:79-81 Horner */
static inline double quartic_eval(const double c[5], double a) {
  return (((c[4] * a + c[3]) * a + c[2]) * a + c[1]) * a + c[0];
}

/* linesearch.cpp:115-131 */
int orc_backtracking(const double c[5], double slope, double alpha0, double cc, double tau,
                     int max_backtracks, double* alpha_out, int* backtracks) {
  if (!(slope < 0.0)) { *alpha_out = 0.0; *backtracks = 0; return 1; }
  const double q0 = quartic_eval(c, 0.0);
  double alpha = alpha0;
  for (int k = 0; k <= max_backtracks; ++k) {
    if (quartic_eval(c, alpha) - q0 <= alpha * cc * slope) {
      *alpha_out = alpha; *backtracks = k; return 0;
    }
    alpha *= tau;
  }
  *alpha_out = 0.0; *backtracks = max_backtracks;
  return 2;
}

/* ------------------------------------------------------------------ als --
 * als.cpp:40-83 restated without Eigen.  Gram/rhs loop and shift follow the
 * reference exactly; Eigen::LLT becomes an unblocked lower Cholesky that
 * fails when a pivot is <= 0 (Eigen's llt_inplace test); the COD least-norm
 * path becomes a pseudo-inverse solve from a cyclic Jacobi eigendecomposition
 * plus the reference's single refinement step (als.cpp:77-79). */
static int chol_solve(const double* a, int n, const double* v, double* u, double* l) {
  for (int j = 0; j < n; ++j) {
    double d = a[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= l[(size_t)j * n + k] * l[(size_t)j * n + k];
    if (d <= 0.0) return 0;
    const double ljj = sqrt(d);
    l[(size_t)j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = a[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= l[(size_t)i * n + k] * l[(size_t)j * n + k];
      l[(size_t)i * n + j] = s / ljj;
    }
  }
  for (int i = 0; i < n; ++i) {             /* L y = v */
    double s = v[i];
    for (int k = 0; k < i; ++k) s -= l[(size_t)i * n + k] * u[k];
    u[i] = s / l[(size_t)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {        /* L^T u = y */
    double s = u[i];
    for (int k = i + 1; k < n; ++k) s -= l[(size_t)k * n + i] * u[k];
    u[i] = s / l[(size_t)i * n + i];
  }
  return 1;
}

/* Symmetric eigendecomposition (cyclic Jacobi) -> pseudo-inverse apply. */
static void pinv_apply(const double* a, int n, const double* v, double* out) {
  double* w = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* q = (double*)malloc(sizeof(double) * (size_t)n * n);
  memcpy(w, a, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n * n; ++i) q[i] = 0.0;
  for (int i = 0; i < n; ++i) q[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double x = w[(size_t)i * n + j] * w[(size_t)i * n + j];
        tot += x;
        if (i != j) off += x;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int r = p + 1; r < n; ++r) {
        const double apr = w[(size_t)p * n + r];
        if (apr == 0.0) continue;
        const double app = w[(size_t)p * n + p], arr = w[(size_t)r * n + r];
        const double theta = (arr - app) / (2.0 * apr);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {        /* columns p, r */
          const double wkp = w[(size_t)k * n + p], wkr = w[(size_t)k * n + r];
          w[(size_t)k * n + p] = c * wkp - s * wkr;
          w[(size_t)k * n + r] = s * wkp + c * wkr;
        }
        for (int k = 0; k < n; ++k) {        /* rows p, r */
          const double wpk = w[(size_t)p * n + k], wrk = w[(size_t)r * n + k];
          w[(size_t)p * n + k] = c * wpk - s * wrk;
          w[(size_t)r * n + k] = s * wpk + c * wrk;
        }
        for (int k = 0; k < n; ++k) {
          const double qkp = q[(size_t)k * n + p], qkr = q[(size_t)k * n + r];
          q[(size_t)k * n + p] = c * qkp - s * qkr;
          q[(size_t)k * n + r] = s * qkp + c * qkr;
        }
      }
  }
  double emax = 0.0;
  for (int i = 0; i < n; ++i) emax = fmax(emax, fabs(w[(size_t)i * n + i]));
  const double thresh = emax * n * 2.220446049250313e-16;
  for (int i = 0; i < n; ++i) out[i] = 0.0;
  for (int e = 0; e < n; ++e) {
    const double lam = w[(size_t)e * n + e];
    if (!(fabs(lam) > thresh)) continue;
    double proj = 0.0;
    for (int k = 0; k < n; ++k) proj += q[(size_t)k * n + e] * v[k];
    proj /= lam;
    for (int k = 0; k < n; ++k) out[k] += proj * q[(size_t)k * n + e];
  }
  free(w);
  free(q);
}

void orc_solve_normal_column(const int* idx, const double* vals, int count,
                             const double* const* cols, int n_f, double lambda,
                             double* out, int* fallback_columns) {
  const size_t nn = (size_t)n_f * n_f;
  double* a = (double*)calloc(nn * 2 + 4 * (size_t)n_f, sizeof(double));
  double* l = a + nn;
  double* v = l + nn;
  double* u = v + n_f;
  double* res = u + n_f;
  double* du = res + n_f;
  for (int t = 0; t < count; ++t) {                                   /* :49-57 */
    const double* m = cols[idx[t]];
    const double r = vals[t];
    for (int i = 0; i < n_f; ++i) {
      const double ma = m[i];
      v[i] += r * ma;
      for (int b = 0; b <= i; ++b) a[(size_t)i * n_f + b] += ma * m[b];
    }
  }
  const double shift = lambda * count;                                /* :58-61 */
  for (int d = 0; d < n_f; ++d) a[(size_t)d * n_f + d] += shift;
  for (int i = 0; i < n_f; ++i)
    for (int b = i + 1; b < n_f; ++b) a[(size_t)i * n_f + b] = a[(size_t)b * n_f + i];
  int solved = 0;
  if (shift > 0.0) solved = chol_solve(a, n_f, v, u, l);              /* :63-70 */
  if (!solved) {                                                      /* :71-81 */
    pinv_apply(a, n_f, v, u);
    for (int i = 0; i < n_f; ++i) {
      double s = 0.0;
      for (int k = 0; k < n_f; ++k) s += a[(size_t)i * n_f + k] * u[k];
      res[i] = v[i] - s;
    }
    pinv_apply(a, n_f, res, du);
    for (int i = 0; i < n_f; ++i) u[i] += du[i];
    ++*fallback_columns;
  }
  for (int k = 0; k < n_f; ++k) out[k] = u[k];
  free(a);
}

typedef struct {
  const orc_ratings* r; int n_f; const double* src; double lambda; double* out;
  int users; int n_tasks; int* fallback;
} upd_ctx;

static void upd_task(int task, void* p) {
  upd_ctx* c = (upd_ctx*)p;
  const orc_ratings* r = c->r;
  const int n_dest = c->users ? r->n_u : r->n_m;
  const int n_src = c->users ? r->n_m : r->n_u;
  const int64_t* ptr = c->users ? r->uptr : r->iptr;
  const int* idx = c->users ? r->uidx : r->iidx;
  const double* val = c->users ? r->uval : r->ival;
  const double** cols = (const double**)malloc(sizeof(double*) * (size_t)(n_src > 0 ? n_src : 1));
  for (int j = 0; j < n_src; ++j) cols[j] = c->src + (size_t)j * c->n_f;
  int fb = 0;
  for (int col = task; col < n_dest; col += c->n_tasks) {             /* als.cpp:93-99 */
    const int64_t b = ptr[col], e = ptr[col + 1];
    if (e == b) continue;
    orc_solve_normal_column(idx + b, val + b, (int)(e - b), cols, c->n_f, c->lambda,
                            c->out + (size_t)col * c->n_f, &fb);
  }
  c->fallback[task] = fb;
  free(cols);
}

static void orc_update(const orc_ratings* r, int n_f, const double* src, double lambda,
                       int n_workers, double* out, int* fallback_columns, int users) {
  const int n_dest = users ? r->n_u : r->n_m;
  memset(out, 0, sizeof(double) * (size_t)n_f * (size_t)n_dest);
  if (n_workers < 1) n_workers = 1;
  upd_ctx c = {r, n_f, src, lambda, out, users, n_workers, NULL};
  c.fallback = (int*)calloc((size_t)n_workers, sizeof(int));
  orc_parallel_for(n_workers, n_workers, upd_task, &c);
  int fb = 0;
  for (int w = 0; w < n_workers; ++w) fb += c.fallback[w];
  free(c.fallback);
  if (fallback_columns) *fallback_columns += fb;
}

/* als.cpp:85-102 */
void orc_update_users(const orc_ratings* r, int n_f, const double* item_data, double lambda,
                      int n_workers, double* out, int* fallback_columns) {
  orc_update(r, n_f, item_data, lambda, n_workers, out, fallback_columns, 1);
}
/* als.cpp:104-121 */
void orc_update_items(const orc_ratings* r, int n_f, const double* user_data, double lambda,
                      int n_workers, double* out, int* fallback_columns) {
  orc_update(r, n_f, user_data, lambda, n_workers, out, fallback_columns, 0);
}

/* parallel.cpp:69-111 + RoutingTable::total_columns (:62-66) */
void orc_routing_totals(const orc_ratings* r, int n_blocks, int64_t* tu_total, int64_t* tm_total) {
  char* seen = (char*)malloc((size_t)(n_blocks > 0 ? n_blocks : 1));
  int64_t tu = 0, tm = 0;
  for (int i = 0; i < r->n_u; ++i) {
    memset(seen, 0, (size_t)n_blocks);
    for (int64_t t = r->uptr[i]; t < r->uptr[i + 1]; ++t) {
      const int d = r->uidx[t] % n_blocks;
      if (!seen[d]) { seen[d] = 1; ++tu; }
    }
  }
  for (int j = 0; j < r->n_m; ++j) {
    memset(seen, 0, (size_t)n_blocks);
    for (int64_t t = r->iptr[j]; t < r->iptr[j + 1]; ++t) {
      const int d = r->iidx[t] % n_blocks;
      if (!seen[d]) { seen[d] = 1; ++tm; }
    }
  }
  free(seen);
  *tu_total = tu;
  *tm_total = tm;
}

/* ------------------------------------------------------------- drivers -- */
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct { double total, t0; int running; } stopwatch; /* src/stopwatch.hpp:23-45 */
static void sw_start(stopwatch* w) { if (!w->running) { w->t0 = now_s(); w->running = 1; } }
static void sw_stop(stopwatch* w) { if (w->running) { w->total += now_s() - w->t0; w->running = 0; } }
static double sw_seconds(const stopwatch* w) { return w->running ? w->total + now_s() - w->t0 : w->total; }

static int validate(const orc_config* c) {                            /* config.cpp:21-34 */
  if (c->lambda < 0.0 || c->n_f < 1 || c->max_iters < 0 || c->alpha0 <= 0.0) return -1;
  if (!(c->armijo_c > 0.0 && c->armijo_c < 1.0) || !(c->tau > 0.0 && c->tau < 1.0)) return -1;
  if (c->max_backtracks < 0 || c->n_blocks < 0 || c->n_workers < 1) return -1;
  if (c->trace_every < 1 || c->snapshot_every < 0) return -1;
  return 0;
}

static int resolved_blocks(const orc_config* c) {                     /* config.hpp:48 */
  return c->n_blocks > 0 ? c->n_blocks : (c->n_workers > 0 ? c->n_workers : 1);
}

static void push_trace(orc_trace_rec* trace, int cap, int* len, orc_trace_rec rec) {
  if (*len < cap) trace[*len] = rec;
  ++*len;
}

/* ncg.cpp:138-307 */
int orc_ncg_solve(const orc_ratings* r, const orc_config* cfg, double* model_u,
                  double* model_m, orc_trace_rec* trace, int trace_cap, int* trace_len,
                  orc_result* res) {
  if (validate(cfg)) return -1;
  const int n_f = cfg->n_f, n_u = r->n_u, n_m = r->n_m;
  const int n_blocks = resolved_blocks(cfg);
  int64_t tu_cols, tm_cols;
  orc_routing_totals(r, n_blocks, &tu_cols, &tm_cols);
  const int64_t sweep_columns = tm_cols + tu_cols;
  const int64_t gradient_columns = sweep_columns;
  const int64_t quartic_columns = 2 * tm_cols;
  const int64_t nu = (int64_t)n_f * n_u, nm = (int64_t)n_f * n_m, N = nu + nm;
  const double lambda = cfg->lambda;
  const int nw = cfg->n_workers;
  memset(res, 0, sizeof *res);
  *trace_len = 0;

  double* buf = (double*)calloc((size_t)N * 10, sizeof(double));
  double *x = buf, *g = buf + N, *gbar = buf + 2 * N, *p = buf + 3 * N, *px = buf + 4 * N;
  double *xn = buf + 5 * N, *gn = buf + 6 * N, *gbn = buf + 7 * N, *pn = buf + 8 * N, *pxn = buf + 9 * N;
  orc_random_init(n_f, n_u, n_m, cfg->seed, x, x + nu);               /* :154-155 */

  stopwatch watch = {0.0, 0.0, 0};
#define INSTRUMENTED(stmt) do { if (cfg->paper_timing) sw_stop(&watch); stmt; if (cfg->paper_timing) sw_start(&watch); } while (0)
#define APPLY_ALS(v, outp) do { \
    orc_update_users(r, n_f, (v) + nu, lambda, nw, (outp), &res->fallback_columns); \
    orc_update_items(r, n_f, (outp), lambda, nw, (outp) + nu, &res->fallback_columns); } while (0)

  orc_gradient(r, n_f, x, x + nu, lambda, nw, g, g + nu);             /* :178-180 */
  double grad_norm = sqrt(orc_dot(nu, nm, g, g + nu, g, g + nu)) / (double)N;
  {
    orc_trace_rec rec = {0, orc_loss(r, n_f, x, x + nu, lambda), grad_norm, 0.0, 0, 0, 0};
    push_trace(trace, trace_cap, trace_len, rec);
  }
  int converged = cfg->tol > 0.0 && grad_norm < cfg->tol;
  int k = 0;
  if (!converged && cfg->max_iters > 0) {
    sw_start(&watch);
    APPLY_ALS(x, px);                                                 /* :187 */
    orc_axpby(nu, nm, 1.0, x, x + nu, -1.0, px, px + nu, gbar, gbar + nu);
    orc_axpby(nu, nm, -1.0, gbar, gbar + nu, 0.0, gbar, gbar + nu, p, p + nu);
    int p_is_neg_gbar = 1, restart_pending = 0;
    int64_t step_columns = sweep_columns + gradient_columns;
    while (!converged && k < cfg->max_iters) {
      int restarted = restart_pending;
      restart_pending = 0;
      double slope = orc_dot(nu, nm, g, g + nu, p, p + nu);           /* :197 */
      if (slope >= 0.0 && !p_is_neg_gbar) {                           /* :198-205 */
        orc_axpby(nu, nm, -1.0, gbar, gbar + nu, 0.0, gbar, gbar + nu, p, p + nu);
        p_is_neg_gbar = 1;
        restarted = 1;
        slope = orc_dot(nu, nm, g, g + nu, p, p + nu);
      }
      int pure = 0, backtracks = 0;
      double alpha = 0.0;
      if (cfg->has_fixed_alpha) {
        alpha = cfg->fixed_alpha;
      } else if (slope >= 0.0) {
        pure = 1;
      } else {
        double q[5];
        orc_quartic(r, n_f, x, x + nu, p, p + nu, lambda, n_blocks, nw, q);
        step_columns += quartic_columns;
        double a_out; int bt;
        const int st = orc_backtracking(q, slope, cfg->alpha0, cfg->armijo_c, cfg->tau,
                                        cfg->max_backtracks, &a_out, &bt);
        if (st == 0) { alpha = a_out; backtracks = bt; } else { pure = 1; }
      }
      if (pure) {                                                     /* :228-241 */
        memcpy(xn, px, sizeof(double) * (size_t)N);
        restarted = 1;
        ++res->fallback_steps;
      } else if (p_is_neg_gbar && alpha == 1.0) {
        memcpy(xn, px, sizeof(double) * (size_t)N);
      } else {
        orc_axpby(nu, nm, 1.0, x, x + nu, alpha, p, p + nu, xn, xn + nu);
      }
      orc_gradient(r, n_f, xn, xn + nu, lambda, nw, gn, gn + nu);     /* :253 */
      step_columns += gradient_columns;
      APPLY_ALS(xn, pxn);                                             /* :255 */
      step_columns += sweep_columns;
      orc_axpby(nu, nm, 1.0, xn, xn + nu, -1.0, pxn, pxn + nu, gbn, gbn + nu);
      double beta = 0.0;
      if (!cfg->force_beta_zero && !pure)
        beta = orc_beta_bar(nu, nm, gn, gn + nu, g, g + nu, gbn, gbn + nu, gbar, gbar + nu);
      if (beta == 0.0) {                                              /* :263-275 */
        orc_axpby(nu, nm, -1.0, gbn, gbn + nu, 0.0, gbn, gbn + nu, pn, pn + nu);
        p_is_neg_gbar = 1;
      } else {
        orc_axpby(nu, nm, -1.0, gbn, gbn + nu, beta, p, p + nu, pn, pn + nu);
        p_is_neg_gbar = 0;
        if (orc_dot(nu, nm, gn, gn + nu, pn, pn + nu) >= 0.0) {
          orc_axpby(nu, nm, -1.0, gbn, gbn + nu, 0.0, gbn, gbn + nu, pn, pn + nu);
          p_is_neg_gbar = 1;
          restart_pending = 1;
        }
      }
      double* t;
      t = x; x = xn; xn = t;
      t = g; g = gn; gn = t;
      t = gbar; gbar = gbn; gbn = t;
      t = px; px = pxn; pxn = t;
      t = p; p = pn; pn = t;
      ++k;
      if (restarted) ++res->restarts;
      grad_norm = sqrt(orc_dot(nu, nm, g, g + nu, g, g + nu)) / (double)N;
      converged = cfg->tol > 0.0 && grad_norm < cfg->tol;
      const int record = k % cfg->trace_every == 0 || converged || k == cfg->max_iters;
      if (record) {
        double lv = 0.0;
        INSTRUMENTED(lv = orc_loss(r, n_f, x, x + nu, lambda));
        orc_trace_rec rec = {k, lv, grad_norm, sw_seconds(&watch), backtracks, step_columns, restarted};
        push_trace(trace, trace_cap, trace_len, rec);
        step_columns = 0;
      }
    }
    sw_stop(&watch);
  }
  memcpy(model_u, x, sizeof(double) * (size_t)nu);
  memcpy(model_m, x + nu, sizeof(double) * (size_t)nm);
  res->converged = converged;
  res->iterations = k;
  res->final_grad_norm = grad_norm;
  res->final_loss = orc_loss(r, n_f, x, x + nu, lambda);
  free(buf);
  return 0;
#undef APPLY_ALS
#undef INSTRUMENTED
}

/* als.cpp:130-195 */
int orc_als_solve(const orc_ratings* r, const orc_config* cfg, double* model_u,
                  double* model_m, orc_trace_rec* trace, int trace_cap, int* trace_len,
                  orc_result* res) {
  if (validate(cfg)) return -1;
  const int n_f = cfg->n_f, n_u = r->n_u, n_m = r->n_m;
  const int n_blocks = resolved_blocks(cfg);
  int64_t tu_cols, tm_cols;
  orc_routing_totals(r, n_blocks, &tu_cols, &tm_cols);
  const int64_t sweep_columns = tm_cols + tu_cols;
  const int64_t nu = (int64_t)n_f * n_u, nm = (int64_t)n_f * n_m, N = nu + nm;
  const double lambda = cfg->lambda;
  const int nw = cfg->n_workers;
  memset(res, 0, sizeof *res);
  *trace_len = 0;
  double* x = (double*)calloc((size_t)N * 3, sizeof(double));
  double* g = x + N;
  double* tmp = g + N;
  orc_random_init(n_f, n_u, n_m, cfg->seed, x, x + nu);
  stopwatch watch = {0.0, 0.0, 0};
  orc_gradient(r, n_f, x, x + nu, lambda, nw, g, g + nu);
  double grad_norm = sqrt(orc_dot(nu, nm, g, g + nu, g, g + nu)) / (double)N;
  {
    orc_trace_rec rec = {0, orc_loss(r, n_f, x, x + nu, lambda), grad_norm, 0.0, 0, 0, 0};
    push_trace(trace, trace_cap, trace_len, rec);
  }
  int converged = cfg->tol > 0.0 && grad_norm < cfg->tol;
  int k = 0;
  sw_start(&watch);
  while (!converged && k < cfg->max_iters) {
    orc_update_users(r, n_f, x + nu, lambda, nw, tmp, &res->fallback_columns);
    memcpy(x, tmp, sizeof(double) * (size_t)nu);
    orc_update_items(r, n_f, x, lambda, nw, tmp, &res->fallback_columns);
    memcpy(x + nu, tmp, sizeof(double) * (size_t)nm);
    ++k;
    if (cfg->paper_timing) sw_stop(&watch);
    orc_gradient(r, n_f, x, x + nu, lambda, nw, g, g + nu);
    grad_norm = sqrt(orc_dot(nu, nm, g, g + nu, g, g + nu)) / (double)N;
    if (cfg->paper_timing) sw_start(&watch);
    converged = cfg->tol > 0.0 && grad_norm < cfg->tol;
    const int record = k % cfg->trace_every == 0 || converged || k == cfg->max_iters;
    if (record) {
      if (cfg->paper_timing) sw_stop(&watch);
      const double lv = orc_loss(r, n_f, x, x + nu, lambda);
      if (cfg->paper_timing) sw_start(&watch);
      orc_trace_rec rec = {k, lv, grad_norm, sw_seconds(&watch), 0, sweep_columns, 0};
      push_trace(trace, trace_cap, trace_len, rec);
    }
  }
  sw_stop(&watch);
  memcpy(model_u, x, sizeof(double) * (size_t)nu);
  memcpy(model_m, x + nu, sizeof(double) * (size_t)nm);
  res->converged = converged;
  res->iterations = k;
  res->final_grad_norm = grad_norm;
  res->final_loss = orc_loss(r, n_f, x, x + nu, lambda);
  free(x);
  return 0;
}
