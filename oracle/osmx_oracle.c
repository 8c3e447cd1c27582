/*
 * osmx_oracle.c -- CPU restatement of the reference `osmx` algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_1805_02867_b200/) links, loads or calls this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it,
 * and only as the checker / the timed CPU baseline.
 *
 * Parity pinned: tests/test_oracle.py checks every function here bit-exactly
 * against the reference itself (oracle/_ref/libosmx_ref.so, compiled from
 * /root/reference/proj/src by oracle/Makefile) and against the frozen
 * constants of /root/reference/proj/tests/test_support.hpp:47-56, via the
 * committed fixtures in tests/golden/.
 *
 * The arithmetic follows the reference operation by operation so that the
 * results are bit-identical on the same libm:
 *   - m is a float max, d is a double sum       kernels.hpp:17-20
 *   - exp arguments / widths exactly as the reference writes them.
 * Status codes instead of exceptions (error.hpp:8-25):
 *   0 ok, 1 empty_input_error, 2 non_finite_error, 3 invalid_k_error,
 *   4 invalid_chunk_error.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EMPTY 1
#define OR_NON_FINITE 2
#define OR_INVALID_K 3
#define OR_INVALID_CHUNK 4

/* ---------------------------------------------------------------- (m,d) --- */

/* norm_state<double>::add, normalizer.hpp:32-41 */
static int norm_add_d(double *m, double *d, double x) {
  if (!isfinite(x)) return OR_NON_FINITE;               /* :33 */
  if (x > *m) {                                         /* :34-37 */
    *d = *d * exp(*m - x) + 1.0;
    *m = x;
  } else {                                              /* :38-40 */
    *d += exp(x - *m);
  }
  return OR_OK;
}

/* norm_state<float>::add, normalizer.hpp:32-41 with T=float (expf) */
static int norm_add_f(float *m, float *d, float x) {
  if (!isfinite(x)) return OR_NON_FINITE;
  if (x > *m) {
    *d = *d * expf(*m - x) + 1.0f;
    *m = x;
  } else {
    *d += expf(x - *m);
  }
  return OR_OK;
}

/* merge(), normalizer.hpp:52-58; identity = (-inf, ..) (:43) */
void oracle_merge_d(double am, double ad, double bm, double bd, double *om, double *od) {
  if (isinf(am) && am < 0) { *om = bm; *od = bd; return; }   /* :54 */
  if (isinf(bm) && bm < 0) { *om = am; *od = ad; return; }   /* :55 */
  const double m = am > bm ? am : bm;                        /* :56 std::max */
  *om = m;
  *od = ad * exp(am - m) + bd * exp(bm - m);                 /* :57 */
}

void oracle_merge_f(float am, float ad, float bm, float bd, float *om, float *od) {
  if (isinf(am) && am < 0) { *om = bm; *od = bd; return; }
  if (isinf(bm) && bm < 0) { *om = am; *od = ad; return; }
  const float m = am > bm ? am : bm;
  *om = m;
  *od = ad * expf(am - m) + bd * expf(bm - m);
}

/* run_normalizer<T>, normalizer.hpp:61-67.  dbl selects T=double. */
int oracle_run_normalizer(const float *x, size_t n, int dbl, double *om, double *od) {
  if (n == 0) return OR_EMPTY;
  if (dbl) {
    double m = -INFINITY, d = 0.0;
    for (size_t i = 0; i < n; ++i) {
      int st = norm_add_d(&m, &d, (double)x[i]);
      if (st) return st;
    }
    *om = m; *od = d;
  } else {
    float m = -INFINITY, d = 0.0f;
    for (size_t i = 0; i < n; ++i) {
      int st = norm_add_f(&m, &d, x[i]);
      if (st) return st;
    }
    *om = m; *od = d;
  }
  return OR_OK;
}

/* run_normalizer_chunked<T>, normalizer.hpp:73-85: contiguous chunks, each
 * reduced sequentially, merged left to right. */
int oracle_run_normalizer_chunked(const float *x, size_t n, size_t chunk, int dbl,
                                  double *om, double *od) {
  if (n == 0) return OR_EMPTY;                               /* :74 */
  if (chunk == 0) return OR_INVALID_CHUNK;                   /* :75-76 */
  if (dbl) {
    double am = -INFINITY, ad = 0.0;
    for (size_t s = 0; s < n; s += chunk) {
      const size_t len = chunk < n - s ? chunk : n - s;
      double pm = -INFINITY, pd = 0.0;
      for (size_t i = s; i < s + len; ++i) {
        int st = norm_add_d(&pm, &pd, (double)x[i]);
        if (st) return st;
      }
      oracle_merge_d(am, ad, pm, pd, &am, &ad);              /* :82 */
    }
    *om = am; *od = ad;
  } else {
    float am = -INFINITY, ad = 0.0f;
    for (size_t s = 0; s < n; s += chunk) {
      const size_t len = chunk < n - s ? chunk : n - s;
      float pm = -INFINITY, pd = 0.0f;
      for (size_t i = s; i < s + len; ++i) {
        int st = norm_add_f(&pm, &pd, x[i]);
        if (st) return st;
      }
      oracle_merge_f(am, ad, pm, pd, &am, &ad);
    }
    *om = am; *od = ad;
  }
  return OR_OK;
}

/* ------------------------------------------------------------- softmax --- */

static int all_finite(const float *x, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

/* naive_softmax_kernel, kernels.hpp:39-46.  d = sum double(expf(x_j));
 * y_i = float(expf(x_i) / d) -- no overflow guard. */
int oracle_naive_softmax(const float *x, size_t n, float *y) {
  if (n == 0) return OR_EMPTY;
  double d = 0.0;
  for (size_t j = 0; j < n; ++j) {
    if (!isfinite(x[j])) return OR_NON_FINITE;                /* checked() :32-35 */
    d += (double)expf(x[j]);
  }
  for (size_t i = 0; i < n; ++i) y[i] = (float)((double)expf(x[i]) / d);
  return OR_OK;
}

/* max pass + double normalizer of safe_softmax_kernel, kernels.hpp:53-56 */
static int safe_md(const float *x, size_t n, float *om, double *od) {
  float m = -INFINITY;
  for (size_t j = 0; j < n; ++j) {
    if (!isfinite(x[j])) return OR_NON_FINITE;
    m = (m < x[j]) ? x[j] : m;                                 /* std::max(m, x) */
  }
  double d = 0.0;
  for (size_t j = 0; j < n; ++j) d += exp((double)x[j] - (double)m);
  *om = m; *od = d;
  return OR_OK;
}

/* safe_softmax_kernel, kernels.hpp:49-58 */
int oracle_safe_softmax(const float *x, size_t n, float *y) {
  if (n == 0) return OR_EMPTY;
  float m; double d;
  int st = safe_md(x, n, &m, &d);
  if (st) return st;
  for (size_t i = 0; i < n; ++i) y[i] = (float)((double)expf(x[i] - m) / d);   /* :57 */
  return OR_OK;
}

/* online_softmax_kernel, kernels.hpp:61-69: norm_state<double> over double(x) */
static int online_md(const float *x, size_t n, float *om, double *od) {
  double m = -INFINITY, d = 0.0;
  for (size_t j = 0; j < n; ++j) {
    int st = norm_add_d(&m, &d, (double)x[j]);                 /* :66 */
    if (st) return st;
  }
  *om = (float)m;                                              /* :67 */
  *od = d;
  return OR_OK;
}

int oracle_online_softmax(const float *x, size_t n, float *y) {
  if (n == 0) return OR_EMPTY;
  float m; double d;
  int st = online_md(x, n, &m, &d);
  if (st) return st;
  for (size_t i = 0; i < n; ++i) y[i] = (float)((double)expf(x[i] - m) / d);   /* :68 */
  return OR_OK;
}

/* ---------------------------------------------------------------- top-K --- */

/* topk_buffer, topk.hpp:25-50: K+1 slots, values -inf, indices -1. */
typedef struct {
  float *v;
  int64_t *z;
  size_t k;
} topk_buf;

static void buf_init(topk_buf *b, size_t k, float *v, int64_t *z) {
  b->v = v; b->z = z; b->k = k;
  for (size_t i = 0; i <= k; ++i) { v[i] = -INFINITY; z[i] = -1; }   /* :27-28 */
}

/* topk_buffer::offer, topk.hpp:34-44 */
static void buf_offer(topk_buf *b, float value, int64_t index) {
  const size_t k = b->k;
  if (!(value > b->v[k - 1]) && b->z[k - 1] >= 0) return;            /* :37 */
  b->v[k] = value;
  b->z[k] = index;
  for (size_t s = k; s >= 1 && b->v[s - 1] < b->v[s]; --s) {          /* :40-43 strict < */
    float tv = b->v[s - 1]; b->v[s - 1] = b->v[s]; b->v[s] = tv;
    int64_t tz = b->z[s - 1]; b->z[s - 1] = b->z[s]; b->z[s] = tz;
  }
}

static int check_k(size_t n, size_t k) {
  if (n == 0) return OR_EMPTY;                                        /* require_nonempty :24-26 */
  if (k == 0 || k > n) return OR_INVALID_K;                           /* require_valid_k :28-30 */
  return OR_OK;
}

#define MAXK_STACK 64

/* topk_kernel / topk_of, kernels.hpp:72-83, topk.cpp:20-28 */
int oracle_topk_of(const float *v, size_t n, size_t k, float *ov, int64_t *oz) {
  int st = check_k(n, k);
  if (st) return st;
  float sv[MAXK_STACK + 1]; int64_t sz[MAXK_STACK + 1];
  float *bv = k <= MAXK_STACK ? sv : (float *)malloc((k + 1) * sizeof(float));
  int64_t *bz = k <= MAXK_STACK ? sz : (int64_t *)malloc((k + 1) * sizeof(int64_t));
  topk_buf b; buf_init(&b, k, bv, bz);
  for (size_t j = 0; j < n; ++j) {
    if (!isfinite(v[j])) { st = OR_NON_FINITE; break; }               /* checked() :78 */
    buf_offer(&b, v[j], (int64_t)j);
  }
  if (!st) for (size_t i = 0; i < k; ++i) { ov[i] = bv[i]; oz[i] = bz[i]; }
  if (bv != sv) free(bv);
  if (bz != sz) free(bz);
  return st;
}

/* safe_softmax_then_topk, topk.cpp:30-35: materialise y, then topk_of(y) */
int oracle_safe_softmax_then_topk(const float *x, size_t n, size_t k, float *ov, int64_t *oz) {
  int st = check_k(n, k);
  if (st) return st;
  float *y = (float *)malloc(n * sizeof(float));
  st = oracle_safe_softmax(x, n, y);
  if (!st) st = oracle_topk_of(y, n, k, ov, oz);
  free(y);
  return st;
}

/* safe_softmax_fused_topk_kernel, kernels.hpp:87-104: selection keyed on
 * float(expf(x-m)/d); the probability vector is never stored. */
int oracle_safe_softmax_fused_topk(const float *x, size_t n, size_t k, float *ov, int64_t *oz) {
  int st = check_k(n, k);
  if (st) return st;
  float m; double d;
  st = safe_md(x, n, &m, &d);
  if (st) return st;
  float sv[MAXK_STACK + 1]; int64_t sz[MAXK_STACK + 1];
  float *bv = k <= MAXK_STACK ? sv : (float *)malloc((k + 1) * sizeof(float));
  int64_t *bz = k <= MAXK_STACK ? sz : (int64_t *)malloc((k + 1) * sizeof(int64_t));
  topk_buf b; buf_init(&b, k, bv, bz);
  for (size_t j = 0; j < n; ++j)
    buf_offer(&b, (float)((double)expf(x[j] - m) / d), (int64_t)j);  /* :98 */
  for (size_t i = 0; i < k; ++i) { ov[i] = bv[i]; oz[i] = bz[i]; }
  if (bv != sv) free(bv);
  if (bz != sz) free(bz);
  return OR_OK;
}

/* online_softmax_topk_kernel, kernels.hpp:108-125: one pass, (m,d) in
 * double plus the raw-logit top-K buffer; only the winners are exponentiated. */
int oracle_online_softmax_topk(const float *x, size_t n, size_t k, float *ov, int64_t *oz) {
  int st = check_k(n, k);
  if (st) return st;
  float sv[MAXK_STACK + 1]; int64_t sz[MAXK_STACK + 1];
  float *bv = k <= MAXK_STACK ? sv : (float *)malloc((k + 1) * sizeof(float));
  int64_t *bz = k <= MAXK_STACK ? sz : (int64_t *)malloc((k + 1) * sizeof(int64_t));
  topk_buf b; buf_init(&b, k, bv, bz);
  double m = -INFINITY, d = 0.0;
  for (size_t j = 0; j < n && !st; ++j) {
    const float e = x[j];
    st = norm_add_d(&m, &d, (double)e);                              /* :116 */
    if (!st) buf_offer(&b, e, (int64_t)j);                           /* :117 */
  }
  if (!st) {
    const float mf = (float)m;                                       /* :120 */
    for (size_t i = 0; i < k; ++i) {
      ov[i] = (float)((double)expf(bv[i] - mf) / d);                 /* :122 */
      oz[i] = bz[i];
    }
  }
  if (bv != sv) free(bv);
  if (bz != sz) free(bz);
  return st;
}

/* ---------------------------------------------------------------- oracle -- */

/* oracle_softmax, oracle.cpp:23-32 (double throughout) */
int oracle_softmax_double(const float *x, size_t n, double *y) {
  if (n == 0) return OR_EMPTY;
  if (!all_finite(x, n)) return OR_NON_FINITE;
  double m = -INFINITY;
  for (size_t i = 0; i < n; ++i) m = (m < (double)x[i]) ? (double)x[i] : m;
  double d = 0.0;
  for (size_t i = 0; i < n; ++i) d += exp((double)x[i] - m);
  for (size_t i = 0; i < n; ++i) y[i] = exp((double)x[i] - m) / d;
  return OR_OK;
}

/* oracle_normalizer, oracle.cpp:34-41 */
int oracle_normalizer_double(const float *x, size_t n, double *om, double *od) {
  if (n == 0) return OR_EMPTY;
  if (!all_finite(x, n)) return OR_NON_FINITE;
  double m = -INFINITY;
  for (size_t i = 0; i < n; ++i) m = (m < (double)x[i]) ? (double)x[i] : m;
  double d = 0.0;
  for (size_t i = 0; i < n; ++i) d += exp((double)x[i] - m);
  *om = m; *od = d;
  return OR_OK;
}

/* oracle_topk, oracle.cpp:43-60: full order on (value desc, index asc).  A
 * stable merge sort on value desc gives exactly that order. */
static void msort(const float *v, int64_t *a, int64_t *tmp, size_t n) {
  if (n < 2) return;
  size_t h = n / 2;
  msort(v, a, tmp, h);
  msort(v, a + h, tmp, n - h);
  size_t i = 0, j = h, o = 0;
  while (i < h && j < n) {
    /* take right only when strictly greater: ties keep the lower index */
    if (v[a[j]] > v[a[i]]) tmp[o++] = a[j++];
    else tmp[o++] = a[i++];
  }
  while (i < h) tmp[o++] = a[i++];
  while (j < n) tmp[o++] = a[j++];
  memcpy(a, tmp, n * sizeof(int64_t));
}

int oracle_topk_sort(const float *v, size_t n, size_t k, float *ov, int64_t *oz) {
  if (n == 0) return OR_EMPTY;
  if (!all_finite(v, n)) return OR_NON_FINITE;
  if (k == 0 || k > n) return OR_INVALID_K;
  int64_t *a = (int64_t *)malloc(n * sizeof(int64_t));
  int64_t *t = (int64_t *)malloc(n * sizeof(int64_t));
  for (size_t i = 0; i < n; ++i) a[i] = (int64_t)i;
  msort(v, a, t, n);
  for (size_t i = 0; i < k; ++i) { ov[i] = v[a[i]]; oz[i] = a[i]; }
  free(a); free(t);
  return OR_OK;
}

/* --------------------------------------------------- access-count model --- */

/* count_accesses, counting.hpp:77-86 (exact element loads / stores).
 * alg: 0 naive 1 safe 2 online 3 safe-unfused-topk 4 safe-fused-topk
 *      5 online-fused-topk (counting.hpp:17-24 order). */
int oracle_count_accesses(int alg, uint64_t v, uint64_t k, uint64_t *loads, uint64_t *stores) {
  if (v == 0) return OR_EMPTY;
  const int topk = alg >= 3;
  if (topk ? (k == 0 || k > v) : (k != 0)) return OR_INVALID_K;
  switch (alg) {
    case 0: *loads = 2 * v; *stores = v; break;                 /* naive 3V */
    case 1: *loads = 3 * v; *stores = v; break;                 /* safe 4V */
    case 2: *loads = 2 * v; *stores = v; break;                 /* online 3V */
    case 3: *loads = 4 * v; *stores = v + 2 * k; break;         /* safe unfused 5V+2K */
    case 4: *loads = 3 * v; *stores = 2 * k; break;             /* safe fused 3V+2K */
    case 5: *loads = v; *stores = 2 * k; break;                 /* online fused V+2K */
    default: return OR_INVALID_K;
  }
  return OR_OK;
}

/* ------------------------------------------------ batched, row-striped --- */

/* Row-parallel driver with the striping of run_batch, bench.cpp:66-96
 * (worker t takes rows t, t+T, ...).  op: 0 naive 1 safe 2 online
 * 3 safe-unfused-topk 4 safe-fused-topk 5 online-fused-topk 6 topk_of.
 * Per-row statuses land in st[row]. */
typedef struct {
  int op;
  const float *x; int64_t ldx;
  float *y; int64_t ldy;
  float *v; int64_t *z;
  int64_t rows, n, k;
  int32_t *st;
  int t, T;
} batch_job;

static void *batch_worker(void *arg) {
  batch_job *j = (batch_job *)arg;
  for (int64_t r = j->t; r < j->rows; r += j->T) {
    const float *xr = j->x + r * j->ldx;
    int s = 0;
    switch (j->op) {
      case 0: s = oracle_naive_softmax(xr, (size_t)j->n, j->y + r * j->ldy); break;
      case 1: s = oracle_safe_softmax(xr, (size_t)j->n, j->y + r * j->ldy); break;
      case 2: s = oracle_online_softmax(xr, (size_t)j->n, j->y + r * j->ldy); break;
      case 3: s = oracle_safe_softmax_then_topk(xr, (size_t)j->n, (size_t)j->k, j->v + r * j->k, j->z + r * j->k); break;
      case 4: s = oracle_safe_softmax_fused_topk(xr, (size_t)j->n, (size_t)j->k, j->v + r * j->k, j->z + r * j->k); break;
      case 5: s = oracle_online_softmax_topk(xr, (size_t)j->n, (size_t)j->k, j->v + r * j->k, j->z + r * j->k); break;
      case 6: s = oracle_topk_of(xr, (size_t)j->n, (size_t)j->k, j->v + r * j->k, j->z + r * j->k); break;
      default: s = -1;
    }
    if (j->st) j->st[r] = s;
  }
  return 0;
}

int oracle_batch(int op, const float *x, int64_t ldx, int64_t rows, int64_t n, int64_t k,
                 float *y, int64_t ldy, float *v, int64_t *z, int32_t *st, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 512) threads = 512;
  batch_job jobs[512];
  pthread_t tid[512];
  for (int t = 0; t < threads; ++t) {
    batch_job jb = {op, x, ldx, y, ldy, v, z, rows, n, k, st, t, threads};
    jobs[t] = jb;
  }
  if (threads == 1) { batch_worker(&jobs[0]); return 0; }
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], 0, batch_worker, &jobs[t]);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], 0);
  return 0;
}
