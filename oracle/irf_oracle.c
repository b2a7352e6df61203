// TEST INFRASTRUCTURE: C restatement of the reference's interval root
// finder baseline, ccdkit.baselines.irf_solve
// (pkg/src/ccdkit/baselines.py:123-206), with IntervalScalar (:37-106:
// every operation widened one representable step outward with nextafter)
// and _interval_F (:109-120).  Pinned against outputs of the reference
// itself (tests/golden/irf_*.npz, tests/golden/make_irf_golden.py); used by
// tests/ as the checker of the GPU IRF and by tools as its CPU baseline.
// Built with -ffp-contract=off (see Makefile).
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double lo, hi;
} iv_t;

// IntervalScalar._outward (baselines.py:56-61)
static inline iv_t outward(double lo, double hi) {
  iv_t r = {nextafter(lo, -INFINITY), nextafter(hi, INFINITY)};
  return r;
}

static inline iv_t iv_pt(double x) {  // IntervalScalar._coerce of a float (:63-66)
  iv_t r = {x, x};
  return r;
}

static inline iv_t iv_add(iv_t a, iv_t b) { return outward(a.lo + b.lo, a.hi + b.hi); }  // :68-70
static inline iv_t iv_sub(iv_t a, iv_t b) { return outward(a.lo - b.hi, a.hi - b.lo); }  // :74-76

// :81-87; min / max with Python's semantics (the first of equal values is
// kept, a later one replaces it only if strictly smaller / larger)
static inline iv_t iv_mul(iv_t a, iv_t b) {
  const double p1 = a.lo * b.lo, p2 = a.lo * b.hi, p3 = a.hi * b.lo, p4 = a.hi * b.hi;
  double mn = p1, mx = p1;
  if (p2 < mn) mn = p2;
  if (p3 < mn) mn = p3;
  if (p4 < mn) mn = p4;
  if (p2 > mx) mx = p2;
  if (p3 > mx) mx = p3;
  if (p4 > mx) mx = p4;
  return outward(mn, mx);
}

// _interval_F (:109-120) on axis ax: the lerped points, then the VF / EE form
static iv_t interval_F(const double *s, const double *e, int kind, int ax, iv_t t, iv_t u,
                       iv_t v) {
  iv_t p[4];
  const iv_t omt = iv_sub(iv_pt(1.0), t);
  for (int j = 0; j < 4; ++j)
    p[j] = iv_add(iv_mul(omt, iv_pt(s[3 * j + ax])), iv_mul(t, iv_pt(e[3 * j + ax])));
  if (kind == 0) {
    const iv_t w = iv_sub(iv_sub(iv_pt(1.0), u), v);
    return iv_sub(p[0], iv_add(iv_add(iv_mul(w, p[1]), iv_mul(u, p[2])), iv_mul(v, p[3])));
  }
  const iv_t l = iv_add(iv_mul(iv_sub(iv_pt(1.0), u), p[0]), iv_mul(u, p[1]));
  const iv_t r = iv_add(iv_mul(iv_sub(iv_pt(1.0), v), p[2]), iv_mul(v, p[3]));
  return iv_sub(l, r);
}

typedef struct {
  double b[6];  // tl, th, ul, uh, vl, vh
  int64_t level, seq;
} node_t;

// heap order: the tuple (t_lo, level, seq) of baselines.py:144,202
static inline int node_less(const node_t *a, const node_t *b) {
  if (a->b[0] != b->b[0]) return a->b[0] < b->b[0];
  if (a->level != b->level) return a->level < b->level;
  return a->seq < b->seq;
}

typedef struct {
  node_t *h;
  int64_t n, cap;
} heap_t;

static int heap_push(heap_t *H, const node_t *x) {
  if (H->n == H->cap) {
    const int64_t nc = H->cap ? 2 * H->cap : 64;
    node_t *nh = (node_t *)realloc(H->h, (size_t)nc * sizeof(node_t));
    if (!nh) return -1;
    H->h = nh;
    H->cap = nc;
  }
  int64_t i = H->n++;
  while (i > 0) {
    const int64_t p = (i - 1) / 2;
    if (!node_less(x, &H->h[p])) break;
    H->h[i] = H->h[p];
    i = p;
  }
  H->h[i] = *x;
  return 0;
}

static node_t heap_pop(heap_t *H) {
  const node_t top = H->h[0];
  const node_t last = H->h[--H->n];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= H->n) break;
    if (c + 1 < H->n && node_less(&H->h[c + 1], &H->h[c])) ++c;
    if (!node_less(&H->h[c], &last)) break;
    H->h[i] = H->h[c];
    i = c;
  }
  if (H->n > 0) H->h[i] = last;
  return top;
}

// status: 0 free, 1 hit, 4 invalid delta / t_max (ValueError), 3 non-finite
// coordinates, 5 allocation failure.  out: toi, tol, codom, witness[6], level
static int irf_one(const double *s, const double *e, int kind, double delta, int64_t max_checks,
                   double t_max, heap_t *H, double *toi, double *tol, double *codom,
                   int64_t *checks_out, uint8_t *early, double *wit, int32_t *level) {
  *toi = INFINITY;
  *tol = 0.0;
  *codom = 0.0;
  *early = 0;
  *level = 0;
  memset(wit, 0, 6 * sizeof(double));
  *checks_out = 0;
  for (int i = 0; i < 12; ++i)
    if (!isfinite(s[i]) || !isfinite(e[i])) return 3;
  if (!(delta > 0.0)) return 4;                     // :139-140
  if (!(isfinite(t_max) && t_max >= 0.0)) return 4;  // IntervalScalar(0, t_max) (:53-54)
  H->n = 0;
  node_t root = {{0.0, t_max, 0.0, 1.0, 0.0, 1.0}, 0, 0};
  if (heap_push(H, &root)) return 5;
  int64_t seq = 0, checks = 0;
  while (H->n > 0) {
    const node_t nd = heap_pop(H);
    const double *b = nd.b;
    const iv_t t = {b[0], b[1]}, u = {b[2], b[3]}, v = {b[4], b[5]};
    iv_t F[3];
    const int budget = checks >= max_checks;  // :147-165
    int all = 1;
    for (int ax = 0; ax < 3; ++ax) {
      F[ax] = interval_F(s, e, kind, ax, t, u, v);
      all = all && (F[ax].lo <= 0.0 && 0.0 <= F[ax].hi);
    }
    double cw = F[0].hi - F[0].lo;  // max(ax.width for ax in F)
    for (int ax = 1; ax < 3; ++ax)
      if (F[ax].hi - F[ax].lo > cw) cw = F[ax].hi - F[ax].lo;
    if (budget) {
      *toi = b[0];
      *tol = b[1] - b[0];
      *codom = cw;
      *checks_out = checks;
      *early = 1;
      memcpy(wit, b, 6 * sizeof(double));
      *level = (int32_t)nd.level;
      return 1;
    }
    ++checks;
    if (!all) continue;  // :172-173
    const double w[3] = {b[1] - b[0], b[3] - b[2], b[5] - b[4]};
    double mw = w[0];
    int dim = 0;  // np.argmax: the first maximum
    for (int k = 1; k < 3; ++k)
      if (w[k] > mw) { mw = w[k]; dim = k; }
    if (mw < delta) {  // :175-185
      *toi = b[0];
      *tol = b[1] - b[0];
      *codom = cw;
      *checks_out = checks;
      memcpy(wit, b, 6 * sizeof(double));
      *level = (int32_t)nd.level;
      return 1;
    }
    const double m = 0.5 * (b[2 * dim] + b[2 * dim + 1]);
    node_t kid[2];
    kid[0].level = kid[1].level = nd.level + 1;
    memcpy(kid[0].b, b, sizeof kid[0].b);
    memcpy(kid[1].b, b, sizeof kid[1].b);
    kid[0].b[2 * dim + 1] = m;
    kid[1].b[2 * dim] = m;
    for (int k = 0; k < 2; ++k) {
      if (kind == 0 && kid[k].b[2] + kid[k].b[4] > 1.0) continue;  // :197-199
      kid[k].seq = ++seq;
      if (heap_push(H, &kid[k])) return 5;
    }
  }
  *checks_out = checks;
  return 0;
}

typedef struct {
  int64_t n;
  const double *points;
  const uint8_t *kind;
  int kind_all;
  const double *delta;
  double delta_all;
  const int64_t *mc;
  int64_t mc_all;
  const double *tmax;
  double tmax_all;
  uint8_t *status;
  double *toi, *tol, *codom, *witness;
  int64_t *checks;
  uint8_t *early;
  int32_t *level;
  int64_t next;
  pthread_mutex_t mu;
} irf_batch_t;

static void *irf_worker(void *arg) {
  irf_batch_t *B = (irf_batch_t *)arg;
  heap_t H = {NULL, 0, 0};
  for (;;) {
    pthread_mutex_lock(&B->mu);
    const int64_t q0 = B->next;
    B->next += 16;
    pthread_mutex_unlock(&B->mu);
    if (q0 >= B->n) break;
    const int64_t q1 = q0 + 16 < B->n ? q0 + 16 : B->n;
    for (int64_t q = q0; q < q1; ++q) {
      const double *p = B->points + 24 * q;
      B->status[q] = (uint8_t)irf_one(
          p, p + 12, B->kind ? B->kind[q] : B->kind_all, B->delta ? B->delta[q] : B->delta_all,
          B->mc ? B->mc[q] : B->mc_all, B->tmax ? B->tmax[q] : B->tmax_all, &H, &B->toi[q],
          &B->tol[q], &B->codom[q], &B->checks[q], &B->early[q], B->witness + 6 * q,
          &B->level[q]);
    }
  }
  free(H.h);
  return NULL;
}

int tccd_oracle_irf_batch(int64_t n, const double *points, const uint8_t *kind, int kind_all,
                          const double *delta, double delta_all, const int64_t *max_checks,
                          int64_t max_checks_all, const double *t_max, double t_max_all,
                          uint8_t *status, double *toi, double *tol, double *codom,
                          int64_t *checks, uint8_t *early, double *witness, int32_t *level,
                          int threads) {
  irf_batch_t B = {n, points, kind, kind_all, delta, delta_all, max_checks, max_checks_all,
                   t_max, t_max_all, status, toi, tol, codom, witness, checks, early, level,
                   0, PTHREAD_MUTEX_INITIALIZER};
  if (threads < 1) threads = 1;
  pthread_t *th = (pthread_t *)malloc((size_t)threads * sizeof(pthread_t));
  if (!th) return 1;
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, irf_worker, &B);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
  return 0;
}
