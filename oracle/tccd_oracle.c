/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the tccd hot path.
 *
 * A plain-C restatement of the reference's conservative bisection solver
 * (ccdkit._kernel.solve_kernel, pkg/src/ccdkit/_kernel.py:136-324) and the
 * per-query filter resolution it is fed with (solver._resolve_filters,
 * pkg/src/ccdkit/solver.py:30-47 -> inclusion.compute_gamma /
 * compute_filters, pkg/src/ccdkit/inclusion.py:85-122).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * the --impl reference arm) may load this library, and only as the checker
 * or the timed CPU baseline.  The product path (paper_2009_13349_b200) never
 * links or calls it.
 *
 * Parity pin: tests/golden/make_golden.py runs the reference itself (numba,
 * imported from /root/reference in the build container) on the handcrafted
 * battery, the KATs and seeded samples of all five workloads, and
 * tests/test_oracle_golden.py asserts this file reproduces every recorded
 * output bit for bit.
 *
 * Floating point: compile with -ffp-contract=off and without -ffast-math so
 * every operation below is one IEEE binary64 round-to-nearest op in the
 * written order (the order the filter constants were derived for,
 * pkg/src/ccdkit/core.py:19-23, inclusion.py:8-15).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ST_FREE 0
#define ST_HIT 1
#define ST_ERR_SEPARATION 2 /* d >= gamma on an axis (inclusion.py:110-113) */
#define ST_ERR_NONFINITE 3  /* non-finite coordinate (core.py:42-53)        */
#define ST_ERR_PARAM 4      /* delta/m_I/d/t_max invalid (core.py:176-184)  */

#define CLS_DISJOINT 0   /* _kernel.py:36-38 */
#define CLS_INTERSECTS 1
#define CLS_CONTAINED 2

/* inclusion.py:35-38 */
static const double COEF_VF = 6.661338147750939e-15;
static const double COEF_EE = 6.217248937900877e-15;
static const double COEF_VF_D = 7.549516567451064e-15;
static const double COEF_EE_D = 7.105427357601002e-15;

typedef struct {
  double t0, t1, u0, u1, v0, v1;
} box_t;

typedef struct {
  int32_t status;
  int32_t early;
  int32_t level;
  int64_t checks;
  double toi, tol, codom;
  double w[6];
} result_t;

/* One corner value of F on one axis; p[k] is point k lerped to time t.
 * VF: core.py:225-238, EE: core.py:241-256 (left-associative order). */
static inline double corner(int kind, const double p[4], double u, double v) {
  if (kind == 0) return p[0] - ((1.0 - u - v) * p[1] + u * p[2] + v * p[3]);
  return ((1.0 - u) * p[0] + u * p[1]) - ((1.0 - v) * p[2] + v * p[3]);
}

/* s, e: [4][3] start/end positions.  Lerp as (1 - t) * s + t * e. */
static inline void lerp_axis(const double *s, const double *e, int ax, double t,
                             double p[4]) {
  double omt = 1.0 - t;
  for (int k = 0; k < 4; ++k) p[k] = omt * s[3 * k + ax] + t * e[3 * k + ax];
}

/* _kernel._hull_axis, _kernel.py:44-67: min/max over the 8 box corners. */
static void hull_axis(const double *s, const double *e, int kind, int ax,
                      const box_t *b, double *mn, double *mx) {
  double lo = INFINITY, hi = -INFINITY;
  double ts[2] = {b->t0, b->t1}, us[2] = {b->u0, b->u1}, vs[2] = {b->v0, b->v1};
  for (int it = 0; it < 2; ++it) {
    double p[4];
    lerp_axis(s, e, ax, ts[it], p);
    for (int iu = 0; iu < 2; ++iu)
      for (int iv = 0; iv < 2; ++iv) {
        double val = corner(kind, p, us[iu], vs[iv]);
        if (val < lo) lo = val;
        if (val > hi) hi = val;
      }
  }
  *mn = lo;
  *mx = hi;
}

/* _kernel._classify, _kernel.py:71-94. */
static int classify(const double *s, const double *e, int kind, const box_t *b,
                    const double eps[3], double sep, double *wb_out) {
  int contained = 1;
  double wb = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    double mn, mx;
    hull_axis(s, e, kind, ax, b, &mn, &mx);
    double lo = mn - sep, hi = mx + sep;
    if (lo > eps[ax] || hi < -eps[ax]) {
      *wb_out = 0.0;
      return CLS_DISJOINT;
    }
    if (!(lo >= -eps[ax] && hi <= eps[ax])) contained = 0;
    double w = mx - mn;
    if (w > wb) wb = w;
  }
  *wb_out = wb;
  return contained ? CLS_CONTAINED : CLS_INTERSECTS;
}

/* _kernel._kappas, _kernel.py:98-132: 3 * max corner-pair |dF| per dim on
 * [0, t_max] x [0,1]^2, corner index 4*t + 2*u + v. */
void tccd_oracle_kappas(const double *s, const double *e, int kind, double t_max,
                        double out[3]) {
  double F[8][3];
  for (int it = 0; it < 2; ++it) {
    double t = it ? t_max : 0.0;
    for (int ax = 0; ax < 3; ++ax) {
      double p[4];
      lerp_axis(s, e, ax, t, p);
      for (int iu = 0; iu < 2; ++iu)
        for (int iv = 0; iv < 2; ++iv)
          F[4 * it + 2 * iu + iv][ax] =
              corner(kind, p, iu ? 1.0 : 0.0, iv ? 1.0 : 0.0);
    }
  }
  static const int strides[3] = {4, 2, 1};
  for (int k = 0; k < 3; ++k) {
    int st = strides[k];
    double best = 0.0;
    for (int i = 0; i < 8; ++i) {
      if (i & st) continue;
      for (int ax = 0; ax < 3; ++ax) {
        double d = fabs(F[i + st][ax] - F[i][ax]);
        if (d > best) best = d;
      }
    }
    out[k] = 3.0 * best;
  }
}

/* compute_gamma + compute_filters (inclusion.py:85-122).  pts: [8][3] (start
 * block then end block).  Returns a status code (ST_HIT on success). */
int tccd_oracle_filters(const double *pts, int kind, double sep, double eps[3]) {
  double g[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < 8; ++i)
    for (int ax = 0; ax < 3; ++ax) {
      double x = pts[3 * i + ax];
      if (!isfinite(x)) return ST_ERR_NONFINITE;
      double a = fabs(x);
      if (a > g[ax]) g[ax] = a;
    }
  for (int ax = 0; ax < 3; ++ax) g[ax] = g[ax] > 1.0 ? g[ax] : 1.0;
  double c;
  if (sep > 0.0) {
    if (!(sep < g[0] && sep < g[1] && sep < g[2])) return ST_ERR_SEPARATION;
    c = kind == 0 ? COEF_VF_D : COEF_EE_D;
  } else {
    c = kind == 0 ? COEF_VF : COEF_EE;
  }
  for (int ax = 0; ax < 3; ++ax) eps[ax] = c * (g[ax] * g[ax] * g[ax]);
  return ST_HIT;
}

/* Stable ascending order of keys[0..n) into ord (merge sort; equal keys keep
 * index order, matching numpy argsort(kind="mergesort"), _kernel.py:174-175). */
static void stable_order(const double *keys, int64_t n, int64_t *ord, int64_t *tmp) {
  for (int64_t i = 0; i < n; ++i) ord[i] = i;
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      int64_t mid = lo + w < n ? lo + w : n;
      int64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t a = lo, b = mid, k = lo;
      while (a < mid && b < hi) {
        if (keys[ord[b]] < keys[ord[a]]) tmp[k++] = ord[b++];
        else tmp[k++] = ord[a++];
      }
      while (a < mid) tmp[k++] = ord[a++];
      while (b < hi) tmp[k++] = ord[b++];
    }
    memcpy(ord, tmp, (size_t)n * sizeof(int64_t));
  }
}

/* diagnostics: boxes visited per level, bucketed by floor(log2(level width))
 * (includes boxes past an early return in their level) */
int64_t tccd_oracle_level_hist[64];

typedef struct {
  box_t *cur, *nxt;
  double *keys;
  int64_t *ord, *tmp;
  int64_t cap;
  int64_t max_frontier; /* diagnostics of the last solve: widest level */
  int64_t levels;       /* and number of levels visited */
} arena_t;

static int arena_reserve(arena_t *a, int64_t need) {
  if (need <= a->cap) return 0;
  int64_t cap = a->cap ? a->cap : 64;
  while (cap < need) cap *= 2;
  box_t *c = realloc(a->cur, (size_t)cap * sizeof(box_t));
  if (!c) return -1;
  a->cur = c;
  box_t *x = realloc(a->nxt, (size_t)cap * sizeof(box_t));
  if (!x) return -1;
  a->nxt = x;
  double *k = realloc(a->keys, (size_t)cap * sizeof(double));
  if (!k) return -1;
  a->keys = k;
  int64_t *o = realloc(a->ord, (size_t)cap * sizeof(int64_t));
  if (!o) return -1;
  a->ord = o;
  int64_t *t = realloc(a->tmp, (size_t)cap * sizeof(int64_t));
  if (!t) return -1;
  a->tmp = t;
  a->cap = cap;
  return 0;
}

static void arena_free(arena_t *a) {
  free(a->cur); free(a->nxt); free(a->keys); free(a->ord); free(a->tmp);
  memset(a, 0, sizeof(*a));
}

static void set_result(result_t *r, const box_t *b, double codom, int64_t checks,
                       int early, int level) {
  r->status = ST_HIT;
  r->toi = b->t0;
  r->tol = b->t1 - b->t0;
  r->codom = codom;
  r->checks = checks;
  r->early = early;
  r->w[0] = b->t0; r->w[1] = b->t1; r->w[2] = b->u0;
  r->w[3] = b->u1; r->w[4] = b->v0; r->w[5] = b->v1;
  r->level = level;
}

/* The level-ordered bisection state machine, _kernel.py:136-324. */
static int solve_one(const double *s, const double *e, int kind, double t_max,
                     double delta, int64_t max_checks, double sep,
                     const double eps[3], arena_t *ar, result_t *r) {
  double kap[3];
  tccd_oracle_kappas(s, e, kind, t_max, kap);
  if (arena_reserve(ar, 64)) return -1;
  box_t *cur = ar->cur, *nxt = ar->nxt;
  cur[0] = (box_t){0.0, t_max, 0.0, 1.0, 0.0, 1.0};
  int64_t ncur = 1, nnxt = 0, checks = 0;
  int level = 0, last_col = -1;
  int have_first = 0, have_drop = 0;
  box_t fb = {0}, db = {0};
  int f_level = 0, d_level = 0;
  double f_codom = 0.0, d_codom = 0.0;

  ar->max_frontier = 0;
  ar->levels = 0;
  extern int64_t tccd_oracle_level_hist[64];
  while (ncur > 0) {
    if (ncur > ar->max_frontier) ar->max_frontier = ncur;
    ar->levels++;
    __atomic_fetch_add(&tccd_oracle_level_hist[63 - __builtin_clzll((unsigned long long)ncur)],
                       ncur, __ATOMIC_RELAXED);
    for (int64_t i = 0; i < ncur; ++i) ar->keys[i] = cur[i].t0;
    stable_order(ar->keys, ncur, ar->ord, ar->tmp);
    for (int64_t oi = 0; oi < ncur; ++oi) {
      box_t b = cur[ar->ord[oi]];
      double wb;
      int cls = classify(s, e, kind, &b, eps, sep, &wb);
      checks += 1;
      if (cls == CLS_DISJOINT) {
        if (checks >= max_checks && (have_drop || oi + 1 < ncur || nnxt > 0)) {
          if (have_drop && (!have_first || db.t0 < fb.t0))
            set_result(r, &db, d_codom, checks, 1, d_level);
          else
            set_result(r, &fb, f_codom, checks, 1, f_level);
          return 0;
        }
        continue;
      }
      if (level != last_col) {
        have_first = 1;
        fb = b;
        f_level = level;
        f_codom = wb;
      }
      if (checks >= max_checks) {
        if (have_drop && db.t0 < fb.t0) set_result(r, &db, d_codom, checks, 1, d_level);
        else set_result(r, &fb, f_codom, checks, 1, f_level);
        return 0;
      }
      int accept = wb < delta || cls == CLS_CONTAINED;
      int sdim = -1;
      double mid = 0.0;
      if (!accept) {
        double ct = (b.t1 - b.t0) * kap[0];
        double cu = (b.u1 - b.u0) * kap[1];
        double cv = (b.v1 - b.v0) * kap[2];
        double best = ct;
        sdim = 0;
        if (cu > best) { sdim = 1; best = cu; }
        if (cv > best) { sdim = 2; best = cv; }
        double lo = sdim == 0 ? b.t0 : (sdim == 1 ? b.u0 : b.v0);
        double hi = sdim == 0 ? b.t1 : (sdim == 1 ? b.u1 : b.v1);
        mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) accept = 1;
      }
      if (accept) {
        if (level != last_col) {
          if (have_drop && db.t0 < b.t0) set_result(r, &db, d_codom, checks, 0, d_level);
          else set_result(r, &b, wb, checks, 0, level);
          return 0;
        }
        if (!have_drop || b.t0 < db.t0) {
          db = b;
          d_level = level;
          d_codom = wb;
        }
        have_drop = 1;
      } else {
        if (arena_reserve(ar, nnxt + 2)) return -1;
        cur = ar->cur; /* realloc may move both buffers (cur not read below) */
        nxt = ar->nxt;
        box_t lo = b, hi = b;
        int push_hi = 1;
        if (sdim == 0) { lo.t1 = mid; hi.t0 = mid; }
        else if (sdim == 1) { lo.u1 = mid; hi.u0 = mid; push_hi = kind != 0 || mid + b.v0 <= 1.0; }
        else { lo.v1 = mid; hi.v0 = mid; push_hi = kind != 0 || b.u0 + mid <= 1.0; }
        nxt[nnxt++] = lo;
        if (push_hi) nxt[nnxt++] = hi;
      }
      last_col = level;
    }
    box_t *t = ar->cur; ar->cur = ar->nxt; ar->nxt = t;
    cur = ar->cur; nxt = ar->nxt;
    ncur = nnxt;
    nnxt = 0;
    level += 1;
  }
  if (have_drop) {
    set_result(r, &db, d_codom, checks, 0, d_level);
    return 0;
  }
  memset(r, 0, sizeof(*r));
  r->status = ST_FREE;
  r->toi = INFINITY;
  r->checks = checks;
  return 0;
}

/* Direct restatement of solve_kernel's signature (_kernel.py:136):
 * s, e: [4][3]; out13 receives (status, toi, tol, codom, checks, early,
 * w_t0, w_t1, w_u0, w_u1, w_v0, w_v1, w_level) as doubles. */
int tccd_oracle_solve_kernel(const double *s, const double *e, int kind,
                             double t_max, double delta, int64_t max_checks,
                             double sep, double ex, double ey, double ez,
                             double *out13) {
  arena_t ar = {0};
  result_t r;
  double eps[3] = {ex, ey, ez};
  int rc = solve_one(s, e, kind, t_max, delta, max_checks, sep, eps, &ar, &r);
  arena_free(&ar);
  if (rc) return rc;
  out13[0] = r.status; out13[1] = r.toi; out13[2] = r.tol; out13[3] = r.codom;
  out13[4] = (double)r.checks; out13[5] = r.early;
  for (int k = 0; k < 6; ++k) out13[6 + k] = r.w[k];
  out13[12] = r.level;
  return 0;
}

/* ---------------------------------------------------------------------
 * Batched driver (host threads).  Layout mirrors include/tccd.h:
 * points [n][8][3]; per-query arrays may be NULL (use the *_all scalar).
 * eps: NULL -> per-query compute_gamma/compute_filters, else [n][3].
 * ------------------------------------------------------------------- */
typedef struct {
  int64_t n;
  const double *points;
  const uint8_t *kind;
  int kind_all;
  const double *delta;
  double delta_all;
  const int64_t *max_checks;
  int64_t max_checks_all;
  const double *sep;
  double sep_all;
  const double *t_max;
  double t_max_all;
  const double *eps;
  uint8_t *status;
  double *toi, *tol, *codom;
  int64_t *checks;
  uint8_t *early;
  double *witness;
  int32_t *level;
  int64_t *frontier; /* optional diagnostics [n][2]: widest level, levels */
  /* work distribution */
  int64_t next;
  int64_t chunk;
  pthread_mutex_t mu;
  int failed;
} batch_t;

static void solve_index(batch_t *B, int64_t q, arena_t *ar) {
  const double *pts = B->points + 24 * q;
  int kind = B->kind ? B->kind[q] : B->kind_all;
  double delta = B->delta ? B->delta[q] : B->delta_all;
  int64_t mc = B->max_checks ? B->max_checks[q] : B->max_checks_all;
  double sep = B->sep ? B->sep[q] : B->sep_all;
  double tm = B->t_max ? B->t_max[q] : B->t_max_all;
  result_t r;
  memset(&r, 0, sizeof(r));
  int st = ST_HIT;
  if (!(delta > 0.0 && isfinite(delta)) || mc < 1 || !(sep >= 0.0 && isfinite(sep)) ||
      !(tm > 0.0 && tm <= 1.0) || (kind != 0 && kind != 1))
    st = ST_ERR_PARAM;
  double eps[3];
  if (st == ST_HIT) {
    if (B->eps) {
      for (int i = 0; i < 24; ++i)
        if (!isfinite(pts[i])) st = ST_ERR_NONFINITE;
      eps[0] = B->eps[3 * q]; eps[1] = B->eps[3 * q + 1]; eps[2] = B->eps[3 * q + 2];
    } else {
      st = tccd_oracle_filters(pts, kind, sep, eps);
    }
  }
  if (st == ST_HIT) {
    if (solve_one(pts, pts + 12, kind, tm, delta, mc, sep, eps, ar, &r)) {
      B->failed = 1;
      return;
    }
  } else {
    r.status = st;
    r.toi = INFINITY;
  }
  B->status[q] = (uint8_t)r.status;
  B->toi[q] = r.toi;
  if (B->tol) B->tol[q] = r.tol;
  if (B->codom) B->codom[q] = r.codom;
  if (B->checks) B->checks[q] = r.checks;
  if (B->early) B->early[q] = (uint8_t)r.early;
  if (B->witness) memcpy(B->witness + 6 * q, r.w, 6 * sizeof(double));
  if (B->level) B->level[q] = r.level;
  if (B->frontier) {
    B->frontier[2 * q] = st == ST_HIT ? ar->max_frontier : 0;
    B->frontier[2 * q + 1] = st == ST_HIT ? ar->levels : 0;
  }
}

static void *worker(void *arg) {
  batch_t *B = arg;
  arena_t ar = {0};
  for (;;) {
    int64_t lo = __atomic_fetch_add(&B->next, B->chunk, __ATOMIC_RELAXED);
    if (lo >= B->n || B->failed) break;
    int64_t hi = lo + B->chunk < B->n ? lo + B->chunk : B->n;
    for (int64_t q = lo; q < hi; ++q) solve_index(B, q, &ar);
  }
  arena_free(&ar);
  return NULL;
}

int tccd_oracle_solve_batch(int64_t n, const double *points, const uint8_t *kind,
                            int kind_all, const double *delta, double delta_all,
                            const int64_t *max_checks, int64_t max_checks_all,
                            const double *sep, double sep_all, const double *t_max,
                            double t_max_all, const double *eps, uint8_t *status,
                            double *toi, double *tol, double *codom, int64_t *checks,
                            uint8_t *early, double *witness, int32_t *level,
                            int64_t *frontier, int threads) {
  batch_t B;
  memset(&B, 0, sizeof(B));
  B.n = n; B.points = points; B.kind = kind; B.kind_all = kind_all;
  B.delta = delta; B.delta_all = delta_all; B.max_checks = max_checks;
  B.max_checks_all = max_checks_all; B.sep = sep; B.sep_all = sep_all;
  B.t_max = t_max; B.t_max_all = t_max_all; B.eps = eps; B.status = status;
  B.toi = toi; B.tol = tol; B.codom = codom; B.checks = checks; B.early = early;
  B.witness = witness; B.level = level; B.frontier = frontier;
  B.chunk = 16;
  if (threads < 1) threads = 1;
  if (threads == 1) {
    worker(&B);
    return B.failed ? -1 : 0;
  }
  pthread_t *tid = calloc((size_t)threads, sizeof(pthread_t));
  if (!tid) return -1;
  int started = 0;
  for (int i = 0; i < threads; ++i)
    if (pthread_create(&tid[i], NULL, worker, &B) == 0) started++;
    else break;
  if (started == 0) worker(&B);
  for (int i = 0; i < started; ++i) pthread_join(tid[i], NULL);
  free(tid);
  return B.failed ? -1 : 0;
}
