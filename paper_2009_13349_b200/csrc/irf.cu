// IRF baseline on the GPU: the reference's interval
// root finder ccdkit.baselines.irf_solve (pkg/src/ccdkit/baselines.py:123-206)
// for a batch of queries, bit-identical to it.
//
// The method is a best-first search: boxes wait in a min-heap keyed by
// (t_lo, level, push sequence) (:144, :202), every interval operation is
// widened one representable step outward (IntervalScalar, :37-106), and the
// first accepted box (F's enclosure contains 0 on every axis and every
// domain side < delta) or the first box popped once the budget is spent is
// the answer.  The pop order decides toi, witness and checks.
//
// Pass 1: one thread per query (queries fetched dynamically), its heap an
// 8-ary heap in a global arena (see Heap), 2048 entries.  A heap can hold at
// most checks + 1 boxes; queries whose heap outgrows that are re-run from
// the root (exact: the search is deterministic) by
// Pass 2: a warp per query over RUNS.  Boxes with equal (t_lo, level) pop
// consecutively in push order: every child has level + 1, so no child of a
// run can pop before the rest of the run.  A run is therefore evaluated 32
// boxes at a time (lane per box) and its outcome replayed in order (the
// first budget index or accepted box ends the search).  Its children go to
// new runs: all lower children and the upper children of u / v splits keep
// t_lo (one run, contiguous in push order); the upper children of t splits
// form runs per distinct midpoint.  Runs live in an 8-ary heap keyed by
// (t_lo, level, creation order): two runs with the same (t_lo, level) come
// from different parent runs and pop in creation order, which is their push
// order.  Boxes are bump-allocated, lower/u/v children upward and t-split
// upper children downward, so each run is one contiguous (possibly
// descending) segment.  A query whose run heap fills up goes to
// Pass 3: pass 1's thread-per-query search with max_checks + 2 heap entries.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstring>

#include "tccd.h"

namespace tccd_irf {

struct Iv {
  double lo, hi;
};

// nextafter(x, -inf) / nextafter(x, +inf) (IEEE, as math.nextafter): one
// step in the bit pattern; +-0 go to -+denorm_min, infinities saturate
__device__ __forceinline__ double next_down(double x) {
  if (isnan(x) || x == -INFINITY) return x;
  if (x == 0.0) return -4.9406564584124654e-324;
  const long long b = __double_as_longlong(x);
  return __longlong_as_double(x > 0.0 ? b - 1 : b + 1);
}
__device__ __forceinline__ double next_up(double x) {
  if (isnan(x) || x == INFINITY) return x;
  if (x == 0.0) return 4.9406564584124654e-324;
  const long long b = __double_as_longlong(x);
  return __longlong_as_double(x > 0.0 ? b + 1 : b - 1);
}

// IntervalScalar._outward (:56-61)
__device__ __forceinline__ Iv outward(double lo, double hi) { return Iv{next_down(lo), next_up(hi)}; }
__device__ __forceinline__ Iv pt(double x) { return Iv{x, x}; }                     // _coerce
__device__ __forceinline__ Iv add(Iv a, Iv b) { return outward(a.lo + b.lo, a.hi + b.hi); }
__device__ __forceinline__ Iv sub(Iv a, Iv b) { return outward(a.lo - b.hi, a.hi - b.lo); }
// :81-87, Python min / max: a later product replaces only if strictly smaller / larger
__device__ __forceinline__ Iv mul(Iv a, Iv b) {
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

// _interval_F (:109-120) on one axis
__device__ __forceinline__ Iv interval_F(const double* P, int kind, int ax, Iv t, Iv u, Iv v) {
  Iv p[4];
  const Iv omt = sub(pt(1.0), t);
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j] = add(mul(omt, pt(P[3 * j + ax])), mul(t, pt(P[12 + 3 * j + ax])));
  if (kind == 0) {
    const Iv w = sub(sub(pt(1.0), u), v);
    return sub(p[0], add(add(mul(w, p[1]), mul(u, p[2])), mul(v, p[3])));
  }
  const Iv l = add(mul(sub(pt(1.0), u), p[0]), mul(u, p[1]));
  const Iv r = add(mul(sub(pt(1.0), v), p[2]), mul(v, p[3]));
  return sub(l, r);
}

struct Args {
  long long n;
  const double* points;
  const uint8_t* kind;
  int kind_all;
  const double* delta;
  double delta_all;
  const long long* max_checks;
  long long max_checks_all;
  const double* t_max;
  double t_max_all;
  uint8_t* status;
  double* toi;
  double* tol;
  double* codom;
  long long* checks;
  uint8_t* early;
  double* witness;
  int* level;
};

struct Ctr {
  unsigned long long next[3];  // next query of pass 1 / overflow entry (pass 2) / fallback (pass 3)
  unsigned long long overflow; // queries handed to pass 2
  unsigned long long fallback; // queries handed from pass 2 to pass 3
};

// The heap of one thread: an 8-ary min-heap of 16-byte keys (t_lo, then
// level << 48 | seq: the tuple order of :144/:202, level < 2^16 and seq <
// 2^48) with the boxes in a parallel array.  The 8 children of a node are
// one 128-byte line, so a pop costs ~log8(n) dependent loads.
struct Key {
  double tl;
  unsigned long long ls;  // level << 48 | seq
};

__device__ __forceinline__ bool key_less(const Key& a, const Key& b) {
  return a.tl < b.tl || (a.tl == b.tl && a.ls < b.ls);  // t_lo is never NaN
}

struct Heap {
  Key* key;     // [cap]
  double2* box; // [cap][3]: (tl, th), (ul, uh), (vl, vh)
  long long cap, n;
  __device__ __forceinline__ void load_box(long long i, double b[6]) const {
    const double2 x = box[3 * i], y = box[3 * i + 1], z = box[3 * i + 2];
    b[0] = x.x; b[1] = x.y; b[2] = y.x; b[3] = y.y; b[4] = z.x; b[5] = z.y;
  }
  __device__ __forceinline__ void store_box(long long i, const double b[6]) {
    box[3 * i] = make_double2(b[0], b[1]);
    box[3 * i + 1] = make_double2(b[2], b[3]);
    box[3 * i + 2] = make_double2(b[4], b[5]);
  }
  __device__ __forceinline__ void move(long long dst, long long src) {
    key[dst] = key[src];
    box[3 * dst] = box[3 * src];
    box[3 * dst + 1] = box[3 * src + 1];
    box[3 * dst + 2] = box[3 * src + 2];
  }
  __device__ void push(const double b[6], unsigned long long ls) {
    const Key k{b[0], ls};
    long long i = n++;
    while (i > 0) {
      const long long p = (i - 1) >> 3;
      const Key kp = key[p];
      if (!key_less(k, kp)) break;
      move(i, p);
      i = p;
    }
    key[i] = k;
    store_box(i, b);
  }
  __device__ __forceinline__ void top(double b[6], unsigned long long& ls) const {
    ls = key[0].ls;
    load_box(0, b);
  }
  // put (k, b) at the root's place and sift it down
  __device__ void sift_down_from_root(const Key& k, const double b[6]) {
    long long i = 0;
    for (;;) {
      const long long c0 = 8 * i + 1;
      if (c0 >= n) break;
      const long long cend = c0 + 8 < n ? c0 + 8 : n;
      long long c = c0;
      Key kc = key[c0];
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        if (c0 + j < cend) {
          const Key kj = key[c0 + j];
          if (key_less(kj, kc)) { kc = kj; c = c0 + j; }
        }
      }
      if (!key_less(kc, k)) break;
      move(i, c);
      i = c;
    }
    key[i] = k;
    store_box(i, b);
  }
  __device__ void pop_discard() {  // remove the root
    if (--n == 0) return;
    const Key last = key[n];
    double lb[6];
    load_box(n, lb);
    sift_down_from_root(last, lb);
  }
  // replace the root by (b, ls): a popped box's first child usually sinks
  // only a level or two, where pop + push would sift it up the whole path
  __device__ void replace_top(const double b[6], unsigned long long ls) {
    sift_down_from_root(Key{b[0], ls}, b);
  }
};

// One query; returns false if the heap outgrew its capacity (re-run later).
// check_cap: pass 1 gives up on a query after this many checks (a long
// best-first search is far faster as a warp's run search, pass 2); the
// fallback pass 3 runs without it
__device__ bool irf_query(const Args& a, long long q, Heap& H, long long check_cap) {
  double P[24];
  bool finite = true;
#pragma unroll
  for (int k = 0; k < 24; ++k) {
    P[k] = a.points[24 * q + k];
    finite &= isfinite(P[k]);
  }
  const int kind = a.kind ? a.kind[q] : a.kind_all;
  const double delta = a.delta ? a.delta[q] : a.delta_all;
  const long long mc = a.max_checks ? a.max_checks[q] : a.max_checks_all;
  const double t_max = a.t_max ? a.t_max[q] : a.t_max_all;
  uint8_t st = 0;
  double toi = INFINITY, tol = 0.0, cw = 0.0, w[6] = {0, 0, 0, 0, 0, 0};
  long long checks = 0;
  int early = 0, level = 0;
  if (!finite) st = TCCD_STATUS_ERR_NONFINITE;
  else if (!(delta > 0.0) || !(isfinite(t_max) && t_max >= 0.0) || (kind != 0 && kind != 1))
    st = TCCD_STATUS_ERR_PARAM;  // ValueError (:139-140, IntervalScalar :53-54)
  if (st == 0) {
    H.n = 0;
    const double root[6] = {0.0, t_max, 0.0, 1.0, 0.0, 1.0};
    H.push(root, 0ull);
    unsigned long long seq = 0;
    while (H.n > 0) {
      double b[6];
      unsigned long long ls;
      H.top(b, ls);  // popped below, or replaced by its first child
      const long long lv = (long long)(ls >> 48);
      const Iv t{b[0], b[1]}, u{b[2], b[3]}, v{b[4], b[5]};
      const bool budget = checks >= mc;  // :147-165
      bool all = true;
      double fw = 0.0;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const Iv F = interval_F(P, kind, ax, t, u, v);
        all = all && F.lo <= 0.0 && 0.0 <= F.hi;
        const double wd = F.hi - F.lo;  // max(ax.width for ax in F)
        if (ax == 0 || wd > fw) fw = wd;
        if (!all && !budget) break;     // (no later axis is observable then)
      }
      if (budget) {
        st = 1; early = 1; toi = b[0]; tol = b[1] - b[0]; cw = fw; level = (int)lv;
        for (int k = 0; k < 6; ++k) w[k] = b[k];
        break;
      }
      ++checks;
      if (checks > check_cap) return false;  // (re-run from the root by pass 2)
      if (!all) {
        H.pop_discard();
        continue;
      }
      const double wt = b[1] - b[0], wu = b[3] - b[2], wv = b[5] - b[4];
      double mw = wt;
      int dim = 0;  // np.argmax: first maximum
      if (wu > mw) { mw = wu; dim = 1; }
      if (wv > mw) { mw = wv; dim = 2; }
      if (mw < delta) {  // :175-185
        st = 1; toi = b[0]; tol = b[1] - b[0]; cw = fw; level = (int)lv;
        for (int k = 0; k < 6; ++k) w[k] = b[k];
        break;
      }
      // (selects, not b[2 * dim]: a dynamic index would put the box in local memory)
      const double lo_d = dim == 0 ? b[0] : (dim == 1 ? b[2] : b[4]);
      const double hi_d = dim == 0 ? b[1] : (dim == 1 ? b[3] : b[5]);
      const double m = 0.5 * (lo_d + hi_d);
      double k0[6], k1[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        k0[k] = (k == 2 * dim + 1) ? m : b[k];
        k1[k] = (k == 2 * dim) ? m : b[k];
      }
      const bool keep0 = !(kind == 0 && k0[2] + k0[4] > 1.0);  // :197-199
      const bool keep1 = !(kind == 0 && k1[2] + k1[4] > 1.0);
      if (H.n - 1 + (keep0 ? 1 : 0) + (keep1 ? 1 : 0) > H.cap) return false;
      // (level <= 3 * 1075: each split halves one side of a binary64 box)
      const unsigned long long lv1 = (unsigned long long)(lv + 1) << 48;
      if (keep0 && keep1) {
        const unsigned long long s0 = lv1 | ++seq, s1 = lv1 | ++seq;
        H.replace_top(k0, s0);
        H.push(k1, s1);
      } else if (keep0 || keep1) {
        H.replace_top(keep0 ? k0 : k1, lv1 | ++seq);
      } else {
        H.pop_discard();
      }
    }
  }
  a.status[q] = st;
  a.toi[q] = toi;
  if (a.tol) a.tol[q] = tol;
  if (a.codom) a.codom[q] = cw;
  if (a.checks) a.checks[q] = checks;
  if (a.early) a.early[q] = (uint8_t)early;
  if (a.witness)
    for (int k = 0; k < 6; ++k) a.witness[6 * q + k] = w[k];
  if (a.level) a.level[q] = level;
  return true;
}

// ---------------------------------------------------------------------------
// pass 2: a warp per query over runs (see the header)

struct REnt {                // a run in the run heap
  double tl;                 // t_lo of its boxes
  unsigned long long ls;     // level << 48 | creation order
  int off, cnt;              // boxes off, off + 1, ... (cnt > 0) or off, off - 1, ... (cnt < 0)
  long long pad;
};

struct RunHeap {             // 8-ary min-heap on (tl, ls); lane 0 only
  REnt* e;
  long long cap, n;
  __device__ void push(const REnt& x) {
    long long i = n++;
    const Key k{x.tl, x.ls};
    while (i > 0) {
      const long long p = (i - 1) >> 3;
      if (!key_less(k, Key{e[p].tl, e[p].ls})) break;
      e[i] = e[p];
      i = p;
    }
    e[i] = x;
  }
  __device__ REnt pop() {
    const REnt top = e[0];
    if (--n > 0) {
      const REnt last = e[n];
      const Key kl{last.tl, last.ls};
      long long i = 0;
      for (;;) {
        const long long c0 = 8 * i + 1;
        if (c0 >= n) break;
        const long long cend = c0 + 8 < n ? c0 + 8 : n;
        long long c = c0;
        Key kc{e[c0].tl, e[c0].ls};
        for (long long j = c0 + 1; j < cend; ++j) {
          const Key kj{e[j].tl, e[j].ls};
          if (key_less(kj, kc)) { kc = kj; c = j; }
        }
        if (!key_less(kc, kl)) break;
        e[i] = e[c];
        i = c;
      }
      e[i] = last;
    }
    return top;
  }
};

constexpr int kWarps2 = 4;  // warps per block in pass 2
constexpr int kFront = 8;   // runs kept in shared memory in front of the run heap

// The run heap with a small front buffer in shared memory (lane 0 only).  A
// best-first dive pushes one or two runs per step and pops one of them next:
// those stay in the buffer, and the global heap (a chain of dependent loads
// per operation) is touched only when the buffer overflows (its largest run
// moves to the heap) or the heap's top (cached) is smaller than every
// buffered run.  Keys are unique, so the pop order is the heap's.
struct FrontRuns {
  REnt* buf;
  int nb;
  RunHeap* H;
  Key top;  // H->e[0]'s key while H->n > 0
  __device__ long long size() const { return nb + H->n; }
  __device__ void refresh() {
    if (H->n) top = Key{H->e[0].tl, H->e[0].ls};
  }
  __device__ void push(const REnt& x) {
    if (nb < kFront) { buf[nb++] = x; return; }
    int mi = -1;  // the largest of the buffer and x goes to the heap
    Key mk{x.tl, x.ls};
    for (int j = 0; j < kFront; ++j) {
      const Key kj{buf[j].tl, buf[j].ls};
      if (key_less(mk, kj)) { mk = kj; mi = j; }
    }
    if (mi < 0) {
      H->push(x);
    } else {
      const REnt y = buf[mi];
      buf[mi] = x;
      H->push(y);
    }
    refresh();
  }
  __device__ REnt pop() {  // size() > 0
    int bi = -1;
    Key bk{0.0, 0ull};
    for (int j = 0; j < nb; ++j) {
      const Key kj{buf[j].tl, buf[j].ls};
      if (bi < 0 || key_less(kj, bk)) { bk = kj; bi = j; }
    }
    if (bi >= 0 && (H->n == 0 || key_less(bk, top))) {
      const REnt r = buf[bi];
      buf[bi] = buf[--nb];
      return r;
    }
    const REnt r = H->pop();
    refresh();
    return r;
  }
};

__device__ __forceinline__ void write_irf_result(const Args& a, long long q, uint8_t st,
                                                 const double b[6], double cw, long long checks,
                                                 int early, int level) {
  a.status[q] = st;
  a.toi[q] = st == 1 ? b[0] : INFINITY;
  if (a.tol) a.tol[q] = st == 1 ? b[1] - b[0] : 0.0;
  if (a.codom) a.codom[q] = st == 1 ? cw : 0.0;
  if (a.checks) a.checks[q] = checks;
  if (a.early) a.early[q] = (uint8_t)early;
  if (a.witness)
    for (int k = 0; k < 6; ++k) a.witness[6 * q + k] = st == 1 ? b[k] : 0.0;
  if (a.level) a.level[q] = st == 1 ? level : 0;
}

// One query by one warp; returns false if its run heap filled up (pass 3).
__device__ bool irf_warp_query(const Args& a, long long q, double2* box, long long bcap,
                               RunHeap& H, double* Psm, REnt* front) {
  const int lane = threadIdx.x & 31;
  bool finite = true;
  if (lane < 24) {
    const double x = a.points[24 * q + lane];
    Psm[lane] = x;
    finite = isfinite(x);
  }
  finite = __all_sync(0xffffffffu, finite);
  __syncwarp();
  const int kind = a.kind ? a.kind[q] : a.kind_all;
  const double delta = a.delta ? a.delta[q] : a.delta_all;
  const long long mc = a.max_checks ? a.max_checks[q] : a.max_checks_all;
  const double t_max = a.t_max ? a.t_max[q] : a.t_max_all;
  const double zero6[6] = {0, 0, 0, 0, 0, 0};
  uint8_t st = 0;
  if (!finite) st = TCCD_STATUS_ERR_NONFINITE;
  else if (!(delta > 0.0) || !(isfinite(t_max) && t_max >= 0.0) || (kind != 0 && kind != 1))
    st = TCCD_STATUS_ERR_PARAM;
  if (st != 0) {
    if (lane == 0) write_irf_result(a, q, st, zero6, 0.0, 0, 0, 0);
    return true;
  }
  auto ldbox = [&](long long i, double b[6]) {
    const double2 x = box[3 * i], y = box[3 * i + 1], z = box[3 * i + 2];
    b[0] = x.x; b[1] = x.y; b[2] = y.x; b[3] = y.y; b[4] = z.x; b[5] = z.y;
  };
  auto stbox = [&](long long i, const double b[6]) {
    box[3 * i] = make_double2(b[0], b[1]);
    box[3 * i + 1] = make_double2(b[2], b[3]);
    box[3 * i + 2] = make_double2(b[4], b[5]);
  };
  FrontRuns F;  // (lane 0's)
  F.buf = front;
  F.nb = 0;
  F.H = &H;
  if (lane == 0) {
    const double root[6] = {0.0, t_max, 0.0, 1.0, 0.0, 1.0};
    stbox(0, root);
    H.n = 0;
    F.push(REnt{0.0, 0ull, 0, 1, 0});
  }
  long long lo_top = 1, hi_top = bcap - 1;  // next free box upward / downward
  unsigned long long cseq = 1;              // run creation order
  long long C = 0;                          // checks before the current run
  for (;;) {
    REnt r;
    int empty = 0;
    if (lane == 0) {
      if (F.size() == 0) empty = 1;
      else r = F.pop();
    }
    if (__shfl_sync(0xffffffffu, empty, 0)) {
      if (lane == 0) write_irf_result(a, q, 0, zero6, 0.0, C, 0, 0);
      return true;
    }
    r.tl = __shfl_sync(0xffffffffu, r.tl, 0);
    r.ls = __shfl_sync(0xffffffffu, r.ls, 0);
    r.off = __shfl_sync(0xffffffffu, r.off, 0);
    r.cnt = __shfl_sync(0xffffffffu, r.cnt, 0);
    const long long lv = (long long)(r.ls >> 48);
    const unsigned long long lv1 = (unsigned long long)(lv + 1) << 48;
    const int nrun = r.cnt > 0 ? r.cnt : -r.cnt;
    const int dir = r.cnt > 0 ? 1 : -1;
    const long long main_off = lo_top;
    long long main_cnt = 0;
    bool up_open = false;
    double up_key = 0.0;
    long long up_start = 0, up_cnt = 0;
    bool full = false;
    for (int base = 0; base < nrun; base += 32) {
      const int idx = base + lane;
      const bool valid = idx < nrun;
      double b[6];
      if (valid) ldbox((long long)r.off + (long long)dir * idx, b);
      else for (int k = 0; k < 6; ++k) b[k] = 0.0;
      const bool budget = valid && C + idx >= mc;  // :147-165
      bool all = valid;
      double fw = 0.0;
      if (valid) {
        const Iv t{b[0], b[1]}, u{b[2], b[3]}, v{b[4], b[5]};
#pragma unroll 1
        for (int ax = 0; ax < 3; ++ax) {
          const Iv F = interval_F(Psm, kind, ax, t, u, v);
          all = all && F.lo <= 0.0 && 0.0 <= F.hi;
          const double wd = F.hi - F.lo;
          if (ax == 0 || wd > fw) fw = wd;
          if (!all && !budget) break;
        }
      }
      const double wt = b[1] - b[0], wu = b[3] - b[2], wv = b[5] - b[4];
      double mw = wt;
      int dim = 0;
      if (wu > mw) { mw = wu; dim = 1; }
      if (wv > mw) { mw = wv; dim = 2; }
      const bool hit = valid && !budget && all && mw < delta;  // :175-185
      const unsigned int ev = __ballot_sync(0xffffffffu, budget || hit);
      if (ev) {
        const int f = __ffs(ev) - 1;  // the first event in push order ends the search
        if (lane == f) {
          if (budget) write_irf_result(a, q, 1, b, fw, C + idx, 1, (int)lv);
          else write_irf_result(a, q, 1, b, fw, C + idx + 1, 0, (int)lv);
        }
        return true;
      }
      const bool split = valid && all;
      const double lo_d = dim == 0 ? b[0] : (dim == 1 ? b[2] : b[4]);
      const double hi_d = dim == 0 ? b[1] : (dim == 1 ? b[3] : b[5]);
      const double m = 0.5 * (lo_d + hi_d);
      double k0[6], k1[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        k0[k] = (k == 2 * dim + 1) ? m : b[k];
        k1[k] = (k == 2 * dim) ? m : b[k];
      }
      const bool keep0 = split && !(kind == 0 && k0[2] + k0[4] > 1.0);  // :197-199
      const bool keep1 = split && !(kind == 0 && k1[2] + k1[4] > 1.0);
      // lower children and u / v upper children: the run (t_lo, level + 1)
      const int nm = (keep0 ? 1 : 0) + (keep1 && dim != 0 ? 1 : 0);
      int pm = nm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, pm, o);
        if (lane >= o) pm += y;
      }
      const int tot_m = __shfl_sync(0xffffffffu, pm, 31);
      pm -= nm;
      {
        long long pos = main_off + main_cnt + pm;
        if (keep0) stbox(pos++, k0);
        if (keep1 && dim != 0) stbox(pos, k1);
      }
      main_cnt += tot_m;
      // t-split upper children: one run per distinct midpoint, in lane order
      const bool up = keep1 && dim == 0;
      // (a midpoint equal to t_lo, only possible at binary64 resolution, would
      // interleave two runs of one key: pass 3 handles such a query)
      if (__any_sync(0xffffffffu, up && m == r.tl)) return false;
      unsigned int um = __ballot_sync(0xffffffffu, up);
      while (um) {
        const int lead = __ffs(um) - 1;
        const double K = __shfl_sync(0xffffffffu, m, lead);
        const unsigned int grp = __ballot_sync(0xffffffffu, up && m == K) & um;
        if (!up_open || K != up_key) {
          if (up_open && up_cnt > 0) {
            if (lane == 0) {
              if (H.n >= H.cap) full = true;
              else F.push(REnt{up_key, lv1 | cseq, (int)up_start, -(int)up_cnt, 0});
            }
            ++cseq;
            hi_top = up_start - up_cnt;
          }
          up_open = true;
          up_key = K;
          up_start = hi_top;
          up_cnt = 0;
        }
        if ((grp >> lane) & 1u) stbox(up_start - (up_cnt + __popc(grp & ((1u << lane) - 1u))), k1);
        up_cnt += __popc(grp);
        um &= ~grp;
      }
    }
    C += nrun;
    if (lane == 0) {
      if (main_cnt > 0) {
        if (H.n >= H.cap) full = true;
        else F.push(REnt{r.tl, lv1 | cseq, (int)main_off, (int)main_cnt, 0});
      }
      if (up_open && up_cnt > 0) {
        if (H.n >= H.cap) full = true;
        else F.push(REnt{up_key, lv1 | (cseq + 1), (int)up_start, -(int)up_cnt, 0});
      }
    }
    cseq += 2;
    lo_top += main_cnt;
    if (up_open) hi_top = up_start - up_cnt;
    if (__shfl_sync(0xffffffffu, full ? 1 : 0, 0)) return false;
  }
}

__global__ void __launch_bounds__(32 * kWarps2) irf_warp_kernel(Args a, Ctr* ctr,
                                                                unsigned char* arena,
                                                                long long bcap, long long hcap,
                                                                const long long* list,
                                                                long long* fallback) {
  __shared__ double Psm[kWarps2][24];
  __shared__ REnt front[kWarps2][kFront];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long slot = (long long)blockIdx.x * kWarps2 + w;
  unsigned char* mine = arena + slot * (bcap * 48 + hcap * (long long)sizeof(REnt));
  double2* box = (double2*)mine;
  RunHeap H;
  H.e = (REnt*)(mine + bcap * 48);
  H.cap = hcap;
  H.n = 0;
  const unsigned long long total = ctr->overflow;
  for (;;) {
    unsigned long long i = 0;
    if (lane == 0) i = atomicAdd(&ctr->next[1], 1ull);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= total) break;
    const long long q = list[i];
    if (!irf_warp_query(a, q, box, bcap, H, Psm[w], front[w]) && lane == 0)
      fallback[atomicAdd(&ctr->fallback, 1ull)] = q;
  }
}

// pass 0: every query (index list = identity); pass 2: pass 2's fallback list.
// Per thread: cap keys (16 B) then cap boxes (48 B), contiguous.
#ifndef TCCD_IRF_PASS1_CHECKS
#define TCCD_IRF_PASS1_CHECKS (1LL << 9)
#endif
constexpr long long kPass1Checks = TCCD_IRF_PASS1_CHECKS;  // pass 1's check cap (see irf_query)

__global__ void __launch_bounds__(128) irf_kernel(Args a, Ctr* ctr, unsigned char* arena,
                                                  long long cap, const long long* list,
                                                  long long* overflow, int pass, int has_pass2) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  Heap H;
  unsigned char* mine = arena + tid * cap * 64;
  H.key = (Key*)mine;
  H.box = (double2*)(mine + cap * 16);
  H.cap = cap;
  H.n = 0;
  const unsigned long long total = pass == 0 ? (unsigned long long)a.n : ctr->fallback;
  for (;;) {
    const unsigned long long i = atomicAdd(&ctr->next[pass], 1ull);
    if (i >= total) break;
    const long long q = pass == 0 ? (long long)i : list[i];
    if (!irf_query(a, q, H, pass == 0 && has_pass2 ? kPass1Checks : LLONG_MAX)) {
      if (pass == 0) overflow[atomicAdd(&ctr->overflow, 1ull)] = q;
      else a.status[q] = 0xFF;  // unreachable: a heap never exceeds checks + 1 <= cap - 1
    }
  }
}

// no pass-2 warp fits: pass 3 reads the overflow list directly
__global__ void irf_fill_fallback(Ctr* ctr) {
  if (threadIdx.x == 0) ctr->fallback = ctr->overflow;
}

// heavy_only: every query goes to pass 2
__global__ void irf_fill_all(long long n, long long* list, Ctr* ctr) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) list[i] = i;
  if (i == 0) ctr->overflow = (unsigned long long)n;
}

}  // namespace tccd_irf

using namespace tccd_irf;

namespace {

constexpr long long kCap1 = 2048;  // heap entries per thread in pass 1
constexpr int kThreads = 128;

size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

struct IrfLayout {
  size_t ctr, overflow, fallback, arena1, arena2, total;
  long long threads1, slots3, cap3, warps2, bcap2, hcap2;
};

int resident_blocks() {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, irf_kernel, kThreads, 0) != cudaSuccess ||
      nb < 1)
    nb = 2;
  return nb;
}

// Pass 2 (warp per query over runs): 2 * (max_checks + 2) boxes (every push
// of a search, never reclaimed) and a run heap per warp, as many warps as
// half of the device memory holds (8 per SM at most): pass 2 carries every
// long search, and its throughput scales with its warp count (a quarter of
// the memory ran config 1's 10^5 queries in 3.4 s, half in 1.9 s).  Pass 3 (the
// fallback): slots3 <= 0 picks as many max_checks + 2-entry heaps as an
// eighth of the memory holds (4096 at most).  Passes 2 and 3 run one after
// the other and share their arena.
IrfLayout irf_layout(long long n, long long mcmax, int slots3, int sms) {
  IrfLayout L;
  L.threads1 = (long long)sms * resident_blocks() * kThreads;
  L.cap3 = (mcmax > 0 ? mcmax : 0) + 2;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) tot = (size_t)16 << 30;
  long long s3 = slots3;
  if (s3 <= 0) {
    s3 = (long long)(tot / 8 / ((size_t)L.cap3 * 64));
    if (s3 > 4096) s3 = 4096;
    if (s3 < sms) s3 = sms;
    if (s3 > n) s3 = n > 0 ? n : 1;  // (no more slots than queries)
  }
  L.slots3 = (s3 + 31) / 32 * 32;
  L.bcap2 = 2 * L.cap3;
  L.hcap2 = L.cap3 < (1ll << 20) ? L.cap3 : (1ll << 20);
  const long long per2 = L.bcap2 * 48 + L.hcap2 * (long long)sizeof(REnt);
  long long w2 = L.bcap2 < (1ll << 31) ? (long long)(tot / 2 / (size_t)per2) : 0;
  if (w2 > 8ll * sms) w2 = 8ll * sms;
  if (w2 > n + kWarps2 - 1) w2 = n + kWarps2 - 1;  // (no more warps than queries)
  L.warps2 = w2 / kWarps2 * kWarps2;
  size_t o = 0;
  L.ctr = o; o += a256(sizeof(Ctr));
  L.overflow = o; o += a256((size_t)(n > 0 ? n : 1) * 8);
  L.fallback = o; o += a256((size_t)(n > 0 ? n : 1) * 8);
  L.arena1 = o; o += a256((size_t)L.threads1 * kCap1 * 64);
  const size_t a2 = (size_t)L.warps2 * per2, a3 = (size_t)L.slots3 * L.cap3 * 64;
  L.arena2 = o; o += a256(a2 > a3 ? a2 : a3);
  L.total = o;
  return L;
}

int sm_count(int hint) {
  if (hint > 0) return hint;
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return v;
}

}  // namespace

extern "C" {

size_t tccd_irf_workspace_bytes(int64_t n, int64_t max_checks_max, int32_t big_slots) {
  return irf_layout(n, max_checks_max, big_slots, sm_count(0)).total;
}

int tccd_irf_batch(const tccd_batch* b, void* stream) {
  if (!b) return TCCD_E_NULL;
  if (b->struct_size != sizeof(tccd_batch)) return TCCD_E_STRUCT;
  if (b->n < 0) return TCCD_E_N;
  if (b->n > 0 && (!b->points || !b->status || !b->toi)) return TCCD_E_NULL;
  if (!b->delta && !(b->delta_all > 0.0)) return TCCD_E_DELTA;
  if (!b->t_max && !(b->t_max_all >= 0.0 && b->t_max_all < 1.0 / 0.0)) return TCCD_E_TMAX;
  if (!b->kind && b->kind_all != 0 && b->kind_all != 1) return TCCD_E_KIND;
  const long long mcmax = b->max_checks ? b->max_checks_max : b->max_checks_all;
  if (mcmax > (1ll << 40)) return TCCD_E_CAPACITY;
  const int sms = sm_count(b->device_sms);
  const IrfLayout L = irf_layout(b->n, mcmax, b->heavy_blocks, sms);
  if (!b->workspace || b->workspace_bytes < L.total) return TCCD_E_WORKSPACE;
  if (b->n == 0) return TCCD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned char* ws = (unsigned char*)b->workspace;
  Args a;
  memset(&a, 0, sizeof a);
  a.n = b->n;
  a.points = b->points;
  a.kind = b->kind;
  a.kind_all = b->kind_all;
  a.delta = b->delta;
  a.delta_all = b->delta_all;
  a.max_checks = (const long long*)b->max_checks;
  a.max_checks_all = b->max_checks_all;
  a.t_max = b->t_max;
  a.t_max_all = b->t_max_all;
  a.status = b->status;
  a.toi = b->toi;
  a.tol = b->tol;
  a.codom = b->codom;
  a.checks = (long long*)b->checks;
  a.early = b->early;
  a.witness = b->witness;
  a.level = b->level;
  Ctr* ctr = (Ctr*)(ws + L.ctr);
  long long* ovf = (long long*)(ws + L.overflow);
  long long* fb = (long long*)(ws + L.fallback);
  if (cudaMemsetAsync(ctr, 0, sizeof(Ctr), st) != cudaSuccess) return TCCD_E_CUDA;
  const bool heavy_only = (b->flags & TCCD_FLAG_HEAVY_ONLY) != 0 && L.warps2 > 0;
  if (heavy_only) {
    irf_fill_all<<<(unsigned)((b->n + 255) / 256), 256, 0, st>>>(b->n, ovf, ctr);
  } else {
    irf_kernel<<<(unsigned)(L.threads1 / kThreads), kThreads, 0, st>>>(
        a, ctr, ws + L.arena1, kCap1, nullptr, ovf, 0, L.warps2 > 0 ? 1 : 0);
  }
  if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  // pass 2 (returns at once when nothing overflowed): warp per query over runs
  if (L.warps2 > 0) {
    irf_warp_kernel<<<(unsigned)(L.warps2 / kWarps2), 32 * kWarps2, 0, st>>>(
        a, ctr, ws + L.arena2, L.bcap2, L.hcap2, ovf, fb);
    if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  } else {  // (no room for a pass-2 warp: pass 3 takes the overflow list)
    irf_fill_fallback<<<1, 32, 0, st>>>(ctr);
    if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  }
  // pass 3 (a no-op when nothing fell back): max_checks + 2 heap entries per slot
  irf_kernel<<<(unsigned)(L.slots3 / 32), 32, 0, st>>>(a, ctr, ws + L.arena2, L.cap3,
                                                       L.warps2 > 0 ? fb : ovf, nullptr, 2, 0);
  if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  return TCCD_OK;
}

}  // extern "C"
