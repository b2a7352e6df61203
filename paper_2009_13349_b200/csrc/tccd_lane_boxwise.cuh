// Lane tier: one query per thread, one box check per loop iteration.
//
// Most queries of simulation-shaped batches (BASELINE config 3) stay shallow:
// their levels hold a handful of boxes (p50 4, p99 54)
// for a few dozen levels.  A group engine that advances many such queries a
// level per round pays its per-round bookkeeping (barriers, scans, layout)
// for very few boxes.  Here every thread runs the reference's state machine
// (ccdkit._kernel.solve_kernel, pkg/src/ccdkit/_kernel.py:173-324) for one
// query at a time, box by box in the reference's visiting order, and takes
// the next query from a shared queue as soon as its query ends, so every
// lane classifies one box per iteration whatever depth its query has.  A
// warp works on one query kind at a time (classify() never diverges on the
// kind).
//
// Boxes as lattice indices.  With a dyadic t_max every box of level L is a
// cell of the lattice with per-dimension split counts (nt, nu, nv), nt + nu
// + nv = L: t0 = ti * (t_max 2^-nt), u0 = ui 2^-nu, v0 = vi 2^-nv, and the
// upper bounds add the width (exact: the reference's midpoints 0.5 (lo +
// hi) of dyadic bounds are exact while every index stays below 2^53).  A box
// is one 64-bit word ti | ui | vi (v in the low bits), a child inserts one
// bit at its split dimension's position.  A level's refining boxes all split
// along one dimension (same widths, same kappas), so its children are
// visited in the order the reference's stable t_lo sort gives them: push
// order after a u / v split; after a t split, per run of equal parent t_lo,
// all lower children then all upper children.  Children are stored in push
// order (lower, upper, lower, upper, ...) with the length of each parent
// run's segment, and a t-split level's successor is visited segment by
// segment, even positions first: no box is ever moved.
//
// Latency: the word of the next box is loaded while the current box is
// classified; a lane that takes a new query copies its 64-byte record
// (index, filters, kappas) and then the query's coordinates and parameters
// into its shared-memory column with cp.async, one iteration apart, and
// starts on it the iteration after, so neither stalls the warp.
//
// A query leaves this tier when its next level has more than kLaneCap
// boxes (the level arrays hold 2 kLaneCap, so a level of at most kLaneCap
// boxes always has room for its children): that level goes to the light
// tier's handover pool, in visiting order with its run heads, with the
// check count and first / drop records, and the light tier resumes the
// query there.  If the handover pool is full, or the lattice would exceed
// its index range, the query restarts from its root in the light tier
// instead (exact: classification is a pure function of the box).
#pragma once

namespace tccd {

#ifndef TCCD_KL
#define TCCD_KL 128
#endif
#ifndef TCCD_NNT
#define TCCD_NNT 128
#endif
#ifndef TCCD_NMINB
#define TCCD_NMINB 4
#endif
constexpr int kLaneCap = TCCD_KL;  // largest level a lane processes
constexpr int kLaneArr = 2 * kLaneCap;  // level array capacity: its children always fit
constexpr int kLaneNT = TCCD_NNT;  // threads per CTA
constexpr int kLaneMaxSplits = 52;  // per dimension: midpoints stay exact (indices < 2^53)
constexpr int kLaneMaxLevel = 62;   // ti | ui | vi fits one 64-bit word
#ifndef TCCD_LANE_TAIL
#define TCCD_LANE_TAIL 128
#endif
constexpr int kLaneTailChecks = TCCD_LANE_TAIL;  // (tail handover threshold)
#ifndef TCCD_LANE_CLAIM
#define TCCD_LANE_CLAIM 32
#endif
constexpr int kLaneClaim = TCCD_LANE_CLAIM;  // queue entries a warp claims at once
// per-lane global scratch: two level arrays of words and two segment tables
// (a level's segments: at most one per refining box of the level before)
constexpr int kLaneSeg = kLaneCap;
constexpr int kLaneScratchWords = 2 * kLaneArr + kLaneSeg;  // (segment tables: 2 x u32 per word)

// A query queued for the lane tier by the prologue: its root box is
// non-disjoint and refined (one check done); its filters and kappas.
struct LaneRec {
  long long q;
  double wb;  // root hull width (the first record's codomain width)
  double eps[3];
  double kap[3];
};
static_assert(sizeof(LaneRec) == 64, "LaneRec layout");
// shared-memory column of one lane: the 24 coordinates, the LaneRec words,
// the per-query parameters, and the first / drop records (lattice word,
// codomain width, split counts | level << 24) -- read only when a query
// ends, so they do not hold registers
constexpr int kLaneCol = 42;
constexpr int kColQ = 24, kColWb = 25, kColEps = 26, kColKap = 29, kColSep = 32, kColDelta = 33,
              kColTmax = 34, kColMc = 35, kColFr = 36, kColDr = 39;

struct LaneIO {
  const LaneRec* rec;             // vertex-face entries from the front, edge-edge from the back
  long long rec_cap;
  const unsigned long long* count;  // [2] entries per kind
  unsigned long long* next;         // [2] next entry to take per kind
  unsigned long long* scratch;      // [grid threads][kLaneScratchWords]
  Pre* out;                         // light-tier queue (evicted queries go there)
  unsigned long long* out_count;
  unsigned long long* stats;        // [8] see Counters::lane
  // handover to the light tier: state records and the pool of level boxes
  Hand* hand;
  long long hand_cap;
  unsigned long long* hand_count;
  Box* pbox;
  uint8_t* pflag;
  long long pool_cap;
  unsigned long long* pool_count;
};

// this thread's column of a [kLaneCol][NT] shared array, read like an array
template <int NT>
struct ColP {
  const double* p;
  __device__ __forceinline__ double operator[](int k) const { return p[k * NT]; }
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// box of lattice word pk at split counts (nt, nu, nv)
__device__ __forceinline__ Box lane_box(unsigned long long pk, int nt, int nu, int nv,
                                        double t_max) {
  // 2^-n (n <= 62) built from its exponent bits: exact, no ldexp call
  const double wt = t_max * __longlong_as_double((long long)(1023 - nt) << 52);
  const double wu = __longlong_as_double((long long)(1023 - nu) << 52);
  const double wv = __longlong_as_double((long long)(1023 - nv) << 52);
  const unsigned long long ti = pk >> (nu + nv);
  const unsigned long long ui = (pk >> nv) & ((1ull << nu) - 1ull);
  const unsigned long long vi = pk & ((1ull << nv) - 1ull);
  Box b;
  b.t0 = (double)ti * wt; b.t1 = b.t0 + wt;
  b.u0 = (double)ui * wu; b.u1 = b.u0 + wu;
  b.v0 = (double)vi * wv; b.v1 = b.v0 + wv;
  return b;
}

// split dimension of a level whose boxes have widths (wt, wu, wv)
// (_kernel.py:219-229: strict >, ties to t, then u)
template <typename KapT>
__device__ __forceinline__ int lane_split_dim(double wt, double wu, double wv, KapT kap) {
  const double ct = wt * kap[0], cu = wu * kap[1], cv = wv * kap[2];
  int sd = 0;
  double best = ct;
  if (cu > best) { sd = 1; best = cu; }
  if (cv > best) sd = 2;
  return sd;
}

// a recorded box in a lane's column (kColFr / kColDr): lattice word, width,
// split counts nt | nu << 8 | nv << 16 | level << 24
__device__ __forceinline__ void lane_record(double* col, int at, unsigned long long pk, double codom,
                                            int meta) {
  col[at * kLaneNT] = __longlong_as_double((long long)pk);
  col[(at + 1) * kLaneNT] = codom;
  col[(at + 2) * kLaneNT] = __longlong_as_double((long long)meta);
}

__device__ __forceinline__ Box lane_record_box(const double* col, int at, double t_max) {
  const unsigned long long pk = (unsigned long long)__double_as_longlong(col[at * kLaneNT]);
  const int m = (int)__double_as_longlong(col[(at + 2) * kLaneNT]);
  return lane_box(pk, m & 255, (m >> 8) & 255, (m >> 16) & 255, t_max);
}

__device__ __forceinline__ int lane_record_level(const double* col, int at) {
  return (int)__double_as_longlong(col[(at + 2) * kLaneNT]) >> 24;
}

__device__ __forceinline__ void lane_emit(const Args& a, long long q, uint8_t status, Box b,
                                       double codom, long long checks, int early, int level) {
  write_result(a, q, status, b, codom, checks, early, level);
}

// the result of a query that ends on the record at column offset `at`
__device__ __forceinline__ void lane_write(const Args& a, const double* col, int at,
                                           long long checks, int early) {
  const long long q = __double_as_longlong(col[kColQ * kLaneNT]);
  const double t_max = col[kColTmax * kLaneNT];
  lane_emit(a, q, kHit, lane_record_box(col, at, t_max), col[(at + 1) * kLaneNT], checks, early,
            lane_record_level(col, at));
}

struct LaneStats {
  unsigned int checks = 0, done = 0, evicted = 0, wasted = 0, handed = 0;
};

// add this warp's counters of one pass to the tier's (warp-reduced)
__device__ __forceinline__ void lane_flush(const LaneIO& io, const LaneStats& st, int kind) {
  // (classifications: the checks on the reference's path + the ones repeated)
  const unsigned int v[6] = {st.checks + st.wasted, st.checks, st.done, st.evicted, st.wasted,
                             st.handed};
  const int slot[6] = {kind, 2 + kind, 4 + kind, 6, 7, 8};
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    unsigned long long x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&io.stats[slot[i]], x);
  }
}

// One kind's queue (kind is warp-uniform; only the classification is
// specialized on it, so the loop's code exists once).
__device__ __forceinline__ void lane_loop(const Args& a, const LaneIO& io, double* col,
                                          unsigned long long* lb, const int kind) {
  LaneStats st;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const ColP<kLaneNT> P{col};
  const ColP<kLaneNT> eps{col + kColEps * kLaneNT};
  const ColP<kLaneNT> kap{col + kColKap * kLaneNT};
  unsigned int* const segs = reinterpret_cast<unsigned int*>(lb + 2 * kLaneArr);  // [2][kLaneSeg]
  const unsigned long long total = io.count[kind];
  bool dry = false;  // (warp-uniform) this kind's queue is empty
  int state = 0;     // 0 idle, 1 record in flight, 2 coordinates in flight, 3 active
  // query
  int mc = 0, C = 0;  // (a lane query stays far below 2^31 checks: <= 62 levels of <= 64 boxes)
  double sep = 0, delta = 0;
  // level: split counts and widths of its boxes, its split dimension
  int L = 0, nt = 0, nu = 0, nv = 0, sd = 0;
  double wt = 1, wu = 1, wv = 1;
  int cb = 0;        // current level array: lb + cb (the next one: lb + (cb ^ kLaneArr))
  int sgb = 0;       // current segment table: segs + sgb (the next one: segs + (sgb ^ kLaneSeg))
  int ncur = 0, k = 0;
  // visiting order of the current level: identity, or (after a t split)
  // segment by segment, even positions first
  bool ilv = false;
  int seg_start = 0, seg_m = 0, seg_k = 0, seg_i = 0, seg_mn = 0, nseg = 0;
  unsigned long long pk = 0, pk_next = 0;
  // next level: children written, segments closed, the current run (t split)
  int nn = 0, nsn = 0, run_m = 0, seg0 = 0;
  unsigned long long run = ~0ull, nxt0 = 0;
  bool col_lvl = false;  // this level has had a non-disjoint box (last_colliding_level)
  double fr_t0 = 0, dr_t0 = 0;  // t_lo of the first / drop records (the rest: in the column)
  bool hf = false, hd = false;

  // The warp claims queue entries kLaneClaim at a time (one atomic on the
  // kind's counter per range, not per query) and hands them to its idle
  // lanes; the next range is claimed while the current one still lasts, and
  // the atomic's result is read an iteration later, so its latency is spent
  // classifying.  (All of this is warp-uniform.)
  unsigned long long r_base = 0, n_base = 0;
  int r_left = 0, n_left = 0;
  bool n_pend = false, n_have = false;
  unsigned long long claim_ret = 0;  // (lane 0's register)
  for (;;) {
    if (n_pend) {
      const unsigned long long base = __shfl_sync(FULL, claim_ret, 0);
      n_pend = false;
      if (base >= total) {
        dry = true;
      } else {
        n_base = base;
        n_left = (int)(total - base < (unsigned long long)kLaneClaim ? total - base : kLaneClaim);
        n_have = true;
      }
    }
    if (r_left == 0 && n_have) {
      r_base = n_base;
      r_left = n_left;
      n_have = false;
    }
    if (!dry && !n_pend && !n_have && r_left < kLaneClaim / 2) {
      if (lane == 0) claim_ret = atomicAdd(&io.next[kind], (unsigned long long)kLaneClaim);
      n_pend = true;
    }
    const unsigned need = __ballot_sync(FULL, state == 0);
    if (need && r_left > 0) {
      const int rank = __popc(need & ((1u << lane) - 1u));
      const int take = __popc(need) < r_left ? __popc(need) : r_left;
      if (state == 0 && rank < take) {
        // start the copy of the entry's record
        const unsigned long long kq = r_base + rank;
        const double* src = reinterpret_cast<const double*>(
            &io.rec[kind ? io.rec_cap - 1 - (long long)kq : (long long)kq]);
#pragma unroll
        for (int i = 0; i < 8; ++i) cp_async8(col + (kColQ + i) * kLaneNT, src + i);
        state = 1;
      }
      r_base += take;
      r_left -= take;
    }
    if (!__any_sync(FULL, state != 0)) {
      // nothing in flight: done once the queue is known empty
      if (dry && r_left == 0 && !n_have && !n_pend) break;
      continue;
    }
    if (state == 0) continue;
    if (state == 1) {
      // the record has landed (one iteration later): copy the coordinates
      // and the per-query parameters
      cp_async_wait_all();
      const long long qn = __double_as_longlong(col[kColQ * kLaneNT]);
      const double* src = a.points + 24 * qn;
#pragma unroll
      for (int i = 0; i < 24; ++i) cp_async8(col + i * kLaneNT, src + i);
      if (a.sep) cp_async8(col + kColSep * kLaneNT, a.sep + qn);
      else col[kColSep * kLaneNT] = a.sep_all;
      if (a.delta) cp_async8(col + kColDelta * kLaneNT, a.delta + qn);
      else col[kColDelta * kLaneNT] = a.delta_all;
      if (a.t_max) cp_async8(col + kColTmax * kLaneNT, a.t_max + qn);
      else col[kColTmax * kLaneNT] = a.t_max_all;
      if (a.max_checks) cp_async8(col + kColMc * kLaneNT, reinterpret_cast<const double*>(a.max_checks + qn));
      else col[kColMc * kLaneNT] = __longlong_as_double(a.max_checks_all);
      state = 2;
      continue;
    }
    if (state == 2) {
      cp_async_wait_all();
      {
        const long long m = __double_as_longlong(col[kColMc * kLaneNT]);
        mc = m < 0x7fffffffLL ? (int)m : 0x7fffffff;
      }
      sep = col[kColSep * kLaneNT];
      delta = col[kColDelta * kLaneNT];
      const double t_max = col[kColTmax * kLaneNT];
      // the root (level 0, one check, the prologue's) is the first record
      // and was refined: level 1 = its two children (never clipped: a root
      // child's lower corner is 0)
      lane_record(col, kColFr, 0ull, col[kColWb * kLaneNT], 0);
      fr_t0 = 0.0;
      hf = true; hd = false;
      C = 1;
      nt = nu = nv = 0;
      wt = t_max; wu = 1.0; wv = 1.0;
      const int s0 = lane_split_dim(wt, wu, wv, kap);
      if (s0 == 0) { nt = 1; wt *= 0.5; } else if (s0 == 1) { nu = 1; wu *= 0.5; } else { nv = 1; wv *= 0.5; }
      cb = 0; sgb = 0;
      lb[0] = 0ull;
      lb[1] = 1ull;
      ncur = 2; k = 0; L = 1;
      // (a t split of the root leaves one run of one parent: order 0, 1 either way)
      ilv = false; seg_start = 0; seg_m = 0; seg_k = 0; seg_i = 0; seg_mn = 0; nseg = 0;
      pk = 0; pk_next = 1;
      nn = 0; nsn = 0; run_m = 0; seg0 = 0; run = ~0ull; nxt0 = 0;
      col_lvl = false;
      sd = lane_split_dim(wt, wu, wv, kap);
      state = 3;
    }
    if (state != 3) continue;  // (idle: this kind's queue ran dry)

    // ---- one box of the current level, in visiting order.  The bookkeeping
    // is written as selects and predicated stores, so the lanes of a warp --
    // each somewhere else in its own query -- run it together; only the
    // writes of a finished query branch.
    unsigned long long* const cur = lb + cb;
    unsigned long long* const nxt = lb + (cb ^ kLaneArr);
    unsigned int* const snx = segs + (sgb ^ kLaneSeg);
    // the next box of this level: its word is loaded now, used next iteration
    const bool more = k + 1 < ncur;
    const bool n_newseg = ilv && seg_k + 1 == 2 * seg_m;
    const int n_start = n_newseg ? seg_start + 2 * seg_m : seg_start;
    const int n_m = n_newseg ? seg_mn : seg_m;
    const int n_k = n_newseg ? 0 : seg_k + 1;
    const int n_i = seg_i + (n_newseg ? 1 : 0);
    const int pos1 = !ilv ? k + 1 : (n_k < n_m ? n_start + 2 * n_k : n_start + 2 * (n_k - n_m) + 1);
    if (more) pk_next = cur[pos1];
    const int suv = nu + nv;
    const unsigned long long ti = pk >> suv;
    // a t-split level: a new run of equal t_lo closes the previous run's
    // segment of the next level
    const bool new_run = sd == 0 && ti != run;
    const bool close_run = new_run && run_m > 0;
    if (close_run) snx[nsn] = (unsigned)run_m;
    seg0 = close_run && nsn == 0 ? run_m : seg0;
    nsn += close_run ? 1 : 0;
    run_m = new_run ? 0 : run_m;
    run = sd == 0 ? ti : run;
    Box b;
    b.t0 = (double)ti * wt; b.t1 = b.t0 + wt;
    b.u0 = (double)((pk >> nv) & ((1ull << nu) - 1ull)) * wu; b.u1 = b.u0 + wu;
    b.v0 = (double)(pk & ((1ull << nv) - 1ull)) * wv; b.v1 = b.v0 + wv;
    double wb;
    const int cls = kind == 0 ? classify_full<0>(P, b, eps, sep, wb)
                              : classify_full<1>(P, b, eps, sep, wb);
    ++C;
    const bool disj = cls == kDisjoint;
    const bool budget = C >= mc;
    const bool accept = !disj && (wb < delta || cls == kContained);  // (:215)
    // first colliding box of this level (:201-206)
    const int meta = nt | (nu << 8) | (nv << 16) | (L << 24);
    const bool first = !disj && !col_lvl;
    if (first) lane_record(col, kColFr, pk, wb, meta);
    fr_t0 = first ? b.t0 : fr_t0;
    hf = hf || first;
    // the ways this box can end the query
    const bool end_disj = disj && budget && (hd || more || nn > 0);   // (:188-199)
    const bool end_budget = !disj && budget;                          // (:208-213)
    const bool end_acc = accept && !budget && !col_lvl;               // (:243-252)
    int outcome = 0;  // 0 continue, 1 ended (result written), 2 evict
    if (end_disj || end_budget || end_acc) {
      const bool use_drop = hd && (end_acc ? dr_t0 < b.t0
                                           : (end_disj ? (!hf || dr_t0 < fr_t0) : dr_t0 < fr_t0));
      // (an accepted first box of its level: the record just written is it)
      lane_write(a, col, use_drop ? kColDr : kColFr, C, end_acc ? 0 : 1);
      outcome = 1;
    }
    // an accepted box after the level's first: the drop record (:253-258)
    const bool drop = accept && !budget && col_lvl && (!hd || b.t0 < dr_t0);
    if (drop) lane_record(col, kColDr, pk, wb, meta);
    dr_t0 = drop ? b.t0 : dr_t0;
    hd = hd || drop;
    // refine along the level's split dimension: insert the child bit; the
    // children are stored in push order.  Vertex-face: the upper child of a
    // u / v split only inside u + v <= 1 (_kernel.py:276-310); t-split
    // children are never clipped.
    const bool refine = !disj && !budget && !accept;
    const bool evict = refine && nn + 2 > kLaneArr;  // (never: levels <= kLaneCap)
    const bool push = refine && !evict;
    const int pos = sd == 0 ? suv : (sd == 1 ? nv : 0);
    const unsigned long long lo = ((pk >> pos) << (pos + 1)) | (pk & ((1ull << pos) - 1ull));
    const unsigned long long hi = lo | (1ull << pos);
    bool push_hi = true;
    if (kind == 0) {
      const bool hu = 0.5 * (b.u0 + b.u1) + b.v0 <= 1.0;
      const bool hv = b.u0 + 0.5 * (b.v0 + b.v1) <= 1.0;
      push_hi = sd == 0 ? true : (sd == 1 ? hu : hv);
    }
    if (push) {
      nxt[nn] = lo;
      if (push_hi) nxt[nn + 1] = hi;
    }
    nxt0 = push && nn == 0 ? lo : nxt0;
    nn += push ? (push_hi ? 2 : 1) : 0;
    run_m += push && sd == 0 ? 1 : 0;
    col_lvl = col_lvl || !disj;
    outcome = evict ? 2 : outcome;
    // advance to the next box
    const bool go = outcome == 0;
    k += go ? 1 : 0;
    seg_start = go ? n_start : seg_start;
    seg_m = go ? n_m : seg_m;
    seg_k = go ? n_k : seg_k;
    seg_i = go ? n_i : seg_i;
    if (go && n_newseg && seg_i + 1 < nseg) seg_mn = (int)segs[sgb + seg_i + 1];
    pk = go ? pk_next : pk;
    // ---- level end
    const bool lvl_end = go && k == ncur;
    const bool close_last = lvl_end && run_m > 0;
    if (close_last) snx[nsn] = (unsigned)run_m;
    seg0 = close_last && nsn == 0 ? run_m : seg0;
    nsn += close_last ? 1 : 0;
    run_m = lvl_end ? 0 : run_m;
    if (lvl_end && nn == 0) {
      // queue exhausted (_kernel.py:321-324)
      if (hd) {
        lane_write(a, col, kColDr, C, 0);
      } else {
        const Box z = {0, 0, 0, 0, 0, 0};
        lane_emit(a, __double_as_longlong(col[kColQ * kLaneNT]), kFree, z, 0.0, C, 0, 0);
      }
      outcome = 1;
    }
    const bool nl = lvl_end && nn > 0;  // the next level becomes current
    cb = nl ? cb ^ kLaneArr : cb;
    sgb = nl ? sgb ^ kLaneSeg : sgb;
    const bool nilv = sd == 0;
    if (nl && nilv && nsn > 1) seg_mn = (int)segs[sgb + 1];
    ilv = nl ? nilv : ilv;
    nseg = nl ? nsn : nseg;
    seg_start = nl ? 0 : seg_start;
    seg_k = nl ? 0 : seg_k;
    seg_i = nl ? 0 : seg_i;
    seg_m = nl ? seg0 : seg_m;
    ncur = nl ? nn : ncur;
    k = nl ? 0 : k;
    pk = nl ? nxt0 : pk;
    nn = nl ? 0 : nn;
    nsn = nl ? 0 : nsn;
    run = nl ? ~0ull : run;
    L += nl ? 1 : 0;
    col_lvl = nl ? false : col_lvl;
    // every refining box of the level split along sd
    const bool st_ = nl && sd == 0, su_ = nl && sd == 1, sv_ = nl && sd == 2;
    nt += st_ ? 1 : 0; wt = st_ ? 0.5 * wt : wt;
    nu += su_ ? 1 : 0; wu = su_ ? 0.5 * wu : wu;
    nv += sv_ ? 1 : 0; wv = sv_ ? 0.5 * wv : wv;
    const int ns = sd == 0 ? nt : (sd == 1 ? nu : nv);
    // a level too large for this tier (or a lattice about to leave its index
    // range) is handed over to the light tier; so is, once this kind's queue
    // is empty, the level of a query that has already run a while: the
    // lane tier's tail (lanes idle while the last queries finish one box at
    // a time) becomes level-parallel work for the light tier
    outcome = nl && (ncur > kLaneCap || ns > kLaneMaxSplits || L > kLaneMaxLevel ||
                     (dry && C >= kLaneTailChecks))
                  ? 3 : outcome;
    sd = nl ? lane_split_dim(wt, wu, wv, kap) : sd;
    if (outcome == 1) {
      st.checks += (unsigned)(C - 1);  // checks of finished queries (root: prologue's)
      st.done += 1;
      state = 0;
    } else if (outcome >= 2) {
      // to the light tier: with the current level handed over (outcome 3,
      // room permitting), else restarting from the root
      unsigned int hidx = 0xffffffffu;
      if (outcome == 3) {
        const unsigned long long h = atomicAdd(io.hand_count, 1ull);
        const unsigned long long off = atomicAdd(io.pool_count, (unsigned long long)ncur);
        if ((long long)h < io.hand_cap && (long long)(off + ncur) <= io.pool_cap) {
          hidx = (unsigned int)h;
          const unsigned long long* cw = lb + cb;
          int ss = 0, sm = seg_m, sk = 0, si = 0;
          double prev = -1.0;
          for (int j = 0; j < ncur; ++j) {
            int pos = j;
            if (ilv) {
              if (sk == 2 * sm) { ss += 2 * sm; ++si; sm = (int)segs[sgb + si]; sk = 0; }
              pos = sk < sm ? ss + 2 * sk : ss + 2 * (sk - sm) + 1;
              ++sk;
            }
            const Box bb = lane_box(cw[pos], nt, nu, nv, col[kColTmax * kLaneNT]);
            io.pbox[off + j] = bb;
            io.pflag[off + j] = (uint8_t)(j == 0 || bb.t0 != prev ? 128 : 0);  // the engine's kHead
            prev = bb.t0;
          }
          Hand& H = io.hand[h];
          H.C = C;
          H.off = (long long)off;
          H.level = L;
          H.n = ncur;
          const double t_max = col[kColTmax * kLaneNT];
          H.rec[0].b = lane_record_box(col, kColFr, t_max);
          H.rec[0].codom = col[(kColFr + 1) * kLaneNT];
          H.rec[0].level = lane_record_level(col, kColFr);
          H.rec[1].b = lane_record_box(col, kColDr, t_max);
          H.rec[1].codom = col[(kColDr + 1) * kLaneNT];
          H.rec[1].level = lane_record_level(col, kColDr);
          H.have_first = hf ? 1 : 0;
          H.have_drop = hd ? 1 : 0;
          st.handed += 1;
        }
      }
      const unsigned long long e = atomicAdd(io.out_count, 1ull);
      io.out[e] = Pre{__double_as_longlong(col[kColQ * kLaneNT]), 0.0, 0u, hidx};
      st.evicted += 1;
      // (a restart repeats the lane's checks in the light tier)
      if (hidx == 0xffffffffu) st.wasted += (unsigned)(C - 1);
      else st.checks += (unsigned)(C - 1);  // (on the reference's path: the light tier goes on)
      state = 0;
    }
  }
  lane_flush(io, st, kind);
}

constexpr size_t kLaneSmemBytes = 0;  // (static shared memory)

__global__ void __launch_bounds__(kLaneNT, TCCD_NMINB) lane_kernel(Args a, LaneIO io) {
  __shared__ double Ps[kLaneCol * kLaneNT];
  const long long gt = (long long)blockIdx.x * kLaneNT + threadIdx.x;
  unsigned long long* lb = io.scratch + gt * kLaneScratchWords;
  double* col = Ps + threadIdx.x;
  const unsigned long long nvf = io.count[0], nee = io.count[1];
  // first kind of this warp: warps split between the kinds in proportion to
  // their queues; a warp whose queue runs dry moves to the other one
  const long long gw = gt >> 5, nw = (long long)gridDim.x * (kLaneNT / 32);
  int kind = (nvf + nee) > 0 && (unsigned long long)gw * (nvf + nee) < nee * (unsigned long long)nw;
  for (int pass = 0; pass < 2; ++pass, kind ^= 1) lane_loop(a, io, col, lb, kind);
}

}  // namespace tccd
