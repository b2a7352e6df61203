// Lane tier: one query per thread, one REFINING box per loop iteration.
//
// Most queries of simulation-shaped batches (BASELINE config 3) stay shallow:
// their levels hold a handful of boxes (p50 4, p99 54)
// for a few dozen levels.  A group engine that advances many such queries a
// level per round pays its per-round bookkeeping (barriers, scans, layout)
// for very few boxes.  Here every thread runs the reference's state machine
// (ccdkit._kernel.solve_kernel, pkg/src/ccdkit/_kernel.py:173-324) for one
// query at a time and takes the next query from a shared queue as soon as its
// query ends.  A warp works on one query kind at a time (the classification
// never diverges on the kind).
//
// Children are classified when their parent is refined.  Half of all boxes
// checked are disjoint (config 3: 49%), and a disjoint box does nothing in
// the reference but count as a check (_kernel.py:186-199, budget aside).  So
// an iteration takes one non-disjoint box of the current level in the
// reference's visiting order, runs the state machine's events for it (first
// box of its level, accept, drop record: _kernel.py:201-258), and, when it
// refines, classifies BOTH children at once -- two independent evaluations a
// thread interleaves -- and stores only the non-disjoint ones, with their
// class and hull width, for the next level.  Disjoint children are counted,
// never stored or visited: per level the lane keeps the number of all
// children (the checks the reference spends on the level) and the visiting
// rank, among all of them, of the first non-disjoint one (the check count of
// a query that ends there, _kernel.py:243-252).  The per-box bookkeeping
// runs once per refining box instead of once per box.  What is classified
// beyond the reference's path is the rest of a level whose first non-disjoint
// box ends the query (config 3: 2% of the checks); the results do not depend
// on it (classification is a pure function of the box).
//
// The check budget: a level whose boxes could reach m_I is never processed
// here (the query restarts in the light tier, which replays budget returns
// exactly), so the lane's state machine has no budget events.
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
// all lower children then all upper children.  A level array is filled from
// both ends: entries that keep their parent's t_lo (lower children, both
// children of u / v splits) upward from the bottom, upper children of t
// splits downward from the top, with one (count, count) segment per run of
// parents; the next level is visited segment by segment, bottom part then
// top part: no entry is ever moved.
//
// Latency: the entry of the next box is loaded while the current box's
// children are classified; with each claimed range of queue entries the warp
// fetches the entries' query indices, so a lane that takes a new query
// copies its 64-byte record (index, filters, kappas), the query's
// coordinates and its parameters into its shared-memory column with
// cp.async in one go and starts on it the iteration after.
//
// A query leaves this tier when its next level has more than kLaneCap
// non-disjoint boxes (the level arrays hold 2 kLaneCap entries, so the
// children of a level of at most kLaneCap always fit): that level's
// non-disjoint boxes go to the light tier's handover pool, in visiting order
// with their run heads, with the check count up to that level plus the
// level's disjoint boxes, and the first / drop records; the light tier
// resumes the query there and classifies exactly the boxes the reference
// still has to count.  (Only when the level's first box is not one that ends
// the query: that one the lane finishes itself.)  If the handover pool is
// full, the budget is near, or the lattice would exceed its index range, the
// query restarts from its root in the light tier instead.
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
constexpr int kLaneCap = TCCD_KL;  // largest level (non-disjoint boxes) a lane processes
constexpr int kLaneArr = 2 * kLaneCap;  // level array capacity: its children always fit
constexpr int kLaneNT = TCCD_NNT;  // threads per CTA
constexpr int kLaneMaxSplits = 52;  // per dimension: midpoints stay exact (indices < 2^53)
constexpr int kLaneMaxLevel = 62;   // ti | ui | vi fits one 64-bit word
#ifndef TCCD_LANE_TAIL
#define TCCD_LANE_TAIL 128
#endif
constexpr int kLaneTailChecks = TCCD_LANE_TAIL;  // (tail handover threshold)
#ifndef TCCD_LANE_TAIL_WIDTH
#define TCCD_LANE_TAIL_WIDTH 0
#endif
constexpr int kLaneTailWidth = TCCD_LANE_TAIL_WIDTH;  // smallest level handed over in the tail
#ifndef TCCD_LANE_TAIL_GRACE
#define TCCD_LANE_TAIL_GRACE 128
#endif
// iterations a warp goes on after its queue ran dry before its lanes hand over
constexpr int kLaneTailGrace = TCCD_LANE_TAIL_GRACE;
#ifndef TCCD_LANE_CLAIM
#define TCCD_LANE_CLAIM 32
#endif
constexpr int kLaneClaim = TCCD_LANE_CLAIM;  // queue entries a warp claims at once

// A stored (non-disjoint) box: its lattice word and its hull width, negated
// (sign bit) when the box is contained in the filter box
struct alignas(16) LaneEnt {
  unsigned long long pk;
  double w;
};
// per-lane global scratch: two level arrays and two segment tables (a
// level's segments are non-empty, so at most one per entry)
constexpr int kLaneSeg = kLaneArr;
constexpr int kLaneScratchWords = 2 * kLaneArr * 2 + kLaneSeg;  // (segment tables: 2 x u32 per word)

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
// codomain width, split counts | level << 24) and the drop record's t_lo --
// read only when a box is accepted, so they do not hold registers
constexpr int kLaneCol = 45;
constexpr int kColQ = 24, kColWb = 25, kColEps = 26, kColKap = 29, kColSep = 32, kColDelta = 33,
              kColTmax = 34, kColMc = 35, kColFr = 36, kColDr = 39, kColDrT0 = 42,
              kColF0 = 43 /* [2]: the next level's first entry */;

struct LaneIO {
  const LaneRec* rec;             // vertex-face entries from the front, edge-edge from the back
  long long rec_cap;
  const unsigned long long* count;  // [2] entries per kind
  unsigned long long* next;         // [2] next entry to take per kind
  unsigned long long* scratch;      // [grid threads][kLaneScratchWords]
  Pre* out;                         // light-tier queue (evicted queries go there)
  unsigned long long* out_count;
  unsigned long long* stats;        // [10] see Counters::lane
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

// the result of a query that ends on the record at column offset `at`
__device__ __forceinline__ void lane_write(const Args& a, const double* col, int at,
                                           long long checks) {
  const long long q = __double_as_longlong(col[kColQ * kLaneNT]);
  const double t_max = col[kColTmax * kLaneNT];
  write_result(a, q, kHit, lane_record_box(col, at, t_max), col[(at + 1) * kLaneNT], checks, 0,
               lane_record_level(col, at));
}

// per-thread 32-bit slots in shared memory: the pass's counters (touched when
// a query ends) and the rank bookkeeping of a level's first box (touched
// once per level) -- none of it holds registers
constexpr int kLaneInt = 9;
constexpr int kIntCls = 0, kIntChecks = 1, kIntDone = 2, kIntEvicted = 3, kIntWasted = 4,
              kIntHanded = 5, kIntPf = 6 /* [2]: by level parity */, kIntRk = 8;

// add this warp's counters of one pass to the tier's (warp-reduced), and
// clear them
__device__ __forceinline__ void lane_flush(const LaneIO& io, unsigned* si, int kind) {
  // (classifications: every child evaluated, on the reference's path or not)
  const int slot[6] = {kind, 2 + kind, 4 + kind, 6, 7, 8};
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    unsigned long long x = si[i * kLaneNT];
    si[i * kLaneNT] = 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&io.stats[slot[i]], x);
  }
}

// 2^(x - 1023) from its exponent field (0 < x < 2047): exact, two integer
// instructions, so a level's widths need no registers of their own
__device__ __forceinline__ double lane_pow2(int x) { return __hiloint2double(x << 20, 0); }

// One kind's queue (kind is warp-uniform; only the classification is
// specialized on it, so the loop's code exists once).  SEP0: the call's
// separation is 0 for every query.
template <bool SEP0>
__device__ __forceinline__ void lane_loop(const Args& a, const LaneIO& io, double* col,
                                          unsigned* si_, unsigned* wq, long long* sq,
                                          unsigned long long* lb, const int kind) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const ColP<kLaneNT> P{col};
  const ColP<kLaneNT> eps{col + kColEps * kLaneNT};
  const ColP<kLaneNT> kap{col + kColKap * kLaneNT};
  LaneEnt* const ent = reinterpret_cast<LaneEnt*>(lb);  // [2][kLaneArr]
  unsigned int* const segs = reinterpret_cast<unsigned int*>(lb + 2 * kLaneArr * 2);  // [2][kLaneSeg]
  // (warp-uniform) 0: this kind's queue has entries; else 1 + the iterations
  // since it was found empty
  int dry = 0;
  int state = 0;     // 0 idle, 2 record and coordinates in flight, 3 active
  // checks before the current level; the level's boxes (all of them, the
  // checks the reference spends on it).  (A lane query stays far below 2^31
  // checks: <= 62 levels of <= 4 kLaneCap boxes.)  The visiting rank, among
  // all of them, of the level's first non-disjoint box: si_[kIntPf + parity].
  int Cb = 0, nall = 0;
  // level: split counts of its boxes (widths 2^(xt - nt - 1023), 2^-nu,
  // 2^-nv; xt: t_max's exponent field), its split dimension
  int nt = 0, nu = 0, nv = 0, xt = 0, sd = 0;
  // current level array ent + cb and segment table segs + cb (the next
  // ones: cb ^ kLaneArr; kLaneSeg == kLaneArr)
  int cb = 0;
  int ncur = 0, k = 0;
  // visiting order of the current level: per segment the bottom part upward,
  // then the top part downward.  rAB: entries left in the segment after the
  // prefetched one (bottom | top << 16), pa: the next bottom position (the
  // next top position follows from k), sn: the next segment.
  unsigned rAB = 0, sn = 0;
  int pa = 0, si = 0, nseg = 0;
  unsigned long long pk = 0;
  double w = 0;
  ulonglong2 nx = make_ulonglong2(0ull, 0ull);  // the next entry (word, width bits)
  // next level: entries (bottom | top << 16), segments closed, the current
  // run of parents (t split: equal t_lo; else the whole level): its entries,
  // its refining parents, the children of the runs before it
  unsigned nAB = 0, runAB = 0;
  int nsn = 0, run_m = 0, run_base = 0, nall_next = 0;
  unsigned seg0 = 0, seg1 = 0;  // (the next level's first two segments)
  bool hd = false;
  static_assert(kLaneSeg == kLaneArr, "one parity offset for both tables");

  // The warp claims queue entries kLaneClaim at a time (one atomic on the
  // kind's counter per range, not per query) and hands them to its idle
  // lanes; the next range is claimed while the current one still lasts, and
  // the atomic's result is read an iteration later, so its latency is spent
  // classifying.  (All of this is warp-uniform; the ranges live in the
  // warp's shared-memory words wq: [0] current base, [1] next base, [2] next
  // length, [3] the queue's length.)  With a range's base the warp fetches
  // the query indices of its entries (one cp.async per lane into sq, double
  // buffered), so a lane that takes an entry knows its query at once and
  // copies record, coordinates and parameters together.
  static_assert(kLaneClaim == 32, "one entry of a claimed range per lane; ranges start at multiples of 32");
  wq[3] = (unsigned)io.count[kind];  // (a chunk's queue: <= 2^26 entries)
  int r_left = 0;
  int qb = 0;  // sq buffer of the current range
  bool n_pend = false, n_have = false;
  unsigned claim_ret = 0;  // (lane 0's register)
  for (;;) {
    dry += dry ? 1 : 0;
    if (n_pend) {
      const unsigned base = __shfl_sync(FULL, claim_ret, 0);
      const unsigned total = wq[3];
      n_pend = false;
      if (base >= total) {
        dry = 1;
      } else {
        const unsigned nl_ = total - base < (unsigned)kLaneClaim ? total - base : (unsigned)kLaneClaim;
        wq[1] = base;
        wq[2] = nl_;
        n_have = true;
        if ((unsigned)lane < nl_) {
          const long long kq = (long long)base + lane;
          cp_async8(reinterpret_cast<double*>(sq + (qb ^ 1) * kLaneClaim + lane),
                    reinterpret_cast<const double*>(&io.rec[kind ? io.rec_cap - 1 - kq : kq]));
        }
      }
    }
    if (r_left == 0 && n_have) {
      // (the range's query indices have landed: fetched an atomic's round
      // trip and at least one iteration ago)
      cp_async_wait_all();
      __syncwarp();
      wq[0] = wq[1];
      r_left = (int)wq[2];
      qb ^= 1;
      n_have = false;
    }
    if (!dry && !n_pend && !n_have && r_left < kLaneClaim / 2) {
      // (the counter's low word: at most the queue's length + warps * kLaneClaim)
      if (lane == 0) claim_ret = (unsigned)atomicAdd(&io.next[kind], (unsigned long long)kLaneClaim);
      n_pend = true;
    }
    const unsigned need = __ballot_sync(FULL, state == 0);
    if (need && r_left > 0) {
      const int rank = __popc(need & ((1u << lane) - 1u));
      const int take = __popc(need) < r_left ? __popc(need) : r_left;
      const unsigned r_base = wq[0];
      if (state == 0 && rank < take) {
        // start the copies of the entry's record, its query's coordinates
        // and the per-query parameters
        const unsigned kq = r_base + rank;
        const double* src = reinterpret_cast<const double*>(
            &io.rec[kind ? io.rec_cap - 1 - (long long)kq : (long long)kq]);
#pragma unroll
        for (int i = 0; i < 8; ++i) cp_async8(col + (kColQ + i) * kLaneNT, src + i);
        const long long qn = sq[qb * kLaneClaim + (kq & (kLaneClaim - 1))];
        const double* pts = a.points + 24 * qn;
#pragma unroll
        for (int i = 0; i < 24; ++i) cp_async8(col + i * kLaneNT, pts + i);
        if (a.sep) cp_async8(col + kColSep * kLaneNT, a.sep + qn);
        else col[kColSep * kLaneNT] = a.sep_all;
        if (a.delta) cp_async8(col + kColDelta * kLaneNT, a.delta + qn);
        else col[kColDelta * kLaneNT] = a.delta_all;
        if (a.t_max) cp_async8(col + kColTmax * kLaneNT, a.t_max + qn);
        else col[kColTmax * kLaneNT] = a.t_max_all;
        if (a.max_checks) cp_async8(col + kColMc * kLaneNT, reinterpret_cast<const double*>(a.max_checks + qn));
        else col[kColMc * kLaneNT] = __longlong_as_double(a.max_checks_all);
        state = 2;
      }
      __syncwarp();
      wq[0] = r_base + take;
      r_left -= take;
    }
    if (!__any_sync(FULL, state != 0)) {
      // nothing in flight: done once the queue is known empty
      if (dry && r_left == 0 && !n_have && !n_pend) break;
      continue;
    }
    if (state == 0) continue;
    if (state == 2) {
      cp_async_wait_all();
      // level 0: the root, classified by the prologue (non-disjoint, to be
      // refined: one check, rank 0); this lane's first iteration records it
      // as the level's first box and classifies its two children
      Cb = 0; nall = 1;
      si_[kIntPf * kLaneNT] = 0u;
      nt = nu = nv = 0;
      // (t_max is a power of two in the normal range: the prologue's test)
      xt = (int)(__double2hiint(col[kColTmax * kLaneNT]) >> 20);
      sd = lane_split_dim(lane_pow2(xt), 1.0, 1.0, kap);
      cb = 0;
      ncur = 1; k = 0;
      rAB = 0; pa = 0; si = 0; nseg = 1; sn = 0;
      pk = 0; w = col[kColWb * kLaneNT];
      nAB = runAB = 0;
      nsn = run_m = run_base = nall_next = 0;
      hd = false;
      state = 3;
    }
    if (state != 3) continue;  // (idle: this kind's queue ran dry)

    // ---- one non-disjoint box of the current level, in visiting order.  The
    // bookkeeping is written as selects and predicated stores, so the lanes
    // of a warp -- each somewhere else in its own query -- run it together;
    // only the rare events (an accepted box, a finished query) branch.
    LaneEnt* const cur = ent + cb;
    LaneEnt* const nxt = ent + (cb ^ kLaneArr);
    unsigned int* const snx = segs + (cb ^ kLaneArr);
    const int par = cb ? 1 : 0;
    // the next entry of this level: loaded now, used next iteration
    const bool more = k + 1 < ncur;
    {
      const bool newseg = rAB == 0;
      rAB = newseg ? sn : rAB;
      si += newseg ? 1 : 0;
      if (more && newseg && si + 1 < nseg) sn = segs[cb + si + 1];
      const bool useA = (rAB & 0xffffu) != 0;
      const int posn = useA ? pa : kLaneArr - 2 - k + pa;
      pa += useA ? 1 : 0;
      rAB -= useA ? 1u : 0x10000u;
      // (loaded unconditionally -- a level's last entry re-reads slot 0 --
      // and straight into the registers that carry it to the next
      // iteration: a predicated load went through temporaries that were
      // copied, and waited for, right behind it)
      TCCD_ASSERT(!more || (posn >= 0 && posn < kLaneArr));
      nx = *reinterpret_cast<const ulonglong2*>(cur + (more ? posn : 0));
    }
    // closing a segment of the next level; its first one fixes the level's
    // first box: the first bottom entry if it has one (kIntRk: its rank),
    // else its first top entry (kIntRk: the children before the run plus its
    // parent's index; the run's lower children, one per refining parent,
    // come before it)
    auto close_segment = [&](bool close) {
      TCCD_ASSERT(!close || nsn < kLaneSeg);
      if (close) snx[nsn] = runAB;
      if (close && nsn == 0) {
        seg0 = runAB;
        si_[(kIntPf + (par ^ 1)) * kLaneNT] =
            si_[kIntRk * kLaneNT] + ((runAB & 0xffffu) ? 0u : (unsigned)run_m);
      }
      seg1 = close && nsn == 1 ? runAB : seg1;
      nsn += close ? 1 : 0;
    };
    const int suv = nu + nv;
    const unsigned long long ti = pk >> suv;
    const double wt = lane_pow2(xt - nt), wu = lane_pow2(1023 - nu), wv = lane_pow2(1023 - nv);
    const double t0 = (double)ti * wt;
    const double u0 = (double)((pk >> nv) & ((1ull << nu) - 1ull)) * wu;
    const double v0 = (double)(pk & ((1ull << nv) - 1ull)) * wv;
    const bool first = k == 0;  // the first non-disjoint box of its level (:201-206)
    // accepted: hull narrower than delta, or contained (sign bit) (:215)
    const bool accept = fabs(w) < col[kColDelta * kLaneNT] || __double_as_longlong(w) < 0;
    const int meta = nt | (nu << 8) | (nv << 16) | ((nt + suv) << 24);
    if (first) lane_record(col, kColFr, pk, fabs(w), meta);
    int outcome = 0;  // 0 continue, 1 ended (result written), 2 restart, 3 hand over
    unsigned cls_n = 0;  // children classified for a query that ends or leaves
    if (accept) {
      if (first) {
        // the level's first non-disjoint box ends the query (:243-252); the
        // reference has checked the boxes up to it
        cls_n = (unsigned)(Cb + nall - 1);
        Cb += (int)si_[(kIntPf + par) * kLaneNT] + 1;
        lane_write(a, col, hd && col[kColDrT0 * kLaneNT] < t0 ? kColDr : kColFr, Cb);
        outcome = 1;
      } else if (!hd || t0 < col[kColDrT0 * kLaneNT]) {
        // an accepted box after the level's first: the drop record (:253-258)
        lane_record(col, kColDr, pk, fabs(w), meta);
        col[kColDrT0 * kLaneNT] = t0;
        hd = true;
      }
    }
    // refine along the level's split dimension: insert the child bit.
    // Vertex-face: the upper child of a u / v split only inside u + v <= 1
    // (_kernel.py:276-310); t-split children are never clipped.
    const bool refine = !accept;
    const int pos = (sd == 0 ? suv : 0) + (sd == 1 ? nv : 0);  // (selects, not a jump table)
    const unsigned long long lo = ((pk >> pos) << (pos + 1)) | (pk & ((1ull << pos) - 1ull));
    const unsigned long long hi = lo | (1ull << pos);
    Box ba, bb;
    ba.t0 = t0; ba.t1 = t0 + wt; ba.u0 = u0; ba.u1 = u0 + wu; ba.v0 = v0; ba.v1 = v0 + wv;
    bb = ba;
    {
      // (midpoints of dyadic bounds: lo + w / 2 = 0.5 (lo + hi), exactly)
      const double mt = t0 + lane_pow2(xt - nt - 1), mu = u0 + lane_pow2(1022 - nu),
                   mv = v0 + lane_pow2(1022 - nv);
      ba.t1 = sd == 0 ? mt : ba.t1; bb.t0 = sd == 0 ? mt : bb.t0;
      ba.u1 = sd == 1 ? mu : ba.u1; bb.u0 = sd == 1 ? mu : bb.u0;
      ba.v1 = sd == 2 ? mv : ba.v1; bb.v0 = sd == 2 ? mv : bb.v0;
    }
    bool push_hi = true;
    if (kind == 0) push_hi = sd == 0 || bb.u0 + bb.v0 <= 1.0;  // (mid + the other lower bound)
    double wa_, wb_;
    int ca, cbx;
    {
      const double sep = SEP0 ? 0.0 : col[kColSep * kLaneNT];
      if (kind == 0) classify_pair<0, SEP0>(P, ba, bb, eps, sep, ca, wa_, cbx, wb_);
      else classify_pair<1, SEP0>(P, ba, bb, eps, sep, ca, wa_, cbx, wb_);
    }
    const bool na = refine && ca != kDisjoint;
    const bool nb = refine && push_hi && cbx != kDisjoint;
    {
      // children: the lower one at the bottom, the upper one of a t split at
      // the top, of a u / v split next at the bottom
      const double ea = ca == kContained ? -wa_ : wa_;
      const double eb = cbx == kContained ? -wb_ : wb_;
      const int nA = (int)(nAB & 0xffffu), nB = (int)(nAB >> 16);
      const int posb = sd == 0 ? kLaneArr - 1 - nB : nA + (na ? 1 : 0);
      // (bottom and top parts never meet: a level of <= kLaneCap boxes has <=
      // kLaneArr children)
      TCCD_ASSERT(!(na || nb) || (ncur <= kLaneCap && nA + nB + (na ? 1 : 0) + (nb ? 1 : 0) <= kLaneArr));
      TCCD_ASSERT(!nb || (posb >= 0 && posb < kLaneArr));
      if (na) nxt[nA] = LaneEnt{lo, ea};
      if (nb) nxt[posb] = LaneEnt{hi, eb};
      const unsigned add = (na ? 1u : 0u) + (nb ? (sd == 0 ? 0x10000u : 1u) : 0u);
      // the first segment's first bottom entry: its rank among all children
      // in visiting order (t split: the run's lower children come first, one
      // per parent; else push order); its first top entry: the children
      // before its run plus its parent's index in the run
      // (one slot each: a top entry's values stand until a bottom entry
      // comes); with it the entry itself, the next level's first
      if (nsn == 0 && (runAB & 0xffffu) == 0) {
        const bool f_a = (add & 0xffffu) != 0;
        const bool f_b = !f_a && (runAB >> 16) == 0 && (add >> 16) != 0;
        if (f_a)
          si_[kIntRk * kLaneNT] = (unsigned)(na ? (sd == 0 ? run_base + run_m : nall_next) : nall_next + 1);
        if (f_b) si_[kIntRk * kLaneNT] = (unsigned)(run_base + run_m);
        if (f_a || f_b) {
          col[kColF0 * kLaneNT] = __longlong_as_double((long long)(f_a && na ? lo : hi));
          col[(kColF0 + 1) * kLaneNT] = f_a && na ? ea : eb;
        }
      }
      runAB += add;
      nAB += add;
      run_m += refine && sd == 0 ? 1 : 0;
      nall_next += refine ? (push_hi ? 2 : 1) : 0;
    }
    // advance to the next entry
    const bool go = outcome == 0;
    k += go ? 1 : 0;
    pk = go ? nx.x : pk;
    w = go ? __longlong_as_double((long long)nx.y) : w;
    // ---- level end; in a t-split level, the end of a run of equal t_lo (the
    // next entry, already loaded, starts another): either closes the run's
    // segment of the next level, if it has entries
    const bool lvl_end = go && k == ncur;
    {
      const bool run_end = lvl_end || (go && sd == 0 && (pk >> suv) != ti);
      close_segment(run_end && runAB != 0);
      run_base += run_end ? 2 * run_m : 0;
      run_m = run_end ? 0 : run_m;
      runAB = run_end ? 0u : runAB;
    }
    const int nnext = (int)((nAB & 0xffffu) + (nAB >> 16));
    if (lvl_end && nnext == 0) {
      const long long m = __double_as_longlong(col[kColMc * kLaneNT]);
      if (Cb + nall + nall_next >= m) {
        // (a budget return among the last level's disjoint boxes,
        // _kernel.py:188-199: the light tier replays it)
        outcome = 2;
      } else {
        // queue exhausted (_kernel.py:321-324): every child was disjoint
        // (and counted)
        Cb += nall + nall_next;
        cls_n = (unsigned)(Cb - 1);
        if (hd) {
          lane_write(a, col, kColDr, Cb);
        } else {
          const Box z = {0, 0, 0, 0, 0, 0};
          write_result(a, __double_as_longlong(col[kColQ * kLaneNT]), kFree, z, 0.0, Cb, 0, 0);
        }
        outcome = 1;
      }
    }
    const bool nl = lvl_end && nnext > 0;  // the next level becomes current
    if (nl) {
      cb ^= kLaneArr;
      Cb += nall;
      nall = nall_next;
      ncur = nnext;
      k = 0;
      // the level's first entry (the first segment's bottom part, else its
      // top part); the visiting state is the one after it
      const bool fa = (seg0 & 0xffffu) != 0;
      pk = (unsigned long long)__double_as_longlong(col[kColF0 * kLaneNT]);
      w = col[(kColF0 + 1) * kLaneNT];
      rAB = seg0 - (fa ? 1u : 0x10000u);
      pa = fa ? 1 : 0;
      si = 0;
      nseg = nsn;
      sn = seg1;
      nAB = runAB = 0u;
      nsn = run_m = run_base = nall_next = 0;
      // every refining box of the level split along sd
      nt += sd == 0 ? 1 : 0;
      nu += sd == 1 ? 1 : 0;
      nv += sd == 2 ? 1 : 0;
      const int ns = sd == 0 ? nt : (sd == 1 ? nu : nv);
      // a lattice about to leave its index range, or a level that could
      // reach the budget: the query restarts in the light tier.  A level too
      // large for this tier is handed over to the light tier; so is,
      // kLaneTailGrace iterations after this kind's queue was found empty, the
      // level of a query that has already run a while: the lane tier's tail
      // (lanes idle while the last queries finish one box at a time) becomes
      // level-parallel work for the light tier.  About one query per lane
      // thread is in flight when the queue runs dry, most of them with fewer
      // than a hundred iterations to go: the grace period lets those finish
      // here instead of arriving at the light tier in one burst (a 6.25e6-
      // query shard: 80k -> 46k handovers, step 14.2 -> 13.5 ms).  (Not a
      // level whose first box ends the query: the lane finishes that one
      // itself.  kLaneTailWidth > 0 would keep narrow levels here: 8 / 16
      // measured no gain on 5e7 config-3 queries and doubled config 0's 1.3 ms.)
      const long long m = __double_as_longlong(col[kColMc * kLaneNT]);
      if (ns > kLaneMaxSplits || nt + nu + nv > kLaneMaxLevel || Cb + nall >= m) {
        outcome = 2;
      } else if (ncur > kLaneCap || (dry > kLaneTailGrace && Cb + nall >= kLaneTailChecks && ncur >= kLaneTailWidth)) {
        const bool acc0 = fabs(w) < col[kColDelta * kLaneNT] || __double_as_longlong(w) < 0;
        outcome = acc0 ? outcome : 3;
      }
      sd = lane_split_dim(lane_pow2(xt - nt), lane_pow2(1023 - nu), lane_pow2(1023 - nv), kap);
    }
    if (outcome == 1) {
      si_[kIntChecks * kLaneNT] += (unsigned)(Cb - 1);  // checks of finished queries (root: prologue's)
      si_[kIntCls * kLaneNT] += cls_n;
      si_[kIntDone * kLaneNT] += 1u;
      state = 0;
    } else if (outcome >= 2) {
      // to the light tier: with the current level handed over (outcome 3,
      // room permitting), else restarting from the root
      unsigned int hidx = 0xffffffffu;
      // checks the reference has spent when it starts on the handed-over
      // boxes' level, plus that level's disjoint boxes
      const int Ch = Cb + nall - ncur;
      if (outcome == 3) {
        const unsigned long long h = atomicAdd(io.hand_count, 1ull);
        const unsigned long long off = atomicAdd(io.pool_count, (unsigned long long)ncur);
        if ((long long)h < io.hand_cap && (long long)(off + ncur) <= io.pool_cap) {
          hidx = (unsigned int)h;
          const LaneEnt* cw = ent + cb;
          const double t_max = col[kColTmax * kLaneNT];
          double prev = -1.0;
          int qa = 0, qb = kLaneArr - 1, j = 0;
          for (int s = 0; s < nseg; ++s) {
            const unsigned sg = s == 0 ? seg0 : segs[cb + s];
            const int ca_ = (int)(sg & 0xffffu), cb_ = (int)(sg >> 16);
            for (int i = 0; i < ca_ + cb_; ++i, ++j) {
              const int p = i < ca_ ? qa++ : qb--;
              TCCD_ASSERT(p >= 0 && p < kLaneArr && j < ncur);
              const Box bx = lane_box(cw[p].pk, nt, nu, nv, t_max);
              io.pbox[off + j] = bx;
              io.pflag[off + j] = (uint8_t)(j == 0 || bx.t0 != prev ? 128 : 0);  // the engine's kHead
              prev = bx.t0;
            }
          }
          Hand& H = io.hand[h];
          H.C = Ch;
          H.off = (long long)off;
          H.level = nt + nu + nv;
          H.n = ncur;
          H.rec[0].b = lane_record_box(col, kColFr, t_max);
          H.rec[0].codom = col[(kColFr + 1) * kLaneNT];
          H.rec[0].level = lane_record_level(col, kColFr);
          H.rec[1].b = lane_record_box(col, kColDr, t_max);
          H.rec[1].codom = col[(kColDr + 1) * kLaneNT];
          H.rec[1].level = lane_record_level(col, kColDr);
          H.have_first = 1;
          H.have_drop = hd ? 1 : 0;
          si_[kIntHanded * kLaneNT] += 1u;
        }
      }
      const unsigned long long e = atomicAdd(io.out_count, 1ull);
      io.out[e] = Pre{__double_as_longlong(col[kColQ * kLaneNT]), 0.0, 0u, hidx};
      si_[kIntEvicted * kLaneNT] += 1u;
      si_[kIntCls * kLaneNT] += (unsigned)(Cb + nall + nall_next - 1);
      // (a restart repeats the lane's checks in the light tier)
      if (hidx == 0xffffffffu) si_[kIntWasted * kLaneNT] += (unsigned)(Cb + nall - 1);
      else si_[kIntChecks * kLaneNT] += (unsigned)(Ch - 1);  // (on the reference's path: the light tier goes on)
      state = 0;
    }
  }
  lane_flush(io, si_, kind);
}

// dynamic shared memory of one lane CTA: the columns, the 32-bit slots, the
// warps' claim words
constexpr size_t kLaneSmemBytes = (size_t)kLaneCol * kLaneNT * 8 + (size_t)kLaneInt * kLaneNT * 4 +
                                  (size_t)(kLaneNT / 32) * (2 * kLaneClaim * 8 + 4 * 4);

template <bool SEP0>
__global__ void __launch_bounds__(kLaneNT, TCCD_NMINB) lane_kernel(Args a, LaneIO io) {
  extern __shared__ __align__(16) unsigned char lane_smem[];
  double* const Ps = reinterpret_cast<double*>(lane_smem);
  long long* const Sq = reinterpret_cast<long long*>(Ps + kLaneCol * kLaneNT);
  unsigned* const Si = reinterpret_cast<unsigned*>(Sq + (kLaneNT / 32) * 2 * kLaneClaim);
  unsigned* const Sw = Si + kLaneInt * kLaneNT;
  const long long gt = (long long)blockIdx.x * kLaneNT + threadIdx.x;
  unsigned long long* lb = io.scratch + gt * kLaneScratchWords;
  double* col = Ps + threadIdx.x;
  unsigned* si = Si + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kLaneInt; ++i) si[i * kLaneNT] = 0u;
  const unsigned long long nvf = io.count[0], nee = io.count[1];
  // first kind of this warp: warps split between the kinds in proportion to
  // their queues; a warp whose queue runs dry moves to the other one
  const long long gw = gt >> 5, nw = (long long)gridDim.x * (kLaneNT / 32);
  int kind = (nvf + nee) > 0 && (unsigned long long)gw * (nvf + nee) < nee * (unsigned long long)nw;
  for (int pass = 0; pass < 2; ++pass, kind ^= 1)
    lane_loop<SEP0>(a, io, col, si, Sw + 4 * (threadIdx.x >> 5),
              Sq + (threadIdx.x >> 5) * 2 * kLaneClaim, lb, kind);
}

}  // namespace tccd
