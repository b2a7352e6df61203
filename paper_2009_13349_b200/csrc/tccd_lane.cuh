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
// written in the order the reference's stable t_lo sort gives them: push
// order for u / v splits; for a t split, per run of equal parent t_lo, all
// lower children then all upper children (the uppers wait in a third array
// until the run ends).
//
// A query leaves this tier (and restarts from its root in the light tier:
// exact, classification is a pure function of the box) when a level would
// exceed kLaneCap boxes or the lattice would exceed its index range.
#pragma once

namespace tccd {

#ifndef TCCD_KL
#define TCCD_KL 64
#endif
#ifndef TCCD_NNT
#define TCCD_NNT 128
#endif
#ifndef TCCD_NMINB
#define TCCD_NMINB 4
#endif
constexpr int kLaneCap = TCCD_KL;  // boxes per level of a lane query
constexpr int kLaneNT = TCCD_NNT;  // threads per CTA
constexpr int kLaneMaxSplits = 52;  // per dimension: midpoints stay exact (indices < 2^53)
constexpr int kLaneMaxLevel = 62;   // ti | ui | vi fits one 64-bit word

// A query queued for the lane tier by the prologue: its root box is
// non-disjoint and refined (one check done).
struct LaneRec {
  long long q;
  double wb;  // root hull width (the first record's codomain width)
  double eps[3];
  double kap[3];
  double sep, delta, t_max;
  long long mc;
};
static_assert(sizeof(LaneRec) == 96, "LaneRec layout");

struct LaneIO {
  const LaneRec* rec;             // vertex-face entries from the front, edge-edge from the back
  long long rec_cap;
  const unsigned long long* count;  // [2] entries per kind
  unsigned long long* next;         // [2] next entry to take per kind
  unsigned long long* scratch;      // [grid threads][3][kLaneCap] level words
  Pre* out;                         // light-tier queue (evicted queries restart there)
  unsigned long long* out_count;
  unsigned long long* stats;        // [8] see Counters::lane
};

// this thread's query coordinates: one column of a [24][NT] shared array
template <int NT>
struct ColP {
  const double* p;
  __device__ __forceinline__ double operator[](int k) const { return p[k * NT]; }
};

// box of lattice word pk at split counts (nt, nu, nv)
__device__ __forceinline__ Box lane_box(unsigned long long pk, int nt, int nu, int nv,
                                        double t_max) {
  const double wt = ldexp(t_max, -nt), wu = ldexp(1.0, -nu), wv = ldexp(1.0, -nv);
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
__device__ __forceinline__ int lane_split_dim(double wt, double wu, double wv, const double* kap) {
  const double ct = wt * kap[0], cu = wu * kap[1], cv = wv * kap[2];
  int sd = 0;
  double best = ct;
  if (cu > best) { sd = 1; best = cu; }
  if (cv > best) sd = 2;
  return sd;
}

// a recorded box (first / drop): lattice word, split counts, level, width, t_lo
struct LaneRecBox {
  unsigned long long pk;
  int shape;  // nt | nu << 8 | nv << 16
  int level;
  double codom;
  double t0;
};

// write record x (or y when !use_x), field by field (no addressable copy)
__device__ __forceinline__ void lane_write(const Args& a, long long q, bool use_x,
                                           const LaneRecBox& x, const LaneRecBox& y,
                                           double t_max, long long checks, int early) {
  const unsigned long long pk = use_x ? x.pk : y.pk;
  const int shape = use_x ? x.shape : y.shape;
  const Box b = lane_box(pk, shape & 255, (shape >> 8) & 255, shape >> 16, t_max);
  write_result(a, q, kHit, b, use_x ? x.codom : y.codom, checks, early, use_x ? x.level : y.level);
}

template <int KIND>
__device__ __forceinline__ void lane_loop(const Args& a, const LaneIO& io, double* colbase,
                                          unsigned long long* lb, unsigned long long (&st)[8]) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const ColP<kLaneNT> P{colbase};
  const unsigned long long total = io.count[KIND];
  bool dry = false;    // (warp-uniform) this kind's queue is empty
  bool active = false;
  // query
  long long q = 0, mc = 0, C = 0;
  double eps[3] = {0, 0, 0}, kap[3] = {0, 0, 0}, sep = 0, delta = 0, t_max = 1;
  // level
  int L = 0, nt = 0, nu = 0, nv = 0, sd = 0, ncur = 0, icur = 0, nn = 0, ntmp = 0, cb = 0;
  double wt = 1, wu = 1, wv = 1;
  bool col = false;
  unsigned long long run = ~0ull;
  LaneRecBox fr{}, dr{};
  bool hf = false, hd = false;

  for (;;) {
    // ---- refill idle lanes (warp-aggregated claim)
    const unsigned need = __ballot_sync(FULL, !active);
    if (need && !dry) {
      const int leader = __ffs(need) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(&io.next[KIND], (unsigned long long)__popc(need));
      base = __shfl_sync(FULL, base, leader);
      if (base + __popc(need) >= total) dry = true;
      if (!active) {
        const unsigned long long k = base + __popc(need & ((1u << lane) - 1u));
        if (k < total) {
          const LaneRec& r = io.rec[KIND ? io.rec_cap - 1 - (long long)k : (long long)k];
          q = r.q;
          const double2* src = reinterpret_cast<const double2*>(a.points + 24 * q);
#pragma unroll
          for (int i = 0; i < 12; ++i) {
            const double2 v = src[i];
            colbase[(2 * i) * kLaneNT] = v.x;
            colbase[(2 * i + 1) * kLaneNT] = v.y;
          }
          eps[0] = r.eps[0]; eps[1] = r.eps[1]; eps[2] = r.eps[2];
          kap[0] = r.kap[0]; kap[1] = r.kap[1]; kap[2] = r.kap[2];
          sep = r.sep; delta = r.delta; t_max = r.t_max; mc = r.mc;
          // the root (level 0, one check, the prologue's) is the first record
          // and was refined: level 1 = its two children (a root child is
          // never clipped: mid + 0 <= 1)
          fr.pk = 0; fr.shape = 0; fr.level = 0; fr.codom = r.wb; fr.t0 = 0.0;
          hf = true; hd = false;
          C = 1;
          nt = nu = nv = 0;
          wt = t_max; wu = 1.0; wv = 1.0;
          const int s0 = lane_split_dim(wt, wu, wv, kap);
          if (s0 == 0) { nt = 1; wt *= 0.5; } else if (s0 == 1) { nu = 1; wu *= 0.5; } else { nv = 1; wv *= 0.5; }
          cb = 0;
          lb[0] = 0ull;
          lb[1] = 1ull;
          ncur = 2; icur = 0; nn = 0; ntmp = 0;
          L = 1;
          col = false;
          run = ~0ull;
          sd = lane_split_dim(wt, wu, wv, kap);
          active = true;
        }
      }
    }
    if (!__any_sync(FULL, active)) break;
    if (!active) continue;

    // ---- one box of the current level, in visiting order
    unsigned long long* const cur = lb + cb;
    unsigned long long* const nxt = lb + (cb ^ kLaneCap);
    unsigned long long* const tmp = lb + 2 * kLaneCap;
    const unsigned long long pk = cur[icur];
    const int suv = nu + nv;
    const unsigned long long ti = pk >> suv;
    if (sd == 0) {
      // t-split level: a new run of equal t_lo starts; the previous run's
      // upper children follow its lower children
      if (ti != run) {
        for (int j = 0; j < ntmp; ++j) nxt[nn + j] = tmp[j];
        nn += ntmp;
        ntmp = 0;
        run = ti;
      }
    }
    Box b;
    b.t0 = (double)ti * wt; b.t1 = b.t0 + wt;
    b.u0 = (double)((pk >> nv) & ((1ull << nu) - 1ull)) * wu; b.u1 = b.u0 + wu;
    b.v0 = (double)(pk & ((1ull << nv) - 1ull)) * wv; b.v1 = b.v0 + wv;
    double wb;
    const int cls = classify_k<KIND, true>(P, b, eps, sep, wb);
    ++C;
    ++st[KIND];
    int outcome = 0;  // 0 continue, 1 ended (result written), 2 evict
    if (cls == kDisjoint) {
      // budget with boxes outstanding: the earliest record (_kernel.py:188-199)
      if (C >= mc && (hd || icur + 1 < ncur || nn + ntmp > 0)) {
        lane_write(a, q, hd && (!hf || dr.t0 < fr.t0), dr, fr, t_max, C, 1);
        outcome = 1;
      }
    } else {
      const LaneRecBox me{pk, nt | (nu << 8) | (nv << 16), L, wb, b.t0};
      if (!col) { fr = me; hf = true; }  // first colliding box of this level (:201-206)
      if (C >= mc) {                     // budget (:208-213)
        lane_write(a, q, hd && dr.t0 < fr.t0, dr, fr, t_max, C, 1);
        outcome = 1;
      } else if (wb < delta || cls == kContained) {  // accept (:215, 243-258)
        if (!col) {
          lane_write(a, q, hd && dr.t0 < b.t0, dr, me, t_max, C, 0);
          outcome = 1;
        } else if (!hd || b.t0 < dr.t0) {
          dr = me;
          hd = true;
        }
      } else if (nn + ntmp + 2 > kLaneCap) {
        outcome = 2;  // the next level outgrows this tier
      } else {
        // refine along the level's split dimension: insert the child bit
        const int pos = sd == 0 ? suv : (sd == 1 ? nv : 0);
        const unsigned long long lo = ((pk >> pos) << (pos + 1)) | (pk & ((1ull << pos) - 1ull));
        const unsigned long long hi = lo | (1ull << pos);
        if (sd == 0) {
          nxt[nn++] = lo;
          tmp[ntmp++] = hi;
        } else {
          nxt[nn++] = lo;
          // vertex-face: the upper child of a u / v split only inside u + v <= 1
          // (_kernel.py:276-310)
          bool push_hi = true;
          if (KIND == 0) {
            if (sd == 1) push_hi = 0.5 * (b.u0 + b.u1) + b.v0 <= 1.0;
            else push_hi = b.u0 + 0.5 * (b.v0 + b.v1) <= 1.0;
          }
          if (push_hi) nxt[nn++] = hi;
        }
      }
      col = true;
    }
    if (outcome == 0 && ++icur == ncur) {
      // ---- level end
      for (int j = 0; j < ntmp; ++j) nxt[nn + j] = tmp[j];
      nn += ntmp;
      ntmp = 0;
      if (nn == 0) {
        // queue exhausted (_kernel.py:321-324)
        if (hd) {
          lane_write(a, q, true, dr, dr, t_max, C, 0);
        } else {
          const Box z = {0, 0, 0, 0, 0, 0};
          write_result(a, q, kFree, z, 0.0, C, 0, 0);
        }
        outcome = 1;
      } else {
        cb ^= kLaneCap;
        ncur = nn;
        nn = 0;
        icur = 0;
        ++L;
        col = false;
        run = ~0ull;
        // every refining box of the level split along sd
        int ns;
        if (sd == 0) { ns = ++nt; wt *= 0.5; }
        else if (sd == 1) { ns = ++nu; wu *= 0.5; }
        else { ns = ++nv; wv *= 0.5; }
        if (ns > kLaneMaxSplits || L > kLaneMaxLevel) outcome = 2;
        sd = lane_split_dim(wt, wu, wv, kap);
      }
    }
    if (outcome == 1) {
      st[2 + KIND] += (unsigned long long)(C - 1);  // checks of finished queries (root: prologue's)
      st[4 + KIND] += 1;
      active = false;
    } else if (outcome == 2) {
      // restart from the root in the light tier (one self-contained record)
      const unsigned long long h = atomicAdd(io.out_count, 1ull);
      Pre& p = io.out[h];
      for (int k = 0; k < 24; ++k) p.P[k] = P[k];
      QueryParams qp;
      qp.eps[0] = eps[0]; qp.eps[1] = eps[1]; qp.eps[2] = eps[2];
      qp.kap[0] = kap[0]; qp.kap[1] = kap[1]; qp.kap[2] = kap[2];
      qp.sep = sep; qp.delta = delta; qp.t_max = t_max; qp.max_checks = mc;
      qp.kind = KIND; qp.tame = 1;
      p.qp = qp;
      p.q = q;
      p.wb = 0.0;
      p.flag = 0;
      p.pad = 0;
      st[6] += 1;
      st[7] += (unsigned long long)(C - 1);  // lane checks that the light tier repeats
      active = false;
    }
  }
}

__global__ void __launch_bounds__(kLaneNT, TCCD_NMINB) lane_kernel(Args a, LaneIO io) {
  __shared__ double Ps[24 * kLaneNT];
  const long long gt = (long long)blockIdx.x * kLaneNT + threadIdx.x;
  unsigned long long* lb = io.scratch + gt * 3 * kLaneCap;
  double* colbase = Ps + threadIdx.x;
  const unsigned long long nvf = io.count[0], nee = io.count[1];
  // first kind of this warp: warps split between the kinds in proportion to
  // their queues; a warp whose queue runs dry moves to the other one
  const long long gw = gt >> 5, nw = (long long)gridDim.x * (kLaneNT / 32);
  int kind = (nvf + nee) > 0 && (unsigned long long)gw * (nvf + nee) < nee * (unsigned long long)nw;
  unsigned long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int pass = 0; pass < 2; ++pass, kind ^= 1) {
    if (kind == 0) lane_loop<0>(a, io, colbase, lb, st);
    else lane_loop<1>(a, io, colbase, lb, st);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    unsigned long long v = st[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&io.stats[k], v);
  }
}

}  // namespace tccd
