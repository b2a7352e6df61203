// libtccd: batched Tight-Inclusion CCD on B200 (sm_100a), FP64, FMA-free.
//
// Reproduces the reference state machine (ccdkit._kernel.solve_kernel,
// pkg/src/ccdkit/_kernel.py:136-324) exactly for every query of a batch.
// Per library chunk (<= kChunk queries):
//
//  1. prologue_kernel, one thread per query: coalesced load of the 24
//     coordinates, parameter validation (core.py:176-184), filters
//     (inclusion.py:85-122), one evaluation of F at the domain's corners for
//     the kappas (_kernel.py:98-132) and the root-box check.  Queries decided
//     at the root are written out; survivors go to the lane queue (dyadic
//     t_max, tame coordinates) or the light queue.
//  2. lane_kernel (tccd_lane.cuh): one query per thread, box by box in the
//     reference's visiting order, for queries whose levels stay within 64
//     boxes; larger levels are handed over to the light tier.
//  3. engine_kernel tiers (tccd_engine.cuh) over the light queue, in
//     sub-chunks of <= kSub entries: persistent grids whose independent
//     groups keep several queries resident and advance them one BFS level
//     per round with lane-per-box classification:
//        light  : 128-thread CTA (5 per SM), 16 queries, levels <= 1024
//                 boxes, per-box bookkeeping in shared memory
//        medium : 256-thread CTA (2 per SM), 8 queries, levels <= 8192
//                 boxes, per-box bookkeeping in shared memory
//        giant  : 512-thread CTA per query, levels up to 2 * m_I boxes
//     A query whose level outgrows its tier moves to the next tier with that
//     level handed over (or restarts there if the handover pool is full).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <type_traits>

#include <cooperative_groups.h>

#include "tccd.h"
#include "tccd_device.cuh"

namespace cg = cooperative_groups;

namespace tccd {

struct Counters {
  // ---- per batch chunk (prologue, lane tier)
  unsigned long long light_count;    // light-queue entries: prologue survivors + lane evictions
  unsigned long long lane_count[2];  // lane-tier queue entries per kind (VF, EE)
  unsigned long long lane_next[2];   // next lane entry to take per kind
  // lane tier: [0..1] classifications VF / EE, [2..3] checks on the
  // reference's path (queries it finished or handed over; root check
  // excluded: the prologue's), [4..5] queries finished, [6] queries sent to
  // the light tier, [7] lane checks of those that restart there, [8] of
  // those, the ones handed over with their current level
  unsigned long long lane[10];
  unsigned long long lane_hand;      // lane-tier handover records used
  unsigned long long lane_pool;      // lane-tier handover pool boxes used
  // ---- per group-tier sub-chunk (zeroed before each)
  unsigned long long q_count[3];  // entries in the medium / giant queues ([0] unused: light_count)
  unsigned long long q_next[3];   // next entry to admit (light: within the sub-chunk's slice)
  unsigned long long rounds;      // engine rounds (diagnostics)
  unsigned long long deferred;    // level deferrals (diagnostics)
  unsigned long long evicted[3];  // evictions out of each tier (diagnostics)
  unsigned long long boxes[3];    // boxes handled per tier (diagnostics)
  unsigned long long pool[3];     // handover pool fill (tiers 1, 2)
  unsigned long long phase[3][16];  // cycles per engine phase (TCCD_PHASE_PROF builds)
  unsigned long long cls[3][2];   // box classifications per tier and kind (VF, EE)
  unsigned long long restarts[3];  // evictions out of tier k that found the handover pool full
  unsigned long long algo[3];      // checks of the reference's path done per group tier (signed sum)
};

// A queued query of a group tier: its index in the batch (the tier loads
// its coordinates and recomputes its constants) and its root class.
struct Pre {
  long long q;         // query index
  double wb;           // root hull width (valid when flag says non-disjoint)
  unsigned int flag;   // root class flag (0: not classified yet)
  unsigned int pad;    // light queue: index of the lane tier's handover (~0: none)
};
static_assert(sizeof(Pre) == 24, "Pre layout");

struct Rec {  // first / drop record of a query (_kernel.py:158-171)
  Box b;
  double codom;
  int level;
  int pad;
};

// Handover state of a query evicted to the next tier with its next level
// materialized (n > 0): the next tier resumes it instead of restarting.
struct Hand {
  long long C;       // checks done
  long long off;     // first box of the level in the tier's handover pool
  int level;         // BFS level of those boxes
  int n;             // boxes (0: restart from the root)
  Rec rec[2];        // first, drop
  unsigned char have_first, have_drop, pad[6];
};

struct Args {
  long long n;
  const double* points;
  const uint8_t* kind;
  int kind_all;
  const double* delta;
  double delta_all;
  const long long* max_checks;
  long long max_checks_all;
  long long max_checks_max;
  const double* sep;
  double sep_all;
  const double* t_max;
  double t_max_all;
  const double* eps;
  uint8_t* status;
  double* toi;
  double* tol;
  double* codom;
  long long* checks;
  uint8_t* early;
  double* witness;
  int* level;
  long long* stats;
  Counters* ctr;
  int heavy_only;
  int no_lane;
  long long* hit_index;    // optional compacted hit list (index, toi)
  double* hit_toi;
  unsigned long long* hit_count;
  long long hit_cap;
  long long hit_base;
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

__device__ __forceinline__ void write_result(const Args& a, long long q, uint8_t status,
                                             const Box& b, double codom, long long checks,
                                             int early, int level) {
  a.status[q] = status;
  const bool hit = status == kHit;
  if (hit && a.hit_index) {
    // compacted hit list: one atomic per group of converged hitting threads
    const cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(a.hit_count, (unsigned long long)g.size());
    base = g.shfl(base, 0) + g.thread_rank();
    if ((long long)base < a.hit_cap) {
      a.hit_index[base] = q + a.hit_base;
      a.hit_toi[base] = b.t0;
    }
  }
  a.toi[q] = hit ? b.t0 : __longlong_as_double(0x7ff0000000000000LL);
  if (a.tol) a.tol[q] = hit ? b.t1 - b.t0 : 0.0;
  if (a.codom) a.codom[q] = hit ? codom : 0.0;
  if (a.checks) a.checks[q] = checks;
  if (a.early) a.early[q] = (uint8_t)(hit ? early : 0);
  if (a.witness) {
    double* w = a.witness + 6 * q;
    if (hit) { w[0] = b.t0; w[1] = b.t1; w[2] = b.u0; w[3] = b.u1; w[4] = b.v0; w[5] = b.v1; }
    else { w[0] = w[1] = w[2] = w[3] = w[4] = w[5] = 0.0; }
  }
  if (a.level) a.level[q] = hit ? level : 0;
}

__device__ __forceinline__ void load_params(const Args& a, long long q, QueryParams& qp) {
  qp.kind = a.kind ? a.kind[q] : a.kind_all;
  qp.delta = a.delta ? a.delta[q] : a.delta_all;
  qp.max_checks = a.max_checks ? a.max_checks[q] : a.max_checks_all;
  qp.sep = a.sep ? a.sep[q] : a.sep_all;
  qp.t_max = a.t_max ? a.t_max[q] : a.t_max_all;
}

}  // namespace tccd

#include "tccd_lane.cuh"

namespace tccd {

// flag byte: bits 0-1 class, bit 2 accepted, bits 3-4 split dim, bit 5 upper
// child pushed, bit 6 classified
__device__ __forceinline__ uint8_t make_flag(int cls, bool acc, int sdim, bool push_hi) {
  return (uint8_t)(cls | (acc ? 4 : 0) | (sdim << 3) | (push_hi ? 32 : 0));
}

// (key, push) lexicographic "less than"
__device__ __forceinline__ bool kp_less(unsigned long long ka, unsigned int pa,
                                        unsigned long long kb, unsigned int pb) {
  return ka < kb || (ka == kb && pa < pb);
}

template <int NT>
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* sw,
                                                              unsigned long long& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long t = lane < NT / 32 ? sw[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < NT / 32) sw[lane] = t;
  }
  __syncthreads();
  const unsigned long long pre = w ? sw[w - 1] : 0ull;
  total = sw[NT / 32 - 1];
  __syncthreads();
  return pre + x - v;
}

// ===========================================================================
// prologue: one thread per query, root check, survivors compacted
// ===========================================================================
constexpr int kPrologueThreads = 128;

#ifndef TCCD_PRO_MINB
#define TCCD_PRO_MINB 4
#endif
__global__ void __launch_bounds__(kPrologueThreads, TCCD_PRO_MINB) prologue_kernel(Args a, long long lo,
                                                                    long long cnt, Pre* queue,
                                                                    unsigned long long* qcount,
                                                                    LaneRec* lq, long long lq_cap,
                                                                    unsigned long long* lcount) {
  __shared__ double tile[kPrologueThreads * 24];
  const long long base = lo + (long long)blockIdx.x * kPrologueThreads;
  const int nb = (int)min((long long)kPrologueThreads, lo + cnt - base);
  // coalesced staging of the block's 24-double records
  {
    // (cp.async: the tile's 12 x 16 bytes per thread are all in flight at
    // once, without a round trip through registers)
    const double2* src = reinterpret_cast<const double2*>(a.points + 24 * base);
    double2* dst = reinterpret_cast<double2*>(tile);
#ifdef TCCD_PRO_SYNC_LOAD
    for (int i = threadIdx.x; i < nb * 12; i += kPrologueThreads) dst[i] = src[i];
#else
    for (int i = threadIdx.x; i < nb * 12; i += kPrologueThreads) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + i);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + i) : "memory");
    }
#endif
  }
  // (the per-query parameters are loaded while the tile is in flight)
  const int t = threadIdx.x;
  QueryParams qp;
  if (t < nb) load_params(a, base + t, qp);
#ifndef TCCD_PRO_SYNC_LOAD
  asm volatile("cp.async.wait_all;\n" ::: "memory");
#endif
  __syncthreads();
  bool survive = false;
  int lane_kind = -1;  // survivor routed to the lane tier (its kind)
  Pre pre;
  LaneRec lr;
  if (t < nb) {
    const long long q = base + t;
    const double* P = tile + 24 * t;
    uint8_t st = kHit;
    if (!params_valid(qp.kind, qp.delta, qp.max_checks, qp.sep, qp.t_max) ||
        qp.max_checks > a.max_checks_max) {
      st = kErrParam;
    } else if (a.eps) {
      for (int i = 0; i < 24; ++i)
        if (!isfinite(P[i])) st = kErrNonfinite;
      qp.eps[0] = a.eps[3 * q];
      qp.eps[1] = a.eps[3 * q + 1];
      qp.eps[2] = a.eps[3 * q + 2];
    } else {
      st = filters(P, qp.kind, qp.sep, qp.eps);
    }
    const Box root = {0.0, qp.t_max, 0.0, 1.0, 0.0, 1.0};
    qp.tame = tame_coords(P);
    if (st != kHit) {
      write_result(a, q, st, root, 0.0, 0, 0, 0);
    } else {
      // one evaluation of F at the domain's corners gives the kappas and the
      // root box's hull
      double F[8][3];
      root_corners(P, qp.kind, qp.t_max, F);
      kappas_from(F, qp.kap);
      double wb;
      const int cls = classify_root(F, qp.eps, qp.sep, wb);
      if (cls == kDisjoint) {
        // the queue empties after one check (_kernel.py:188-199, 321-324)
        write_result(a, q, kFree, root, 0.0, 1, 0, 0);
      } else {
        int sdim; double mid; bool ph;
        const bool acc = split_decision(root, cls, wb, qp.kap, qp.delta, qp.kind, sdim, mid, ph);
        if (qp.max_checks <= 1) {
          write_result(a, q, kHit, root, wb, 1, 1, 0);  // budget (_kernel.py:208-213)
        } else if (acc) {
          write_result(a, q, kHit, root, wb, 1, 0, 0);  // accepted at the root
        } else {
          survive = true;
          int ex;
          // lane tier: dyadic t_max (lattice boxes) and tame coordinates
          if (lq && qp.tame && frexp(qp.t_max, &ex) == 0.5 && qp.t_max >= 0x1p-900) {
            lane_kind = qp.kind;
            lr.q = q;
            lr.wb = wb;
            for (int k = 0; k < 3; ++k) { lr.eps[k] = qp.eps[k]; lr.kap[k] = qp.kap[k]; }
          } else {
            pre.q = q;
            pre.wb = wb;
#ifdef TCCD_DEBUG_ROOT_UNCLASSIFIED
            pre.flag = 0;
#else
            pre.flag = make_flag(cls, acc, sdim, ph) | 64u;
#endif
            pre.pad = 0xffffffffu;
          }
        }
      }
    }
  }
  // warp-aggregated compaction: light-tier records, lane records per kind
  // (vertex-face from the front of the lane queue, edge-edge from the back)
  const int lane = threadIdx.x & 31;
  const unsigned int below = (1u << lane) - 1u;
  const unsigned int m = __ballot_sync(0xffffffffu, survive && lane_kind < 0);
  const unsigned int m0 = __ballot_sync(0xffffffffu, lane_kind == 0);
  const unsigned int m1 = __ballot_sync(0xffffffffu, lane_kind == 1);
  unsigned long long wb0 = 0, wb1 = 0, wb2 = 0;
  if (lane == 0) {
    if (m) wb0 = atomicAdd(qcount, (unsigned long long)__popc(m));
    if (m0) wb1 = atomicAdd(&lcount[0], (unsigned long long)__popc(m0));
    if (m1) wb2 = atomicAdd(&lcount[1], (unsigned long long)__popc(m1));
  }
  wb0 = __shfl_sync(0xffffffffu, wb0, 0);
  wb1 = __shfl_sync(0xffffffffu, wb1, 0);
  wb2 = __shfl_sync(0xffffffffu, wb2, 0);
  if (survive && lane_kind < 0) queue[wb0 + __popc(m & below)] = pre;
  if (lane_kind == 0) lq[wb1 + __popc(m0 & below)] = lr;
  if (lane_kind == 1) lq[lq_cap - 1 - (long long)(wb2 + __popc(m1 & below))] = lr;
}

}  // namespace tccd

#include "tccd_engine.cuh"

namespace tccd {

//                   G    NT   Q   CAP    QCAP   ADMIT  SMEM   MINB
#ifndef TCCD_LQ
#define TCCD_LQ 16
#endif
#ifndef TCCD_LADMIT
#define TCCD_LADMIT 1280
#endif
#ifndef TCCD_LQCAP
#define TCCD_LQCAP 1024
#endif
#ifndef TCCD_MSMEM
#define TCCD_MSMEM 1
#endif
#ifndef TCCD_LNT
#define TCCD_LNT 128
#endif
#ifndef TCCD_LCAP
#define TCCD_LCAP 3840
#endif
#ifndef TCCD_LMINB
#define TCCD_LMINB 5
#endif
#ifndef TCCD_LG
#define TCCD_LG TCCD_LNT
#endif
using LightCfg = EngineCfg<TCCD_LG, TCCD_LNT, TCCD_LQ, TCCD_LCAP, TCCD_LQCAP, TCCD_LADMIT, true,
                           TCCD_LMINB>;
#ifndef TCCD_MNT
#define TCCD_MNT 256
#endif
#ifndef TCCD_MQ
#define TCCD_MQ 8
#endif
#ifndef TCCD_MCAP
#define TCCD_MCAP 16384
#endif
#ifndef TCCD_MADMIT
#define TCCD_MADMIT 8192
#endif
#ifndef TCCD_MMINB
#define TCCD_MMINB 2
#endif
#if TCCD_MSMEM
using MediumCfg = EngineCfg<TCCD_MNT, TCCD_MNT, TCCD_MQ, TCCD_MCAP, 8192, TCCD_MADMIT, true,
                            TCCD_MMINB>;
#else
using MediumCfg = EngineCfg<512, 512, 16, 65536, 32768, 16384, false, 1>;
#endif
#ifndef TCCD_GNT
#define TCCD_GNT 512
#endif
#ifndef TCCD_GMINB
#define TCCD_GMINB 1
#endif
using GiantCfg = EngineCfg<TCCD_GNT, TCCD_GNT, 1, 0, 0, 0, false, TCCD_GMINB>;

template <class Cfg>
constexpr int groups_per_cta() { return Cfg::NT / Cfg::G; }

// Diagnostic counters of one group-tier sub-chunk (and, with batch != 0,
// of the chunk's prologue and lane tier) added to the caller's stats.
__global__ void stats_kernel(Args a, int heavy_only, long long cnt, int batch, long long sub_base,
                             long long sub_len) {
  if (threadIdx.x == 0 && a.stats) {
    const Counters& c = *a.ctr;
    long long* S = a.stats;
    const long long in_sub = (long long)c.light_count - sub_base;
    S[TCCD_STAT_GIANT_QUERIES] +=
        heavy_only ? (in_sub < 0 ? 0 : (in_sub < sub_len ? in_sub : sub_len)) : (long long)c.evicted[1];
    S[TCCD_STAT_ROUNDS] += (long long)c.rounds;
    S[TCCD_STAT_DEFERRALS] += (long long)c.deferred;
    S[TCCD_STAT_MEDIUM_QUERIES] += (long long)c.evicted[0];
    for (int k = 0; k < 3; ++k) S[TCCD_STAT_BOXES + k] += (long long)c.boxes[k];
    for (int k = 0; k < 6; ++k) S[TCCD_STAT_CLS + k] += (long long)c.cls[k / 2][k % 2];
    for (int k = 0; k < 2; ++k) {
      S[TCCD_STAT_POOL_DEMAND + k] += (long long)c.pool[1 + k];
      S[TCCD_STAT_RESTARTS + k] += (long long)c.restarts[k];
    }
    for (int k = 0; k < 3; ++k) S[TCCD_STAT_TIER_CHECKS + k] += (long long)c.algo[k];
    if (batch) {
      S[TCCD_STAT_LANE_QUERIES] += (long long)(c.lane_count[0] + c.lane_count[1]);
      for (int k = 0; k < 2; ++k) {
        S[TCCD_STAT_LANE_CLS + k] += (long long)c.lane[k];
        S[TCCD_STAT_LANE_CHECKS + k] += (long long)c.lane[2 + k];
        S[TCCD_STAT_LANE_DONE + k] += (long long)c.lane[4 + k];
      }
      S[TCCD_STAT_LANE_EVICTED] += (long long)c.lane[6];
      S[TCCD_STAT_LANE_WASTED] += (long long)c.lane[7];
      S[TCCD_STAT_LANE_HANDED] += (long long)c.lane[8];
      // survivors of the root check: the lane queue plus the prologue's
      // light-queue entries (the lane tier's evictions joined that queue)
      const unsigned long long into_light = c.light_count - c.lane[6];
      S[TCCD_STAT_PROLOGUE_DONE] +=
          cnt - (long long)(c.lane_count[0] + c.lane_count[1] + into_light);
      S[TCCD_STAT_CHUNKS] += 1;
    }
  }
}

// Device -> mapped pinned host copy as a kernel (tccd_copy_to_host): 16-byte
// stores when both ends are 16-byte aligned, bytes otherwise.
__global__ void copy_out_kernel(const unsigned char* src, unsigned char* dst, long long bytes) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const bool vec = (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
  const long long n16 = vec ? bytes / 16 : 0;
  for (long long i = t; i < n16; i += stride)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (long long i = n16 * 16 + t; i < bytes; i += stride) dst[i] = src[i];
}

// The same for the first min(*count, max_elems) elements of an array whose
// length a kernel wrote (a compacted hit list): only those bytes cross.
__global__ void copy_counted_kernel(const unsigned char* src, unsigned char* dst, long long elem,
                                    const unsigned long long* count, long long max_elems,
                                    unsigned long long* host_count) {
  const unsigned long long c = *count;
  const long long n = (long long)(c < (unsigned long long)max_elems ? c : (unsigned long long)max_elems);
  const long long bytes = n * elem;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (t == 0 && host_count) *host_count = c;
  const bool vec = (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
  const long long n16 = vec ? bytes / 16 : 0;
  for (long long i = t; i < n16; i += stride)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (long long i = n16 * 16 + t; i < bytes; i += stride) dst[i] = src[i];
}

// Admission order of the giant tier's queue: largest handed-over level
// first (longest-processing-time-first, so the heaviest queries do not start
// last and leave the other SMs idle).  Only a scheduling order: every query's
// result is independent of it.  Queues up to kOrderMax are sorted exactly
// (bitonic, one CTA); longer ones are ordered by a counting sort on the
// level size's power of two (descending; arbitrary within a bucket), up to
// the sub-chunk's capacity.
constexpr int kOrderMax = 4096;
__global__ void __launch_bounds__(1024) order_kernel(const Hand* hand,
                                                     const unsigned long long* count,
                                                     unsigned int* perm, long long cap) {
  __shared__ unsigned long long key[kOrderMax];
  __shared__ unsigned int bucket[33];
  const unsigned long long n = *count;
  if (n < 2) return;
  if (n > (unsigned long long)kOrderMax) {
    if (n > (unsigned long long)cap) return;
    // bucket b holds the entries with 2^(32-b-1) <= level boxes < 2^(32-b) (b = 32: no level)
    auto bkt = [&](unsigned long long i) -> int {
      const int h = hand[i].n;
      return h > 0 ? __clz(h) : 32;
    };
    for (int i = threadIdx.x; i < 33; i += blockDim.x) bucket[i] = 0;
    __syncthreads();
    for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&bucket[bkt(i)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int sum = 0;
      for (int k = 0; k < 33; ++k) {
        const unsigned int c = bucket[k];
        bucket[k] = sum;
        sum += c;
      }
    }
    __syncthreads();
    for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x)
      perm[atomicAdd(&bucket[bkt(i)], 1u)] = (unsigned int)i;
    return;
  }
  int P = 2;
  while (P < (int)n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const unsigned int w = i < (int)n && hand[i].n > 0 ? (unsigned int)hand[i].n : 0u;
    key[i] = i < (int)n ? ((unsigned long long)(0xffffffffu - w) << 32) | (unsigned int)i : ~0ull;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = key[i], b = key[l];
          if (((i & k) == 0) == (a > b)) { key[i] = b; key[l] = a; }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < (int)n; i += blockDim.x) perm[i] = (unsigned int)(key[i] & 0xffffffffu);
}

}  // namespace tccd

// ===========================================================================
// host side
// ===========================================================================
using namespace tccd;

namespace {

#ifndef TCCD_CHUNK
#define TCCD_CHUNK (1LL << 26)
#endif
#ifndef TCCD_SUB
#define TCCD_SUB (1LL << 23)
#endif
#ifndef TCCD_POOL
#define TCCD_POOL (1LL << 25)
#endif
// A call is split into chunks of at most kChunk queries: prologue and lane
// tier over the whole chunk (one launch each: the lane tier's tail -- lanes
// idle while the last queries finish -- is paid once per chunk), then the
// group tiers over the chunk's light queue in sub-chunks of kSub entries
// (their queues, handover records and pools are sized by the sub-chunk).
constexpr long long kChunk = TCCD_CHUNK;
constexpr long long kSub = TCCD_SUB;
constexpr long long kPoolDefault = TCCD_POOL;  // handover pool boxes per tier transition

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  return dev;
}

int device_sm_count(int hint) {
  if (hint > 0) return hint;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device()) != cudaSuccess)
    return 148;
  return sms > 0 ? sms : 148;
}

long long giant_cap(long long mcmax) { return 2 * mcmax + 2; }

#ifndef TCCD_LANE_HAND
#define TCCD_LANE_HAND (1LL << 21)
#endif
constexpr long long kLaneHandMax = TCCD_LANE_HAND;  // lane-tier handover records per chunk
#ifndef TCCD_LANE_POOL
#define TCCD_LANE_POOL (1LL << 26)
#endif
constexpr long long kLanePoolDefault = TCCD_LANE_POOL;  // lane-tier handover pool boxes per chunk

struct Layout {
  size_t ctr, light_q, lq, lscratch, queue[3], hand[3], pbox[3], pflag[3], perm, light, medium,
      giant, total;
  long long hand0;
  size_t light_b, medium_b, giant_b;
  long long chunk, sub, pool[3];
  int light_blocks, medium_blocks, giant_blocks, lane_blocks;
};

// Everything scales with the chunk (min(n, kChunk) queries) and the
// sub-chunk (min(chunk, kSub)): queues, lane scratch, one group per query at
// most in every tier, and handover pools no larger than the sub-chunk's
// largest possible handover (a query leaves the light tier with at most
// 2 * LightCfg::QCAP boxes, the medium tier with at most 2 * MediumCfg::QCAP).
Layout layout(long long n, long long mcmax, int giant_blocks, int sms, long long pool_boxes) {
  Layout L;
  const long long chunk = n < kChunk ? (n > 0 ? n : 1) : kChunk;
  const long long sub = chunk < kSub ? chunk : kSub;
  L.chunk = chunk;
  L.sub = sub;
  const long long pool = pool_boxes > 0 ? pool_boxes : kPoolDefault;
  L.pool[0] = std::min(pool_boxes > 0 ? pool_boxes : kLanePoolDefault, chunk * kLaneArr);
  L.hand0 = std::min(chunk, kLaneHandMax);
  L.pool[1] = std::min(pool, sub * 2 * LightCfg::QCAP);
  L.pool[2] = std::min(pool, sub * 2 * MediumCfg::QCAP);
  L.lane_blocks = (int)std::min<long long>((long long)TCCD_NMINB * sms, (chunk + kLaneNT - 1) / kLaneNT);
  L.light_blocks = (int)std::min<long long>((long long)TCCD_LMINB * sms, sub);
  L.medium_blocks = (int)std::min<long long>((long long)MediumCfg::MINB * sms, sub);
  L.giant_blocks = (int)std::min<long long>(giant_blocks, sub);
  L.light_b = align256(EngineArena<LightCfg>::bytes(LightCfg::CAP));
  L.medium_b = align256(EngineArena<MediumCfg>::bytes(MediumCfg::CAP));
  L.giant_b = align256(EngineArena<GiantCfg>::bytes(giant_cap(mcmax)));
  size_t o = 0;
  L.ctr = o; o += align256(sizeof(Counters));
  // per chunk
  L.light_q = o; o += align256((size_t)chunk * sizeof(Pre));
  L.lq = o; o += align256((size_t)chunk * sizeof(LaneRec));
  L.lscratch = o; o += align256((size_t)L.lane_blocks * kLaneNT * kLaneScratchWords * 8);
  L.hand[0] = o; o += align256((size_t)L.hand0 * sizeof(Hand));
  L.pbox[0] = o; o += align256((size_t)L.pool[0] * sizeof(Box));
  L.pflag[0] = o; o += align256((size_t)L.pool[0]);
  // per sub-chunk
  L.queue[0] = L.light_q;
  for (int k = 1; k < 3; ++k) {
    L.queue[k] = o; o += align256((size_t)sub * sizeof(Pre));
    L.hand[k] = o; o += align256((size_t)sub * sizeof(Hand));
    L.pbox[k] = o; o += align256((size_t)L.pool[k] * sizeof(Box));
    L.pflag[k] = o; o += align256((size_t)L.pool[k]);
  }
  L.perm = o; o += align256((size_t)sub * 4);
  L.light = o; o += L.light_b * (size_t)L.light_blocks * groups_per_cta<LightCfg>();
  L.medium = o; o += L.medium_b * (size_t)L.medium_blocks * groups_per_cta<MediumCfg>();
  L.giant = o; o += L.giant_b * (size_t)L.giant_blocks;
  L.total = o;
  return L;
}

// the dynamic shared-memory limit is a per-device attribute of the function
template <class Cfg>
int configure() {
  static bool done[256] = {};
  const int dev = current_device();
  if (dev >= 0 && dev < 256 && done[dev]) return TCCD_OK;
  const int smem = (int)(engine_smem_bytes<Cfg>() * groups_per_cta<Cfg>());
  if (cudaFuncSetAttribute(engine_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem) != cudaSuccess)
    return TCCD_E_CUDA;
  if (dev >= 0 && dev < 256) done[dev] = true;
  return TCCD_OK;
}

int configure_lane() {
  static bool done[256] = {};
  const int dev = current_device();
  if (dev >= 0 && dev < 256 && done[dev]) return TCCD_OK;
  if (cudaFuncSetAttribute(lane_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kLaneSmemBytes) != cudaSuccess ||
      cudaFuncSetAttribute(lane_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kLaneSmemBytes) != cudaSuccess)
    return TCCD_E_CUDA;
  if (dev >= 0 && dev < 256) done[dev] = true;
  return TCCD_OK;
}

template <class Cfg>
int launch_tier(const Args& a, const TierIO& io, int blocks, cudaStream_t st) {
  if (configure<Cfg>() != TCCD_OK) return TCCD_E_CUDA;
  engine_kernel<Cfg><<<blocks, Cfg::NT, engine_smem_bytes<Cfg>() * groups_per_cta<Cfg>(), st>>>(a, io);
  return cudaGetLastError() == cudaSuccess ? TCCD_OK : TCCD_E_CUDA;
}

// tccd_solve_kernel's cached device scratch, per device
struct ScratchCache {
  unsigned char* buf = nullptr;
  size_t bytes = 0;
};
std::mutex g_sk_mutex;
ScratchCache g_sk[256];

}  // namespace

extern "C" {

int tccd_abi_version(void) { return TCCD_ABI_VERSION; }

int tccd_copy_to_host(const void* src, void* host_dst, int64_t bytes, void* stream) {
  if (bytes < 0) return TCCD_E_N;
  if (bytes == 0) return TCCD_OK;
  if (!src || !host_dst) return TCCD_E_NULL;
  void* dst = nullptr;
  if (cudaHostGetDevicePointer(&dst, host_dst, 0) != cudaSuccess || !dst) {
    cudaGetLastError();  // (clear: the caller falls back to a copy-engine transfer)
    return TCCD_E_CUDA;
  }
  const long long n16 = bytes / 16;
  const int blocks = (int)min(2LL * device_sm_count(0), max(1LL, (n16 + 255) / 256));
  copy_out_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (const unsigned char*)src, (unsigned char*)dst, (long long)bytes);
  return cudaGetLastError() == cudaSuccess ? TCCD_OK : TCCD_E_CUDA;
}

int tccd_copy_counted_to_host(const void* src, void* host_dst, int64_t elem_bytes,
                              const uint64_t* count, int64_t max_elems, void* host_count,
                              void* stream) {
  if (elem_bytes <= 0 || max_elems < 0) return TCCD_E_N;
  if (!src || !host_dst || !count) return TCCD_E_NULL;
  void* dst = nullptr;
  void* dcount = nullptr;
  if (cudaHostGetDevicePointer(&dst, host_dst, 0) != cudaSuccess || !dst ||
      (host_count && (cudaHostGetDevicePointer(&dcount, host_count, 0) != cudaSuccess || !dcount))) {
    cudaGetLastError();
    return TCCD_E_CUDA;
  }
  const long long n16 = (max_elems * elem_bytes) / 16;
  const int blocks = (int)min(2LL * device_sm_count(0), max(1LL, (n16 + 255) / 256));
  copy_counted_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (const unsigned char*)src, (unsigned char*)dst, (long long)elem_bytes,
      (const unsigned long long*)count, (long long)max_elems, (unsigned long long*)dcount);
  return cudaGetLastError() == cudaSuccess ? TCCD_OK : TCCD_E_CUDA;
}

const char* tccd_error_string(int code) {
  switch (code) {
    case TCCD_OK: return "ok";
    case TCCD_E_NULL: return "a required pointer is NULL";
    case TCCD_E_N: return "n must be >= 0";
    case TCCD_E_DELTA: return "delta must be positive and finite";
    case TCCD_E_MAXCHECKS: return "max_checks must be >= 1";
    case TCCD_E_TMAX: return "t_max must lie in (0, 1]";
    case TCCD_E_SEPARATION: return "separation must be >= 0 and finite";
    case TCCD_E_KIND: return "kind must be 0 (vertex-face) or 1 (edge-edge)";
    case TCCD_E_WORKSPACE: return "workspace missing or smaller than tccd_workspace_bytes()";
    case TCCD_E_CUDA: return "CUDA runtime error";
    case TCCD_E_STRUCT: return "tccd_batch struct_size mismatch (ABI version skew)";
    case TCCD_E_CAPACITY: return "max_checks_max too large for the workspace layout";
    default: return "unknown tccd error";
  }
}

size_t tccd_workspace_bytes_ex(int64_t n, int64_t max_checks_max, int32_t heavy_blocks,
                               int64_t pool_boxes) {
  if (n < 0 || max_checks_max < 1 || pool_boxes < 0) return 0;
  const int sms = device_sm_count(0);
  const int gb = heavy_blocks > 0 ? heavy_blocks : sms;
  return layout(n, max_checks_max, gb, sms, pool_boxes).total;
}

size_t tccd_workspace_bytes(int64_t n, int64_t max_checks_max, int32_t heavy_blocks) {
  return tccd_workspace_bytes_ex(n, max_checks_max, heavy_blocks, 0);
}

int tccd_solve_batch(const tccd_batch* b_in, void* stream) {
  if (!b_in) return TCCD_E_NULL;
  if (b_in->struct_size != sizeof(tccd_batch)) return TCCD_E_STRUCT;
  tccd_batch* out_b = const_cast<tccd_batch*>(b_in);
  out_b->launches = 0;
  out_b->events_used = 0;
  const tccd_batch* b = b_in;
  if (b->n < 0) return TCCD_E_N;
  if (b->n > 0 && (!b->points || !b->status || !b->toi)) return TCCD_E_NULL;
  if (!b->delta && !(b->delta_all > 0.0 && b->delta_all < 1.0 / 0.0)) return TCCD_E_DELTA;
  if (!b->max_checks && b->max_checks_all < 1) return TCCD_E_MAXCHECKS;
  if (!b->t_max && !(b->t_max_all > 0.0 && b->t_max_all <= 1.0)) return TCCD_E_TMAX;
  if (!b->separation && !(b->separation_all >= 0.0 && b->separation_all < 1.0 / 0.0))
    return TCCD_E_SEPARATION;
  if (!b->kind && b->kind_all != 0 && b->kind_all != 1) return TCCD_E_KIND;
  const long long mcmax = b->max_checks ? b->max_checks_max : b->max_checks_all;
  if (b->max_checks && mcmax < 1) return TCCD_E_MAXCHECKS;
  if (giant_cap(mcmax) > (long long)kRefSrcMask) return TCCD_E_CAPACITY;
  if (b->pool_boxes < 0) return TCCD_E_WORKSPACE;
  if (b->hit_index && (!b->hit_toi || !b->hit_count || b->hit_capacity < 0)) return TCCD_E_NULL;
  const int sms = device_sm_count(b->device_sms);
  const int gb = b->heavy_blocks > 0 ? b->heavy_blocks : sms;
  const Layout L = layout(b->n, mcmax, gb, sms, b->pool_boxes);
  if (!b->workspace || b->workspace_bytes < L.total) return TCCD_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  if (b->stats && cudaMemsetAsync(b->stats, 0, TCCD_NUM_STATS * sizeof(int64_t), st) != cudaSuccess)
    return TCCD_E_CUDA;
  if (b->n == 0) return TCCD_OK;
  unsigned char* ws = (unsigned char*)b->workspace;

  Args a;
  memset(&a, 0, sizeof(a));
  a.n = b->n;
  a.points = b->points;
  a.kind = b->kind;
  a.kind_all = b->kind_all;
  a.delta = b->delta;
  a.delta_all = b->delta_all;
  a.max_checks = (const long long*)b->max_checks;
  a.max_checks_all = b->max_checks_all;
  a.max_checks_max = mcmax;
  a.sep = b->separation;
  a.sep_all = b->separation_all;
  a.t_max = b->t_max;
  a.t_max_all = b->t_max_all;
  a.eps = b->eps;
  a.status = b->status;
  a.toi = b->toi;
  a.tol = b->tol;
  a.codom = b->codom;
  a.checks = (long long*)b->checks;
  a.early = b->early;
  a.witness = b->witness;
  a.level = b->level;
  a.stats = (long long*)b->stats;
  a.ctr = (Counters*)(ws + L.ctr);
  a.heavy_only = (b->flags & TCCD_FLAG_HEAVY_ONLY) ? 1 : 0;
  a.no_lane = (b->flags & TCCD_FLAG_NO_LANE) ? 1 : 0;
  a.hit_index = (long long*)b->hit_index;
  a.hit_toi = b->hit_toi;
  a.hit_count = (unsigned long long*)b->hit_count;
  a.hit_cap = b->hit_capacity;
  a.hit_base = b->hit_index_base;
  const bool lanes = !a.heavy_only && !a.no_lane;

  Pre* queue[3];
  for (int k = 0; k < 3; ++k) queue[k] = (Pre*)(ws + L.queue[k]);
  Counters* const ctr = a.ctr;
  // group tier `tier` over sub-chunk `sub` of the chunk's light queue
  auto io_for = [&](int tier, long long sub) {
    TierIO io;
    // (heavy-only: the giant tier reads the prologue's queue directly)
    const bool from_light = tier == 0 || a.heavy_only;
    io.in = from_light ? queue[0] : queue[tier];
    io.in_count = from_light ? &ctr->light_count : &ctr->q_count[tier];
    io.in_base = from_light ? sub * L.sub : 0;
    io.in_limit = from_light ? L.sub : (long long)(1ull << 62);
    io.in_next = &ctr->q_next[tier];
    // (light: the lane tier's handovers, indexed by the queue records)
    io.in_hand = !a.heavy_only && (tier > 0 || lanes) ? (const Hand*)(ws + L.hand[tier]) : nullptr;
    io.hand_in_record = tier == 0;
    io.in_pbox = !a.heavy_only && (tier > 0 || lanes) ? (const Box*)(ws + L.pbox[tier]) : nullptr;
    io.in_pflag = !a.heavy_only && (tier > 0 || lanes) ? (const uint8_t*)(ws + L.pflag[tier]) : nullptr;
    io.in_pool_cap = L.pool[tier];
    // (light tier: the lane tier's evictions restart there and are known to
    // reach levels above kLaneCap boxes: admit them as if they had that many)
    io.in_maxsz = a.heavy_only ? 1
                  : (tier == 0 ? (lanes ? kLaneArr : 1)
                               : 2 * (tier == 1 ? LightCfg::QCAP : MediumCfg::QCAP));
    io.in_perm = tier == 2 && !a.heavy_only ? (const unsigned int*)(ws + L.perm) : nullptr;
    io.perm_max = L.sub;
    io.out_hand = tier < 2 ? (Hand*)(ws + L.hand[tier + 1]) : nullptr;
    io.out_pbox = tier < 2 ? (Box*)(ws + L.pbox[tier + 1]) : nullptr;
    io.out_pflag = tier < 2 ? (uint8_t*)(ws + L.pflag[tier + 1]) : nullptr;
    io.out_pool_count = tier < 2 ? &ctr->pool[tier + 1] : nullptr;
    io.pool_cap = tier < 2 ? L.pool[tier + 1] : 0;
    io.out = tier < 2 ? queue[tier + 1] : nullptr;
    io.out_count = tier < 2 ? &ctr->q_count[tier + 1] : nullptr;
    io.rounds = &ctr->rounds;
    io.deferred = &ctr->deferred;
    io.evicted = &ctr->evicted[tier];
    io.boxes = &ctr->boxes[tier];
    io.phase = ctr->phase[tier];
    io.cls = ctr->cls[tier];
    io.restarts = &ctr->restarts[tier];
    io.algo = &ctr->algo[tier];
    if (tier == 0) { io.arenas = ws + L.light; io.arena_bytes = L.light_b; io.cap = LightCfg::CAP; }
    if (tier == 1) { io.arenas = ws + L.medium; io.arena_bytes = L.medium_b; io.cap = MediumCfg::CAP; }
    if (tier == 2) { io.arenas = ws + L.giant; io.arena_bytes = L.giant_b; io.cap = giant_cap(mcmax); }
    return io;
  };
  LaneIO lio;
  lio.rec = (const LaneRec*)(ws + L.lq);
  lio.rec_cap = L.chunk;
  lio.count = ctr->lane_count;
  lio.next = ctr->lane_next;
  lio.scratch = (unsigned long long*)(ws + L.lscratch);
  lio.out = queue[0];
  lio.out_count = &ctr->light_count;
  lio.stats = ctr->lane;
  lio.hand = (Hand*)(ws + L.hand[0]);
  lio.hand_cap = L.hand0;
  lio.hand_count = &ctr->lane_hand;
  lio.pbox = (Box*)(ws + L.pbox[0]);
  lio.pflag = (uint8_t*)(ws + L.pflag[0]);
  lio.pool_cap = L.pool[0];
  lio.pool_count = &ctr->lane_pool;

  // optional caller events, one after each stage launch, in launch order
  int n_ev = 0;
  auto mark = [&](int stage) {
    if (!b->events || n_ev >= b->n_events) return cudaSuccess;
    const cudaError_t e = cudaEventRecord((cudaEvent_t)b->events[n_ev], st);
    if (b->event_stage) b->event_stage[n_ev] = stage;
    ++n_ev;
    return e;
  };
  const size_t sub_off = offsetof(Counters, q_count);
  long long launches = 0;
  for (long long lo = 0; lo < b->n; lo += kChunk) {
    const long long cnt = b->n - lo < kChunk ? b->n - lo : kChunk;
    if (cudaMemsetAsync(ctr, 0, sizeof(Counters), st) != cudaSuccess) return TCCD_E_CUDA;
    // prologue, one launch per input-ready piece (the whole chunk without
    // input events)
    const long long piece = b->input_events && b->input_chunk > 0 ? b->input_chunk : cnt;
    for (long long p0 = lo; p0 < lo + cnt; p0 += piece) {
      const long long pc = std::min(piece, lo + cnt - p0);
      if (b->input_events) {
        const long long c = p0 / b->input_chunk;
        if (c < b->n_input_events && b->input_events[c] &&
            cudaStreamWaitEvent(st, (cudaEvent_t)b->input_events[c], 0) != cudaSuccess)
          return TCCD_E_CUDA;
      }
      const unsigned pblocks = (unsigned)((pc + kPrologueThreads - 1) / kPrologueThreads);
      prologue_kernel<<<pblocks, kPrologueThreads, 0, st>>>(
          a, p0, pc, queue[0], &ctr->light_count, lanes ? (LaneRec*)(ws + L.lq) : nullptr,
          L.chunk, ctr->lane_count);
      ++launches;
      if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
    }
    if (mark(TCCD_STAGE_PROLOGUE) != cudaSuccess) return TCCD_E_CUDA;
    if (lanes) {
      if (configure_lane() != TCCD_OK) return TCCD_E_CUDA;
      // (every query of the call at separation 0: the hull is compared as is)
      if (!a.sep && a.sep_all == 0.0) lane_kernel<true><<<L.lane_blocks, kLaneNT, kLaneSmemBytes, st>>>(a, lio);
      else lane_kernel<false><<<L.lane_blocks, kLaneNT, kLaneSmemBytes, st>>>(a, lio);
      ++launches;
      if (cudaGetLastError() != cudaSuccess || mark(TCCD_STAGE_LANE) != cudaSuccess)
        return TCCD_E_CUDA;
    }
    // group tiers over the light queue, sub-chunk by sub-chunk (a sub-chunk
    // past the queue's end exits at once: the count is only known on the device)
    const long long nsub = (cnt + L.sub - 1) / L.sub;
    for (long long sub = 0; sub < nsub; ++sub) {
      if (cudaMemsetAsync((unsigned char*)ctr + sub_off, 0, sizeof(Counters) - sub_off, st) !=
          cudaSuccess)
        return TCCD_E_CUDA;
#ifdef TCCD_PHASE_PROF
      for (int k = 0; k < 3; ++k)  // phase[k][14] is a running min (start time)
        if (cudaMemsetAsync(&ctr->phase[k][14], 0xFF, 8, st) != cudaSuccess) return TCCD_E_CUDA;
#endif
      int rc;
      if (!a.heavy_only) {
        if ((rc = launch_tier<LightCfg>(a, io_for(0, sub), L.light_blocks, st)) != TCCD_OK) return rc;
        ++launches;
        if (mark(TCCD_STAGE_LIGHT) != cudaSuccess) return TCCD_E_CUDA;
        if ((rc = launch_tier<MediumCfg>(a, io_for(1, sub), L.medium_blocks, st)) != TCCD_OK) return rc;
        ++launches;
        if (mark(TCCD_STAGE_MEDIUM) != cudaSuccess) return TCCD_E_CUDA;
        order_kernel<<<1, 1024, 0, st>>>((const Hand*)(ws + L.hand[2]), &ctr->q_count[2],
                                         (unsigned int*)(ws + L.perm), L.sub);
        ++launches;
        if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
      }
      if ((rc = launch_tier<GiantCfg>(a, io_for(2, sub), L.giant_blocks, st)) != TCCD_OK) return rc;
      ++launches;
      if (mark(TCCD_STAGE_GIANT) != cudaSuccess) return TCCD_E_CUDA;
      if (a.stats) {
        stats_kernel<<<1, 32, 0, st>>>(a, a.heavy_only, cnt, sub == 0 ? 1 : 0, sub * L.sub, L.sub);
        ++launches;
        if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
      }
    }
  }
  out_b->events_used = n_ev;
  out_b->launches = launches;
  return TCCD_OK;
}

int tccd_solve_kernel(const double* s, const double* e, int kind, double t_max, double delta,
                      int64_t max_checks, double sep, double ex, double ey, double ez,
                      double* out13) {
  if (!s || !e || !out13) return TCCD_E_NULL;
  if (kind != 0 && kind != 1) return TCCD_E_KIND;
  if (max_checks < 1) return TCCD_E_MAXCHECKS;
  double hpts[24], heps[3] = {ex, ey, ez};
  memcpy(hpts, s, 12 * sizeof(double));
  memcpy(hpts + 12, e, 12 * sizeof(double));
  const int gb = 1;
  const size_t ws_bytes = tccd_workspace_bytes(1, max_checks, gb);
  const size_t in_b = 256, out_b = 256;  // inputs | outputs | workspace
  std::lock_guard<std::mutex> lock(g_sk_mutex);
  const int dev = current_device();
  if (dev < 0 || dev >= 256) return TCCD_E_CUDA;
  ScratchCache& sc = g_sk[dev];
  if (sc.bytes < in_b + out_b + ws_bytes) {
    if (sc.buf) cudaFree(sc.buf);
    sc.buf = nullptr;
    sc.bytes = 0;
    if (cudaMalloc(&sc.buf, in_b + out_b + ws_bytes) != cudaSuccess) {
      cudaGetLastError();
      return TCCD_E_CUDA;
    }
    sc.bytes = in_b + out_b + ws_bytes;
  }
  unsigned char* d = sc.buf;
  double* d_pts = (double*)d;
  double* d_eps = d_pts + 24;
  unsigned char* o = d + in_b;
  double* d_toi = (double*)o;
  double* d_tol = d_toi + 1;
  double* d_codom = d_toi + 2;
  double* d_wit = d_toi + 3;  // 6
  long long* d_checks = (long long*)(d_toi + 9);
  int* d_level = (int*)(d_toi + 10);
  uint8_t* d_status = (uint8_t*)(d_toi + 11);
  uint8_t* d_early = d_status + 1;
  // (a private non-blocking stream would need its own synchronization: the
  // legacy stream orders these copies with the solve)
  if (cudaMemcpy(d_pts, hpts, sizeof hpts, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(d_eps, heps, sizeof heps, cudaMemcpyHostToDevice) != cudaSuccess)
    return TCCD_E_CUDA;
  tccd_batch b;
  memset(&b, 0, sizeof b);
  b.struct_size = sizeof b;
  b.flags = 0;
  b.n = 1;
  b.points = d_pts;
  b.kind_all = kind;
  b.delta_all = delta;
  b.max_checks_all = max_checks;
  b.separation_all = sep;
  b.t_max_all = t_max;
  b.eps = d_eps;
  b.status = d_status;
  b.toi = d_toi;
  b.tol = d_tol;
  b.codom = d_codom;
  b.checks = (int64_t*)d_checks;
  b.early = d_early;
  b.witness = d_wit;
  b.level = d_level;
  b.workspace = o + out_b;
  b.workspace_bytes = ws_bytes;
  b.heavy_blocks = gb;
  int rc = tccd_solve_batch(&b, nullptr);
  unsigned char host[out_b];
  if (rc == TCCD_OK && cudaMemcpy(host, o, out_b, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = TCCD_E_CUDA;
  if (rc != TCCD_OK) return rc;
  const double* hd = (const double*)host;
  long long chk;
  int lvl;
  memcpy(&chk, hd + 9, 8);
  memcpy(&lvl, hd + 10, 4);
  const uint8_t hs = host[11 * 8], he = host[11 * 8 + 1];
  out13[0] = hs;
  out13[1] = hd[0];
  out13[2] = hd[1];
  out13[3] = hd[2];
  out13[4] = (double)chk;
  out13[5] = he;
  for (int k = 0; k < 6; ++k) out13[6 + k] = hd[3 + k];
  out13[12] = lvl;
  return TCCD_OK;
}

void tccd_release_cached(void) {
  std::lock_guard<std::mutex> lock(g_sk_mutex);
  int cur = current_device();
  for (int d = 0; d < 256; ++d) {
    if (!g_sk[d].buf) continue;
    cudaSetDevice(d);
    cudaFree(g_sk[d].buf);
    g_sk[d].buf = nullptr;
    g_sk[d].bytes = 0;
  }
  cudaSetDevice(cur);
}

}  // extern "C"
