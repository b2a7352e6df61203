// libtccd: batched Tight-Inclusion CCD on B200 (sm_100a), FP64, FMA-free.
//
// Two engines share the device numerics in tccd_device.cuh and reproduce the
// reference state machine (ccdkit._kernel.solve_kernel, pkg/src/ccdkit/
// _kernel.py:136-324) exactly, per query:
//
//  * pool engine (pool_kernel, tccd_pool.cuh): a persistent CTA keeps up to
//    kPQ queries resident and advances all of them one BFS level per
//    round.  Every thread classifies boxes of the flat list of all resident
//    levels (lane per box, queries mixed, so trivially separated queries do
//    not idle a warp); the in-level event sequence of each query (budget
//    cut, first/drop records, accept, children in push order, stable t_lo
//    order of the next level) is recovered with segmented block-wide mins,
//    scans and merge-by-rank; finished slots are refilled from a global
//    work counter (dynamic load balance across CTAs).
//  * heavy engine (heavy_kernel): one CTA per query with the level in a
//    global-memory arena sized for the worst case (2 * m_I boxes), used for
//    queries whose frontier outgrows the light pool.  The level is
//    classified in parallel; the sequential semantics are recovered with a
//    block-wide min (first non-disjoint box), a second min (first accepted
//    later box = the drop candidate), the budget cut index, block scans for
//    the children's push positions, and a merge-by-rank of the two sorted
//    child subsequences for the next level's stable order.
//
// Evicted queries restart from the root in the heavy engine (classification
// is a pure function of the box, so the replay is exact).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "tccd.h"
#include "tccd_device.cuh"

namespace tccd {

// ---------------------------------------------------------------------------
// launch geometry / pool sizes
constexpr int kHB = 256;    // heavy engine threads per CTA

struct Counters {
  unsigned long long light_next;   // next query index the pool admits
  unsigned long long heavy_count;  // entries in the heavy queue
  unsigned long long heavy_next;   // next heavy queue entry to solve
  unsigned long long rounds;       // pool rounds (diagnostics)
  unsigned long long deferred;     // pool level deferrals (diagnostics)
  unsigned long long pad[3];
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
  long long* heavy_queue;
  unsigned char* pool_arenas;
  size_t pool_arena_bytes;
  unsigned char* arenas;
  size_t arena_bytes;
  long long cap;  // boxes per heavy arena buffer
  int heavy_only;
};

__device__ __forceinline__ void write_result(const Args& a, long long q, uint8_t status,
                                             const Box& b, double codom, long long checks,
                                             int early, int level) {
  a.status[q] = status;
  const bool hit = status == kHit;
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

// Load a query's per-query parameters, validate them, and resolve filters
// and kappas.  P must already hold its 24 coordinates.  Returns kHit or an
// error status.
template <typename PtrT>
__device__ __forceinline__ uint8_t prologue(const Args& a, long long q, PtrT P, QueryParams& qp) {
  qp.kind = a.kind ? a.kind[q] : a.kind_all;
  qp.delta = a.delta ? a.delta[q] : a.delta_all;
  qp.max_checks = a.max_checks ? a.max_checks[q] : a.max_checks_all;
  qp.sep = a.sep ? a.sep[q] : a.sep_all;
  qp.t_max = a.t_max ? a.t_max[q] : a.t_max_all;
  if (!params_valid(qp.kind, qp.delta, qp.max_checks, qp.sep, qp.t_max) ||
      qp.max_checks > a.max_checks_max)
    return kErrParam;
  uint8_t st;
  if (a.eps) {
    st = kHit;
    for (int i = 0; i < 24; ++i)
      if (!isfinite(P[i])) st = kErrNonfinite;
    qp.eps[0] = a.eps[3 * q];
    qp.eps[1] = a.eps[3 * q + 1];
    qp.eps[2] = a.eps[3 * q + 2];
  } else {
    st = filters(P, qp.kind, qp.sep, qp.eps);
  }
  if (st != kHit) return st;
  kappas(P, qp.kind, qp.t_max, qp.kap);
  return kHit;
}

// ---------------------------------------------------------------------------
// block scan (NT threads)
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
// heavy engine: one CTA per query, level in a global arena
// ===========================================================================
struct Arena {
  Box* cur;   // level in sorted order; reused for the next level
  Box* ab;    // children: A subsequence from the front, B from the back
  unsigned long long* key;
  unsigned int* push;
  uint8_t* flag;
  double* wb;  // also reused as the B permutation in the fallback sort
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

__host__ __device__ inline size_t arena_bytes_for(long long cap) {
  return align256(cap * sizeof(Box)) * 2 + align256(cap * 8) + align256(cap * 4) +
         align256(cap) + align256(cap * 8);
}

__device__ inline Arena arena_at(unsigned char* base, long long cap) {
  Arena r;
  size_t o = 0;
  r.cur = (Box*)(base + o); o += align256(cap * sizeof(Box));
  r.ab = (Box*)(base + o); o += align256(cap * sizeof(Box));
  r.key = (unsigned long long*)(base + o); o += align256(cap * 8);
  r.push = (unsigned int*)(base + o); o += align256(cap * 4);
  r.flag = (uint8_t*)(base + o); o += align256(cap);
  r.wb = (double*)(base + o);
  return r;
}

// flag byte: bits 0-1 class, bit 2 accepted, bits 3-4 split dim, bit 5 upper child pushed
__device__ __forceinline__ uint8_t make_flag(int cls, bool acc, int sdim, bool push_hi) {
  return (uint8_t)(cls | (acc ? 4 : 0) | (sdim << 3) | (push_hi ? 32 : 0));
}

// (key, push) lexicographic "less than"
__device__ __forceinline__ bool kp_less(unsigned long long ka, unsigned int pa,
                                        unsigned long long kb, unsigned int pb) {
  return ka < kb || (ka == kb && pa < pb);
}

struct HeavyShared {
  double P[24];
  QueryParams qp;
  Box fbox, dbox;
  double fcodom, dcodom;
  int flevel, dlevel;
  int have_first, have_drop;
  long long C;        // checks before the current level
  long long n;        // boxes in the current level
  int level;
  long long j, acc;   // first non-disjoint, first accepted after j
  int done;
  int b_unsorted;
  unsigned long long runA, runB;
  unsigned long long sw[kHB / 32];
};

__device__ void heavy_finish(const Args& a, long long q, HeavyShared& S, bool early) {
  // report min(drop, first) by t_lo, drop only when strictly earlier
  // (_kernel.py:192-199, 208-213)
  if (S.have_drop && (!S.have_first || S.dbox.t0 < S.fbox.t0))
    write_result(a, q, kHit, S.dbox, S.dcodom, 0, early, S.dlevel);
  else
    write_result(a, q, kHit, S.fbox, S.fcodom, 0, early, S.flevel);
}

__device__ void heavy_solve(const Args& a, long long q, HeavyShared& S, const Arena& ar) {
  const int tid = threadIdx.x;
  if (tid < 24) S.P[tid] = a.points[24 * q + tid];
  __syncthreads();
  if (tid == 0) {
    const uint8_t st = prologue(a, q, (const double*)S.P, S.qp);
    S.done = st != kHit;
    if (S.done) {
      Box z = {0, 0, 0, 0, 0, 0};
      write_result(a, q, st, z, 0.0, 0, 0, 0);
    }
    S.C = 0; S.n = 1; S.level = 0;
    S.have_first = S.have_drop = 0;
    ar.cur[0] = Box{0.0, S.qp.t_max, 0.0, 1.0, 0.0, 1.0};
  }
  __syncthreads();
  if (S.done) return;
  const int kind = S.qp.kind;
  const long long mc = S.qp.max_checks;
  const long long cap = a.cap;

  for (;;) {
    const long long n = S.n, C = S.C;
    const long long cut = mc - C - 1;  // index where checks reaches m_I
    const long long ecls = n < cut + 1 ? n : cut + 1;
    if (tid == 0) { S.j = LLONG_MAX; S.acc = LLONG_MAX; }
    __syncthreads();
    // ---- classify the level's prefix that the budget lets run
    long long myj = LLONG_MAX;
    for (long long i = tid; i < ecls; i += kHB) {
      const Box b = ar.cur[i];
      double wb;
      const int cls = classify(S.P, kind, b, S.qp.eps, S.qp.sep, wb);
      uint8_t f = (uint8_t)cls;
      if (cls != kDisjoint) {
        int sdim; double mid; bool ph;
        const bool acc = split_decision(b, cls, wb, S.qp.kap, S.qp.delta, kind, sdim, mid, ph);
        f = make_flag(cls, acc, sdim, ph);
        if (i < myj) myj = i;
      }
      ar.flag[i] = f;
      ar.wb[i] = wb;
    }
    if (myj != LLONG_MAX) atomicMin((long long*)&S.j, myj);
    __syncthreads();
    const long long j = S.j;
    // ---- outcome at the first non-disjoint box / the budget cut
    if (j >= ecls) {
      if (tid == 0) {
        if (cut < n) {
          if (S.have_drop || cut + 1 < n) heavy_finish(a, q, S, true);
          else { Box z = {0, 0, 0, 0, 0, 0}; write_result(a, q, kFree, z, 0.0, 0, 0, 0); }
          if (a.checks) a.checks[q] = mc;
        } else {
          // every box disjoint: the queue empties (_kernel.py:321-324)
          if (S.have_drop) write_result(a, q, kHit, S.dbox, S.dcodom, 0, 0, S.dlevel);
          else { Box z = {0, 0, 0, 0, 0, 0}; write_result(a, q, kFree, z, 0.0, 0, 0, 0); }
          if (a.checks) a.checks[q] = C + n;
        }
      }
      return;
    }
    if (tid == 0) {
      S.have_first = 1;
      S.fbox = ar.cur[j];
      S.fcodom = ar.wb[j];
      S.flevel = S.level;
      S.done = 0;
      const uint8_t fj = ar.flag[j];
      if (j == cut) {
        heavy_finish(a, q, S, true);
        if (a.checks) a.checks[q] = mc;
        S.done = 1;
      } else if (fj & 4) {
        // first colliding box of a fresh level accepted (_kernel.py:243-252)
        if (S.have_drop && S.dbox.t0 < S.fbox.t0)
          write_result(a, q, kHit, S.dbox, S.dcodom, 0, 0, S.dlevel);
        else
          write_result(a, q, kHit, S.fbox, S.fcodom, 0, 0, S.level);
        if (a.checks) a.checks[q] = C + j + 1;
        S.done = 1;
      }
    }
    __syncthreads();
    if (S.done) return;
    // ---- boxes strictly between j and the cut: first accepted one is the drop candidate
    const long long eend = n < cut ? n : cut;
    long long mya = LLONG_MAX;
    for (long long i = j + 1 + tid; i < eend; i += kHB) {
      const uint8_t f = ar.flag[i];
      if ((f & 3) != kDisjoint && (f & 4)) { mya = i; break; }
    }
    if (mya != LLONG_MAX) atomicMin((long long*)&S.acc, mya);
    __syncthreads();
    if (tid == 0) {
      const long long ai = S.acc;
      if (ai < eend) {
        const Box b = ar.cur[ai];
        if (!S.have_drop || b.t0 < S.dbox.t0) {
          S.dbox = b;
          S.dcodom = ar.wb[ai];
          S.dlevel = S.level;
        }
        S.have_drop = 1;
      }
      if (cut < n) {
        // budget ends inside this level after children were pushed
        heavy_finish(a, q, S, true);
        if (a.checks) a.checks[q] = mc;
        S.done = 1;
      }
      S.runA = 0;
      S.runB = 0;
      S.b_unsorted = 0;
    }
    __syncthreads();
    if (S.done) return;
    // ---- children of every non-disjoint, non-accepted box in [j, n), push order
    for (long long base = j; base < n; base += kHB) {
      const long long i = base + tid;
      uint8_t f = 0;
      bool valid = false;
      if (i < n) {
        f = ar.flag[i];
        valid = (f & 3) != kDisjoint && !(f & 4);
      }
      const int sdim = (f >> 3) & 3;
      const bool ph = (f & 32) != 0;
      const unsigned long long cA = valid ? (1ull + ((sdim != 0 && ph) ? 1ull : 0ull)) : 0ull;
      const unsigned long long cB = (valid && sdim == 0) ? 1ull : 0ull;
      unsigned long long tot;
      const unsigned long long pre = block_excl_scan<kHB>((cA << 32) | cB, S.sw, tot);
      const unsigned long long posA = S.runA + (pre >> 32), posB = S.runB + (pre & 0xffffffffull);
      if (valid) {
        const Box b = ar.cur[i];
        const double lo = sdim == 0 ? b.t0 : (sdim == 1 ? b.u0 : b.v0);
        const double hi = sdim == 0 ? b.t1 : (sdim == 1 ? b.u1 : b.v1);
        const double mid = 0.5 * (lo + hi);
        Box c0, c1;
        children(b, sdim, mid, c0, c1);
        const unsigned int push = (unsigned int)(posA + posB);
        ar.ab[posA] = c0;
        ar.key[posA] = tkey(c0.t0);
        ar.push[posA] = push;
        if (sdim != 0) {
          if (ph) {
            ar.ab[posA + 1] = c1;
            ar.key[posA + 1] = tkey(c1.t0);
            ar.push[posA + 1] = push + 1;
          }
        } else {
          const long long kb = cap - 1 - (long long)posB;
          ar.ab[kb] = c1;
          ar.key[kb] = tkey(c1.t0);
          ar.push[kb] = push + 1;
        }
      }
      __syncthreads();
      if (tid == 0) { S.runA += tot >> 32; S.runB += tot & 0xffffffffull; }
      __syncthreads();
    }
    const long long nA = (long long)S.runA, nB = (long long)S.runB;
    // ---- B (upper children of t-splits) sorted by t_lo?  (always, for dyadic t_max)
    for (long long k = tid; k + 1 < nB; k += kHB)
      if (ar.key[cap - 1 - k] > ar.key[cap - 2 - k]) S.b_unsorted = 1;
    __syncthreads();
    unsigned int* perm = (unsigned int*)ar.wb;  // B order (identity unless unsorted)
    const bool use_perm = S.b_unsorted != 0;
    if (use_perm) {
      // general fallback: bitonic sort of B's positions by (t_lo, push)
      long long m = 1;
      while (m < nB) m <<= 1;
      for (long long k = tid; k < m; k += kHB) perm[k] = k < nB ? (unsigned int)k : 0xffffffffu;
      __syncthreads();
      for (long long size = 2; size <= m; size <<= 1) {
        for (long long stride = size >> 1; stride > 0; stride >>= 1) {
          for (long long t = tid; t < m / 2; t += kHB) {
            const long long lo = 2 * t - (t & (stride - 1));
            const long long hi = lo + stride;
            const bool up = (lo & size) == 0;
            const unsigned int pl = perm[lo], phh = perm[hi];
            bool gt;
            if (pl == 0xffffffffu) gt = phh != 0xffffffffu;
            else if (phh == 0xffffffffu) gt = false;
            else {
              const long long il = cap - 1 - pl, ih = cap - 1 - phh;
              gt = kp_less(ar.key[ih], ar.push[ih], ar.key[il], ar.push[il]);
            }
            if (gt == up) { perm[lo] = phh; perm[hi] = pl; }
          }
          __syncthreads();
        }
      }
    }
    // ---- merge by rank into the next level (sorted by (t_lo, push))
    for (long long k = tid; k < nA; k += kHB) {
      const unsigned long long kk = ar.key[k];
      const unsigned int pp = ar.push[k];
      long long lo = 0, hi = nB;  // count B elements < (kk, pp)
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        const long long ib = cap - 1 - (use_perm ? (long long)perm[mid] : mid);
        if (kp_less(ar.key[ib], ar.push[ib], kk, pp)) lo = mid + 1;
        else hi = mid;
      }
      ar.cur[k + lo] = ar.ab[k];
    }
    for (long long k = tid; k < nB; k += kHB) {
      const long long ib = cap - 1 - (use_perm ? (long long)perm[k] : k);
      const unsigned long long kk = ar.key[ib];
      const unsigned int pp = ar.push[ib];
      long long lo = 0, hi = nA;  // count A elements < (kk, pp)
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (kp_less(ar.key[mid], ar.push[mid], kk, pp)) lo = mid + 1;
        else hi = mid;
      }
      ar.cur[k + lo] = ar.ab[ib];
    }
    __syncthreads();
    if (tid == 0) {
      S.C = C + n;
      S.n = nA + nB;
      S.level += 1;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kHB) heavy_kernel(Args a) {
  __shared__ HeavyShared S;
  __shared__ long long s_item;
  const Arena ar = arena_at(a.arenas + (size_t)blockIdx.x * a.arena_bytes, a.cap);
  for (;;) {
    if (threadIdx.x == 0) s_item = (long long)atomicAdd(&a.ctr->heavy_next, 1ull);
    __syncthreads();
    const long long item = s_item;
    const long long total = a.heavy_only ? a.n : (long long)*(volatile unsigned long long*)&a.ctr->heavy_count;
    if (item >= total) break;
    const long long q = a.heavy_only ? item : a.heavy_queue[item];
    heavy_solve(a, q, S, ar);
    __syncthreads();
  }
}

}  // namespace tccd

#include "tccd_pool.cuh"

namespace tccd {

__global__ void stats_kernel(Args a) {
  if (threadIdx.x == 0 && a.stats) {
    a.stats[0] = a.heavy_only ? a.n : (long long)a.ctr->heavy_count;
    a.stats[1] = (long long)a.ctr->rounds;
    a.stats[2] = (long long)a.ctr->deferred;
    a.stats[3] = 0;
  }
}

}  // namespace tccd

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace tccd;

namespace {

int device_sm_count(int hint) {
  if (hint > 0) return hint;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return sms > 0 ? sms : 148;
}

long long heavy_cap(long long mcmax) { return 2 * mcmax + 2; }

int default_heavy_blocks(int sms) { return sms; }

int pool_blocks(int sms) { return 2 * sms; }

size_t layout(long long n, long long mcmax, int hb, int sms, size_t* off_queue,
              size_t* off_pool, size_t* off_arenas, size_t* arena_b) {
  const size_t ctr = align256(sizeof(Counters));
  const size_t q = align256((size_t)(n > 0 ? n : 1) * sizeof(long long));
  const size_t pool = pool_arena_bytes() * (size_t)pool_blocks(sms);
  const size_t ab = arena_bytes_for(heavy_cap(mcmax));
  if (off_queue) *off_queue = ctr;
  if (off_pool) *off_pool = ctr + q;
  if (off_arenas) *off_arenas = ctr + q + pool;
  if (arena_b) *arena_b = ab;
  return ctr + q + pool + ab * (size_t)hb;
}

bool pool_configured = false;

}  // namespace

extern "C" {

int tccd_abi_version(void) { return TCCD_ABI_VERSION; }

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

size_t tccd_workspace_bytes(int64_t n, int64_t max_checks_max, int32_t heavy_blocks) {
  if (n < 0 || max_checks_max < 1) return 0;
  const int sms = device_sm_count(0);
  const int hb = heavy_blocks > 0 ? heavy_blocks : default_heavy_blocks(sms);
  return layout(n, max_checks_max, hb, sms, nullptr, nullptr, nullptr, nullptr);
}

int tccd_solve_batch(const tccd_batch* b, void* stream) {
  if (!b) return TCCD_E_NULL;
  if (b->struct_size != sizeof(tccd_batch)) return TCCD_E_STRUCT;
  if (b->n < 0) return TCCD_E_N;
  if (b->n > 0 && (!b->points || !b->status || !b->toi)) return TCCD_E_NULL;
  if (!b->delta && !(b->delta_all > 0.0 && b->delta_all < 1.0 / 0.0)) return TCCD_E_DELTA;
  if (!b->max_checks && b->max_checks_all < 1) return TCCD_E_MAXCHECKS;
  if (!b->t_max && !(b->t_max_all > 0.0 && b->t_max_all <= 1.0)) return TCCD_E_TMAX;
  if (!b->separation && !(b->separation_all >= 0.0 && b->separation_all < 1.0 / 0.0))
    return TCCD_E_SEPARATION;
  if (!b->kind && b->kind_all != 0 && b->kind_all != 1) return TCCD_E_KIND;
  long long mcmax = b->max_checks ? b->max_checks_max : b->max_checks_all;
  if (b->max_checks && mcmax < 1) return TCCD_E_MAXCHECKS;
  if (mcmax > (1LL << 30)) return TCCD_E_CAPACITY;  // push indices are u32
  const int sms = device_sm_count(b->device_sms);
  const int hb = b->heavy_blocks > 0 ? b->heavy_blocks : default_heavy_blocks(sms);
  size_t off_q, off_pool, off_ar, arena_b;
  const size_t need = layout(b->n, mcmax, hb, sms, &off_q, &off_pool, &off_ar, &arena_b);
  if (!b->workspace || b->workspace_bytes < need) return TCCD_E_WORKSPACE;
  if (b->n == 0) return TCCD_OK;
  cudaStream_t st = (cudaStream_t)stream;
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
  a.ctr = (Counters*)ws;
  a.heavy_queue = (long long*)(ws + off_q);
  a.pool_arenas = ws + off_pool;
  a.pool_arena_bytes = pool_arena_bytes();
  a.arenas = ws + off_ar;
  a.arena_bytes = arena_b;
  a.cap = heavy_cap(mcmax);
  a.heavy_only = (b->flags & TCCD_FLAG_HEAVY_ONLY) ? 1 : 0;

  if (cudaMemsetAsync(ws, 0, sizeof(Counters), st) != cudaSuccess) return TCCD_E_CUDA;
  if (!a.heavy_only) {
    const int smem = (int)sizeof(PoolShared);
    if (!pool_configured) {
      if (cudaFuncSetAttribute(pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
          cudaSuccess)
        return TCCD_E_CUDA;
      pool_configured = true;
    }
    long long grid = pool_blocks(sms);
    const long long need_blocks = (b->n + kPQ - 1) / kPQ;
    if (grid > need_blocks) grid = need_blocks;
    pool_kernel<<<(unsigned)grid, kPT, smem, st>>>(a);
    if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  }
  long long hgrid = hb;
  if (a.heavy_only && hgrid > b->n) hgrid = b->n;
  heavy_kernel<<<(unsigned)hgrid, kHB, 0, st>>>(a);
  if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  if (a.stats) {
    stats_kernel<<<1, 32, 0, st>>>(a);
    if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  }
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
  const int hb = 1;
  const size_t ws_bytes = tccd_workspace_bytes(1, max_checks, hb);  // pool arenas unused (heavy-only)
  // one allocation: inputs | outputs | workspace
  const size_t in_b = 256, out_b = 256;
  unsigned char* d = nullptr;
  if (cudaMalloc(&d, in_b + out_b + ws_bytes) != cudaSuccess) return TCCD_E_CUDA;
  int rc = TCCD_OK;
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
  if (cudaMemcpy(d_pts, hpts, sizeof hpts, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(d_eps, heps, sizeof heps, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return TCCD_E_CUDA;
  }
  tccd_batch b;
  memset(&b, 0, sizeof b);
  b.struct_size = sizeof b;
  b.flags = TCCD_FLAG_HEAVY_ONLY;
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
  b.heavy_blocks = hb;
  rc = tccd_solve_batch(&b, nullptr);
  unsigned char host[out_b];
  if (rc == TCCD_OK && cudaMemcpy(host, o, out_b, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = TCCD_E_CUDA;
  cudaFree(d);
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

}  // extern "C"
