// Level engine: an independent group of threads (a CTA) keeps up to Q
// queries resident and advances all of them one BFS level per round.  One
// template, three tiers (see tccd.cu): light (128-thread CTAs, 5 per SM, 40
// queries, levels up to 1024 boxes) and medium (256-thread CTAs, 2 per SM,
// 8 queries, levels up to 8192 boxes), both with their per-box bookkeeping
// in shared memory, and giant (a 512-thread CTA per query for levels of up
// to 2 * m_I boxes, bookkeeping in global memory).  A query whose level
// outgrows its tier moves to the next tier with that level handed over (or,
// if the handover pool is full, restarts there: classification is a pure
// function of the box, so the replay is exact).
//
// Representation.  The current levels of all resident queries form one flat
// list of 4-byte references, one segment per query, each segment in the
// reference's visiting order (stable by t_lo, _kernel.py:174-175).  A
// reference names a box of the PREVIOUS round's materialized box array:
// "child cb of box src" (the child is the parent with one bound replaced by
// the midpoint of the parent's split dimension, which the parent's flag
// byte records), "box src itself" (a deferred level), a box of the tier's
// handover pool, or the query's root.  Children never travel through memory
// as boxes: the classify phase materializes each box once, in visiting
// order.
//
// A round:
//   P1 materialize + classify every box (lane per box, queries mixed);
//      group-wide atomicMin per query = first non-disjoint box j
//      and atomicMin = first accepted box (if not j itself, the only
//      candidate for the "drop" record, since boxes are in t_lo order)
//   P3 one thread per query replays the reference's in-level events from
//      (j, drop, cut) in O(1): normal return, budget return, queue
//      exhaustion or continue (_kernel.py:176-324)
//   P4 group scan of child counts over the flat list; children split into
//      two flat subsequences, A (t_lo = parent t_lo: lower children and u/v
//      upper children) and B (t-split upper children), each sorted by
//      (t_lo, push order)
//   P5 next-level layout (slot order); eviction of queries whose level
//      outgrew the tier; deferral of queries that do not fit this round
//      (their level re-runs: record updates are idempotent, the check count
//      is rolled back)
//   P6 every child computes its rank in its query's next level by binary
//      search of the other subsequence (merge by rank); a query whose B run
//      is not sorted (non-dyadic t_max) uses an exact O(n) rank count
//   P7 commit; admission refills free slots from the tier's input queue.
#pragma once

namespace tccd {

constexpr int kIntMax = 0x7fffffff;

constexpr uint8_t kClassified = 64;  // flag bit: box already classified
constexpr uint8_t kHead = 128;       // flag bit: first box of a run of equal t_lo
// P4c modes of a slot: children kept here (closed form), level carried
// (deferred), children handed over to the next tier's pool (closed form)
constexpr uint8_t kPcKeep = 1, kPcCarry = 2, kPcHand = 3;

// reference encoding
constexpr unsigned kRefSrcMask = (1u << 29) - 1;  // position in the previous box array
constexpr unsigned kRefCb = 1u << 29;             // upper child
constexpr unsigned kRefSelf = 1u << 30;           // the box itself (deferred level)
constexpr unsigned kRefRoot = 1u << 31;           // the query's root box
constexpr unsigned kRefExt = kRefRoot | kRefSelf;  // box src of the handover pool


template <int G_, int NT_, int Q_, int CAP_, int QCAP_, int ADMIT_, bool SMEM_, int MINB_>
struct EngineCfg {
  static constexpr int G = G_;          // threads per independent group (32 = warp)
  static constexpr int NT = NT_;        // threads per CTA (NT / G groups)
  static constexpr int Q = Q_;          // query slots per group
  static constexpr int CAP = CAP_;      // boxes per level list (0: runtime)
  static constexpr int QCAP = QCAP_;    // largest per-query level (0: = cap)
  static constexpr int ADMIT = ADMIT_;  // admit below this fill (0: = cap)
  static constexpr bool SMEM = SMEM_;   // per-box bookkeeping in shared memory
  static constexpr int MINB = MINB_;    // CTAs per SM (launch bounds)
};

template <int G>
__device__ __forceinline__ void gsync() {
  if constexpr (G == 32) __syncwarp();
  else __syncthreads();
}

// exclusive scan over a group (warp: shuffles; CTA: block scan)
template <int G>
__device__ __forceinline__ unsigned long long group_excl_scan(unsigned long long v,
                                                              unsigned long long* sw,
                                                              unsigned long long& total) {
  if constexpr (G == 32) {
    const int lane = threadIdx.x & 31;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
  } else {
    return block_excl_scan<G>(v, sw, total);
  }
}

// two exclusive sums over a group in one pass (shared barriers)
template <int G>
__device__ __forceinline__ void group_excl_scan2(unsigned long long v0, unsigned long long v1,
                                                 unsigned long long* sw, unsigned long long& e0,
                                                 unsigned long long& e1, unsigned long long& t0,
                                                 unsigned long long& t1) {
  const int lane = threadIdx.x & 31;
  unsigned long long x0 = v0, x1 = v1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y0 = __shfl_up_sync(0xffffffffu, x0, o);
    const unsigned long long y1 = __shfl_up_sync(0xffffffffu, x1, o);
    if (lane >= o) { x0 += y0; x1 += y1; }
  }
  if constexpr (G == 32) {
    t0 = __shfl_sync(0xffffffffu, x0, 31);
    t1 = __shfl_sync(0xffffffffu, x1, 31);
    e0 = x0 - v0;
    e1 = x1 - v1;
  } else {
    constexpr int NW = G / 32;
    const int w = (threadIdx.x % G) >> 5;
    if (lane == 31) { sw[w] = x0; sw[NW + w] = x1; }
    __syncthreads();
    if (w == 0) {
      unsigned long long a0 = lane < NW ? sw[lane] : 0ull, a1 = lane < NW ? sw[NW + lane] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y0 = __shfl_up_sync(0xffffffffu, a0, o);
        const unsigned long long y1 = __shfl_up_sync(0xffffffffu, a1, o);
        if (lane >= o) { a0 += y0; a1 += y1; }
      }
      if (lane < NW) { sw[lane] = a0; sw[NW + lane] = a1; }
    }
    __syncthreads();
    e0 = (w ? sw[w - 1] : 0ull) + x0 - v0;
    e1 = (w ? sw[NW + w - 1] : 0ull) + x1 - v1;
    t0 = sw[NW - 1];
    t1 = sw[2 * NW - 1];
    // (no trailing barrier: the caller's next write to sw is behind one)
  }
}

// exclusive scans of ints over a group in one pass: forward max of vm, and
// reverse min of vn (over the ranks above this one)
template <int G>
__device__ __forceinline__ void group_scan_maxfwd_minrev(int vm, int vn, int* swi, int& em,
                                                         int& en) {
  const int lane = threadIdx.x & 31;
  int xm = vm, xn = vn;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ym = __shfl_up_sync(0xffffffffu, xm, o);
    const int yn = __shfl_down_sync(0xffffffffu, xn, o);
    if (lane >= o) xm = max(xm, ym);
    if (lane + o < 32) xn = min(xn, yn);
  }
  int exm = __shfl_up_sync(0xffffffffu, xm, 1);
  int exn = __shfl_down_sync(0xffffffffu, xn, 1);
  if (lane == 0) exm = -1;
  if (lane == 31) exn = kIntMax;
  if constexpr (G == 32) {
    em = exm;
    en = exn;
  } else {
    constexpr int NW = G / 32;
    const int w = (threadIdx.x % G) >> 5;
    if (lane == 31) swi[w] = xm;
    if (lane == 0) swi[NW + w] = xn;
    __syncthreads();
    if (w == 0) {
      int am = lane < NW ? swi[lane] : -1, an = lane < NW ? swi[NW + lane] : kIntMax;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ym = __shfl_up_sync(0xffffffffu, am, o);
        const int yn = __shfl_down_sync(0xffffffffu, an, o);
        if (lane >= o) am = max(am, ym);
        if (lane + o < NW) an = min(an, yn);
      }
      int pm = __shfl_up_sync(0xffffffffu, am, 1);
      int pn = __shfl_down_sync(0xffffffffu, an, 1);
      if (lane == 0) pm = -1;
      if (lane == NW - 1) pn = kIntMax;
      if (lane < NW) { swi[2 * NW + lane] = pm; swi[3 * NW + lane] = pn; }
    }
    __syncthreads();
    em = max(swi[2 * NW + w], exm);
    en = min(swi[3 * NW + w], exn);
    // (no trailing barrier: the caller's next write to swi is behind one)
  }
}

// exclusive scans of ints over a group: forward max, and reverse min (over
// the ranks above this one)
template <int G, bool REV, bool MAX>
__device__ __forceinline__ int group_scan_excl_int(int v, int ident, int* swi) {
  const int lane = threadIdx.x & 31;
  auto op = [](int a, int b) { return MAX ? (a > b ? a : b) : (a < b ? a : b); };
  int x = v;  // inclusive in scan direction
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = REV ? __shfl_down_sync(0xffffffffu, x, o) : __shfl_up_sync(0xffffffffu, x, o);
    if (REV ? lane + o < 32 : lane >= o) x = op(x, y);
  }
  int ex = REV ? __shfl_down_sync(0xffffffffu, x, 1) : __shfl_up_sync(0xffffffffu, x, 1);
  if (REV ? lane == 31 : lane == 0) ex = ident;
  if constexpr (G == 32) {
    return ex;
  } else {
    constexpr int NW = G / 32;
    const int w = (threadIdx.x % G) >> 5;
    if (REV ? lane == 0 : lane == 31) swi[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = lane < NW ? swi[lane] : ident;
      int ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = REV ? __shfl_down_sync(0xffffffffu, ti, o) : __shfl_up_sync(0xffffffffu, ti, o);
        if (REV ? lane + o < NW : lane >= o) ti = op(ti, y);
      }
      int te = REV ? __shfl_down_sync(0xffffffffu, ti, 1) : __shfl_up_sync(0xffffffffu, ti, 1);
      if (REV ? lane == NW - 1 : lane == 0) te = ident;
      if (lane < NW) swi[NW + lane] = te;  // exclusive prefix over warps
    }
    __syncthreads();
    const int r = op(swi[NW + w], ex);
    __syncthreads();
    return r;
  }
}

// Per-chunk bookkeeping of a level list: one entry per 32 consecutive boxes
// (one warp's boxes in P1).  Masks (bit = box of the chunk): refining (non-
// disjoint, not accepted), second A child (u/v split with an upper child),
// B child (t split), run head.  Bases: exclusive prefixes over the list of
// A children, B children and refining boxes at the chunk start; M = refining
// count before the last run head before the chunk, N = refining count
// before the first run head after the chunk (the list total if none).
// Any box's prefixes are then O(1): base + popc(mask & lanes below).
struct Chunks {
  unsigned int* m[4];  // R, U, T, H
  int* c[5];           // A, B, P, M, N
};
constexpr int kMR = 0, kMU = 1, kMT = 2, kMH = 3;
constexpr int kCA = 0, kCB = 1, kCP = 2, kCM = 3, kCN = 4;

__device__ __forceinline__ unsigned int lowmask(int k) { return (1u << k) - 1u; }  // k < 32

// a[k] of a two-entry pointer array as a select: dynamic indexing would put
// the array in local memory and turn shared-memory accesses through the
// pointer into generic ones
template <class T>
__device__ __forceinline__ T* pick(T* const (&a)[2], int k) { return k ? a[1] : a[0]; }

// global arena of one group
template <class Cfg>
struct EngineArena {
  Box* box[2];
  double* wb[2];
  unsigned int* ref[2];
  unsigned long long* akey;  // [2 cap]
  unsigned int* apush;
  unsigned int* aref;
  unsigned long long* bkey;  // [cap]
  unsigned int* bpush;
  unsigned int* bref;
  // per-box / per-chunk bookkeeping when it lives in global memory
  uint8_t* slot_of[2];
  uint8_t* flag[2];
  Chunks ch;

  __host__ __device__ static long long chunks(long long cap) { return cap / 32 + 1; }

  __host__ __device__ static size_t bytes(long long cap) {
    size_t b = 2 * align256(cap * sizeof(Box)) + 2 * align256(cap * 8) + 2 * align256(cap * 4) +
               align256(2 * cap * 8) + 2 * align256(2 * cap * 4) + align256(cap * 8) +
               2 * align256(cap * 4);
    if (!Cfg::SMEM) b += 4 * align256(cap) + 9 * align256(chunks(cap) * 4);
    return b;
  }

  __device__ void init(unsigned char* base, long long cap) {
    size_t o = 0;
    for (int k = 0; k < 2; ++k) { box[k] = (Box*)(base + o); o += align256(cap * sizeof(Box)); }
    for (int k = 0; k < 2; ++k) { wb[k] = (double*)(base + o); o += align256(cap * 8); }
    for (int k = 0; k < 2; ++k) { ref[k] = (unsigned int*)(base + o); o += align256(cap * 4); }
    akey = (unsigned long long*)(base + o); o += align256(2 * cap * 8);
    apush = (unsigned int*)(base + o); o += align256(2 * cap * 4);
    aref = (unsigned int*)(base + o); o += align256(2 * cap * 4);
    bkey = (unsigned long long*)(base + o); o += align256(cap * 8);
    bpush = (unsigned int*)(base + o); o += align256(cap * 4);
    bref = (unsigned int*)(base + o); o += align256(cap * 4);
    if (!Cfg::SMEM) {
      for (int k = 0; k < 2; ++k) { slot_of[k] = base + o; o += align256(cap); }
      for (int k = 0; k < 2; ++k) { flag[k] = base + o; o += align256(cap); }
      for (int k = 0; k < 4; ++k) { ch.m[k] = (unsigned int*)(base + o); o += align256(chunks(cap) * 4); }
      for (int k = 0; k < 5; ++k) { ch.c[k] = (int*)(base + o); o += align256(chunks(cap) * 4); }
    }
  }
};

template <class Cfg>
struct EngineShared {
  static constexpr int Q = Cfg::Q;
  double P[Q][24];
  QueryParams qp[Q];
  Rec rec[Q][2];         // [0] first, [1] drop
  long long C[Q];        // checks before the current level
  long long C0[Q];       // checks when the query entered this tier
  long long qidx[Q];     // -1: free slot
  double root_wb[Q];
  int level[Q];
  int seg_off[Q], seg_n[Q];
  int j[Q], acc[Q];       // P1: flat position of the first non-disjoint / accepted box
  int cutpos[Q];         // flat position of the segment's last box within the budget
  int segA0[Q], segB0[Q], segA1[Q], segB1[Q];
  int next_off[Q];
  int tot[Q];
  long long hoff[Q];     // evicted with handover: pool offset of the level (-1: restart)
  int adm_n[Q], adm_pos[Q], adm_slot[Q];
  long long adm_off[Q];
  uint8_t root_flag[Q];
  uint8_t have_first[Q], have_drop[Q];
  uint8_t cont[Q];       // 1: children kept; 2: deferred; 3: evicted (children counted)
  uint8_t unsorted[Q];
  uint8_t uniform[Q];    // dyadic t_max: every level has uniform widths (closed-form order)
  int segP0[Q], segP1[Q];  // flat count of refining boxes before / after the segment
  unsigned long long sw[2 * (Cfg::G / 32)];
  int swi[4 * (Cfg::G / 32)];
  int any_general;
  int4 pc[Q];            // P4c view of a slot: next offset, segment P0 (carry: offset), P1, A0
  uint8_t pc_mode[Q];    // P4c: 0 skip, kPcKeep, kPcCarry, kPcHand (set where decided)
  // dyadic t_max: every box of a query's level has the same widths, so in a
  // round whose resident queries are all dyadic a materialized box is stored
  // as its lower corner (t0, u0, v0) only
  double w[Q][3];        // widths of the current level's boxes
  double wp[Q][3];       // widths of the previous level's (the parents')
  int lvl_sdim[Q];       // split dimension of the current level's refining boxes
  int allu;              // every resident query dyadic (this round's arrays compact)
  int n_cur, n_next, admit_k, exhausted, A_tot, B_tot, P_tot, rot;
  unsigned long long deferred;
  int deferred_last;     // queries deferred in the previous round
  long long admit_base;
  unsigned int free_mask[(Q + 31) / 32];
};

template <class Cfg>
struct EngineSmemBoxes {
  static constexpr int CAP = Cfg::SMEM ? Cfg::CAP : 32;
  static_assert(CAP % 32 == 0, "level lists are whole chunks");
  static constexpr int CH = CAP / 32;
  unsigned int m[4][CH];
  int c[5][CH];
  uint8_t slot_of[2][CAP];
  uint8_t flag[2][CAP];
};

// shared memory of ONE group (16-byte aligned); a CTA holds NT / G groups
template <class Cfg>
__host__ __device__ constexpr size_t engine_smem_bytes() {
  return (sizeof(EngineShared<Cfg>) + (Cfg::SMEM ? sizeof(EngineSmemBoxes<Cfg>) : 0) + 15) & ~size_t(15);
}

// split dimension and midpoint of a box that is refined (_kernel.py:219-241)
__device__ __forceinline__ int split_dim(const Box& b, const double* kap, double& mid) {
  const double ct = (b.t1 - b.t0) * kap[0];
  const double cu = (b.u1 - b.u0) * kap[1];
  const double cv = (b.v1 - b.v0) * kap[2];
  int sdim = 0;
  double best = ct;
  if (cu > best) { sdim = 1; best = cu; }
  if (cv > best) { sdim = 2; }
  const double lo = sdim == 0 ? b.t0 : (sdim == 1 ? b.u0 : b.v0);
  const double hi = sdim == 0 ? b.t1 : (sdim == 1 ? b.u1 : b.v1);
  mid = 0.5 * (lo + hi);
  return sdim;
}

#ifdef TCCD_PHASE_PROF
// per-phase cycle accounting (diagnostic builds only)
#define TCCD_PHASE(k)                                     \
  do {                                                    \
    if (tid == 0) {                                       \
      const long long now_ = clock64();                   \
      ph_acc[k] += (unsigned long long)(now_ - ph_last);  \
      ph_last = now_;                                     \
    }                                                     \
  } while (0)
#else
#define TCCD_PHASE(k) \
  do {                \
  } while (0)
#endif

struct TierIO {
  const Pre* in;            // input queue
  const Hand* in_hand;      // handover state of the input entries (nullptr: none)
  const Box* in_pbox;       // handover pool the input levels live in
  const uint8_t* in_pflag;
  int in_maxsz;             // largest handed-over level
  const unsigned int* in_perm;  // admission order of the input queue (nullptr: queue order)
  long long perm_max;       // in_perm holds an order only for queues up to this size
  Hand* out_hand;           // handover state / pool of the next tier
  Box* out_pbox;
  uint8_t* out_pflag;
  unsigned long long* out_pool_count;
  long long pool_cap;
  unsigned long long* in_count;
  unsigned long long* in_next;
  long long in_base;        // this launch's slice of the input queue
  long long in_limit;
  int hand_in_record;       // in_hand indexed by Pre::pad (else by entry)
  long long in_pool_cap;    // boxes in the input handover pool
  Pre* out;                 // eviction queue of the next tier (nullptr: none)
  unsigned long long* out_count;
  unsigned char* arenas;
  size_t arena_bytes;
  long long cap;            // boxes per level list
  unsigned long long* rounds;
  unsigned long long* deferred;
  unsigned long long* evicted;
  unsigned long long* boxes;
  unsigned long long* phase;  // [16] cycles per phase (TCCD_PHASE_PROF builds)
  unsigned long long* cls;    // [2] box classifications (VF, EE)
  unsigned long long* restarts;  // evictions that found the handover pool full
  unsigned long long* algo;      // checks of the reference's path done here
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT, Cfg::MINB) engine_kernel(Args a, TierIO io) {
  // Each group of G threads runs an independent engine instance with its own
  // shared-memory state and global arena; groups never synchronize with one
  // another (G = 32: warp-synchronous, no block barriers).
  constexpr int G = Cfg::G, Q = Cfg::Q;
  constexpr int NT = G;  // stride of the per-group loops
  // one query per group (giant tier): every box belongs to slot 0, so the
  // per-box slot bytes are never read
  constexpr bool ONEQ = Q == 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int group = threadIdx.x / G;
  unsigned char* gsmem = smem_raw + (size_t)group * engine_smem_bytes<Cfg>();
  EngineShared<Cfg>& S = *reinterpret_cast<EngineShared<Cfg>*>(gsmem);
  EngineArena<Cfg> ar;
  ar.init(io.arenas + ((size_t)blockIdx.x * (Cfg::NT / G) + group) * io.arena_bytes, io.cap);
  uint8_t* slot_of[2];
  uint8_t* flags[2];
  Chunks ch;
  if (Cfg::SMEM) {
    auto* SB = reinterpret_cast<EngineSmemBoxes<Cfg>*>(gsmem + sizeof(EngineShared<Cfg>));
    slot_of[0] = SB->slot_of[0]; slot_of[1] = SB->slot_of[1];
    flags[0] = SB->flag[0]; flags[1] = SB->flag[1];
    for (int k = 0; k < 4; ++k) ch.m[k] = SB->m[k];
    for (int k = 0; k < 5; ++k) ch.c[k] = SB->c[k];
  } else {
    slot_of[0] = ar.slot_of[0]; slot_of[1] = ar.slot_of[1];
    flags[0] = ar.flag[0]; flags[1] = ar.flag[1];
    ch = ar.ch;
  }
  const int lane = threadIdx.x & 31;
  const int cap = Cfg::CAP ? Cfg::CAP : (int)io.cap;
  const int qcap = Cfg::QCAP ? Cfg::QCAP : cap;
  const int admit_lim = Cfg::ADMIT ? Cfg::ADMIT : cap;
  // this launch's slice of the input queue: entries [in_base, in_base + in_limit)
  const unsigned long long in_all = *(volatile unsigned long long*)io.in_count;
  const unsigned long long in_total =
      in_all <= (unsigned long long)io.in_base ? 0ull
      : (in_all - io.in_base < (unsigned long long)io.in_limit ? in_all - io.in_base
                                                               : (unsigned long long)io.in_limit);
  const Pre* const inq = io.in + io.in_base;
  // queue entry admitted at position k
  const bool use_perm = io.in_perm && in_total >= 2 && (long long)in_total <= io.perm_max;
  auto entry = [&](long long k) -> long long { return use_perm ? (long long)io.in_perm[k] : k; };
  const int tid = threadIdx.x % G;  // rank within the group
  for (int s = tid; s < Q; s += NT) S.qidx[s] = -1;
  if (tid == 0) { S.n_cur = 0; S.exhausted = 0; S.rot = 0; S.deferred = 0; S.deferred_last = 0; }
  gsync<G>();
  int cur = 0;
  bool cprv = false;  // the previous round's level arrays are compact
  long long rounds = 0;
  unsigned long long evicted = 0, boxes = 0;
  long long algo = 0;  // this thread's share of the tier's algorithmic checks
  unsigned int ncls_vf = 0, ncls_ee = 0;  // this thread's classifications per kind
#ifdef TCCD_PHASE_PROF
  unsigned long long ph_acc[16] = {0};
  long long ph_last = clock64();
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif

  // Evict slot s (its next level has t boxes) to the next tier.  With room in
  // the handover pool, the next level is materialized there (P4c / P6) and
  // the next tier resumes the query; otherwise it restarts from the root.
  auto evict = [&](int s, int t) {
    const unsigned long long h = atomicAdd(io.out_count, 1ull);
    io.out[h] = Pre{S.qidx[s], 0.0, 0u, 0xffffffffu};
    long long off = -1;
    if (io.out_hand) {
      const unsigned long long o = atomicAdd(io.out_pool_count, (unsigned long long)t);
      if ((long long)o + t <= io.pool_cap) off = (long long)o;
      if (off < 0) {
        // restart from the root: this tier's checks of the query are redone
        atomicAdd(io.restarts, 1ull);
        algo -= S.C[s] - S.C0[s];
      }
      Hand& hd = io.out_hand[h];
      hd.n = off >= 0 ? t : 0;
      hd.off = off;
      hd.C = S.C[s];
      hd.level = S.level[s] + 1;
      hd.rec[0] = S.rec[s][0];
      hd.rec[1] = S.rec[s][1];
      hd.have_first = S.have_first[s];
      hd.have_drop = S.have_drop[s];
    }
    S.hoff[s] = off;
    if (off >= 0 && S.uniform[s]) S.pc_mode[s] = kPcHand;
    S.qidx[s] = -1;
    S.cont[s] = 3;
    ++evicted;
  };
  auto finish = [&](int s, bool early, long long checks) {
    // report min(drop, first) (_kernel.py:192-199, 208-213)
    const bool use_drop =
        S.have_drop[s] && (!S.have_first[s] || S.rec[s][1].b.t0 < S.rec[s][0].b.t0);
    const Rec& r = S.rec[s][use_drop ? 1 : 0];
    write_result(a, S.qidx[s], kHit, r.b, r.codom, checks, early, r.level);
  };
  auto free_result = [&](int s, long long checks) {
    const Box z = {0, 0, 0, 0, 0, 0};
    write_result(a, S.qidx[s], kFree, z, 0.0, checks, 0, 0);
  };

  for (;;) {
    const int prv = cur ^ 1;
    // ================= P0: admission
    if (tid < 32) {
      unsigned int cnt = 0;
      for (int w = 0; w < (Q + 31) / 32; ++w) {
        const int s = w * 32 + tid;
        const unsigned int m = __ballot_sync(0xffffffffu, s < Q && S.qidx[s] < 0);
        if (tid == 0) S.free_mask[w] = m;
        cnt += __popc(m);
      }
      if (tid == 0) {
        S.allu = 1;
        int k = (int)cnt;
        int room = admit_lim - S.n_cur;
        if (room < 0) room = 0;
        if (k > room) k = room;
        // fair share of what is left, so a short queue spreads over all groups
        const unsigned long long taken = *(volatile unsigned long long*)io.in_next;
        const unsigned long long left = taken < in_total ? in_total - taken : 0ull;
        const unsigned long long groups = (unsigned long long)gridDim.x * (Cfg::NT / G);
        const long long share = (long long)((left + groups - 1) / groups);
        if (k > share) k = (int)(share > 0 ? share : 1);
        if (io.in_maxsz > 1) {  // handed-over levels: keep room for the largest
          int kk = room / io.in_maxsz;
          if (kk < 1 && S.n_cur == 0) kk = 1;
          if (k > kk) k = kk;
        }
        long long base = 0;
        if (S.exhausted) k = 0;
        if (S.deferred_last) k = 0;  // deferred queries get the room first (no starvation)
        if (k > 0) {
          base = (long long)atomicAdd(io.in_next, (unsigned long long)k);
          if ((unsigned long long)base >= in_total) { k = 0; S.exhausted = 1; }
          else if ((unsigned long long)(base + k) >= in_total) {
            k = (int)(in_total - base);
            S.exhausted = 1;
          }
        }
        S.admit_k = k;
        S.admit_base = base;
      }
    }
    gsync<G>();
    TCCD_PHASE(0);
    const int k_adm = S.admit_k;  // (group-uniform: branch and barriers below are safe)
    if (k_adm > 0) {
    // step 1a: free slot of each admitted entry
    for (int s = tid; s < Q; s += NT) {
      if (S.qidx[s] < 0 && k_adm > 0) {
        const int w = s >> 5, lane = s & 31;
        int r = __popc(S.free_mask[w] & ((1u << lane) - 1u));
        for (int ww = 0; ww < w; ++ww) r += __popc(S.free_mask[ww]);
        if (r < k_adm) S.adm_slot[r] = s;
      }
    }
    gsync<G>();
    // step 1b: the queue records (query index, root class) and, warp-
    // cooperatively, the query's 24 coordinates from the batch (192 bytes,
    // coalesced)
    {
      constexpr int NWARP = (NT + 31) / 32;
      const int wid = tid >> 5, lane = tid & 31;
      for (int r = wid; r < k_adm; r += NWARP) {
        const int s = S.adm_slot[r];
        const Pre& e = inq[entry(S.admit_base + r)];
        const long long q = e.q;
        if (lane < 24) S.P[s][lane] = a.points[24 * q + lane];
        if (lane == 0) {
          S.qidx[s] = q;
          S.root_wb[s] = e.wb;
          S.root_flag[s] = (uint8_t)(e.flag & 0xffu);
        }
      }
    }
    gsync<G>();
    // step 1b': per-query constants, recomputed from the coordinates exactly
    // as the prologue did (parameters, filters, kappas): a queue record is an
    // index, not a copy
    for (int r = tid; r < k_adm; r += NT) {
      const int s = S.adm_slot[r];
      const long long q = S.qidx[s];
      QueryParams qp;
      load_params(a, q, qp);
      const double* P = S.P[s];
      if (a.eps) {
        qp.eps[0] = a.eps[3 * q]; qp.eps[1] = a.eps[3 * q + 1]; qp.eps[2] = a.eps[3 * q + 2];
      } else {
        filters(P, qp.kind, qp.sep, qp.eps);  // (valid: the prologue checked it)
      }
      qp.tame = tame_coords(P);
      kappas(P, qp.kind, qp.t_max, qp.kap);
      S.qp[s] = qp;
    }
    gsync<G>();
    // step 1c: per-slot state (fresh root, or a level handed over by the
    // previous tier)
    for (int r = tid; r < k_adm; r += NT) {
      const int s = S.adm_slot[r];
      int ex;
      S.uniform[s] = frexp(S.qp[s].t_max, &ex) == 0.5;  // t_max a power of two
      int nr = 1;
      long long off = -1;
      // (root widths; a handed-over level's below)
      S.w[s][0] = S.qp[s].t_max; S.w[s][1] = 1.0; S.w[s][2] = 1.0;
      // handover state: the entry's own slot (medium / giant queues), or the
      // index the lane tier stored in the record (light queue)
      long long hi = -1;
      if (io.in_hand) {
        if (io.hand_in_record) {
          const unsigned int x = inq[entry(S.admit_base + r)].pad;
          if (x != 0xffffffffu) hi = x;
        } else {
          hi = entry(S.admit_base + r);
        }
      }
      if (hi >= 0 && io.in_hand[hi].n > 0) {
        const Hand& hd = io.in_hand[hi];
        nr = hd.n;
        off = hd.off;
        {
          const Box pb = io.in_pbox[off];
          S.w[s][0] = pb.t1 - pb.t0; S.w[s][1] = pb.u1 - pb.u0; S.w[s][2] = pb.v1 - pb.v0;
        }
        S.C[s] = hd.C;
        S.C0[s] = hd.C;
        S.level[s] = hd.level;
        S.rec[s][0] = hd.rec[0];
        S.rec[s][1] = hd.rec[1];
        S.have_first[s] = hd.have_first;
        S.have_drop[s] = hd.have_drop;
      } else {
        S.C[s] = 0;
        S.C0[s] = 0;
        S.level[s] = 0;
        S.have_first[s] = 0;
        S.have_drop[s] = 0;
      }
      S.adm_n[r] = nr;
      S.adm_off[r] = off;
    }
    gsync<G>();
    // step 2: segment offsets of the admitted levels
    if (tid == 0) {
      int pos = S.n_cur;
      for (int r = 0; r < k_adm; ++r) {
        S.adm_pos[r] = pos;
        pos += S.adm_n[r];
      }
      S.n_next = pos;  // new fill (reused as scratch until P5)
      S.n_cur = pos;
    }
    gsync<G>();
    // step 3: reference lists of the admitted levels
    for (int r = 0; r < k_adm; ++r) {
      const int s = S.adm_slot[r], pos = S.adm_pos[r], nr = S.adm_n[r];
      const long long off = S.adm_off[r];
      if (tid == 0) { S.seg_off[s] = pos; S.seg_n[s] = nr; }
      if (off < 0) {
        if (tid == 0) {
          TCCD_ASSERT(pos < cap);
          pick(ar.ref, cur)[pos] = kRefRoot;
          pick(slot_of, cur)[pos] = (uint8_t)s;
          pick(flags, cur)[pos] = S.root_flag[s] | kHead;
        }
      } else {
        for (int b = tid; b < nr; b += NT) {
          TCCD_ASSERT(pos + b < cap && off + b < io.in_pool_cap);
          pick(ar.ref, cur)[pos + b] = kRefExt | (unsigned)(off + b);
          pick(slot_of, cur)[pos + b] = (uint8_t)s;
          pick(flags, cur)[pos + b] = io.in_pflag[off + b];
        }
      }
    }
    gsync<G>();  // (seg_off, written by thread 0 above, sets every slot's budget cut below)
    }  // k_adm > 0
    for (int s = tid; s < Q; s += NT) {
      S.hoff[s] = -1;
      S.j[s] = kIntMax;
      S.acc[s] = kIntMax;
      S.cont[s] = 0;
      S.unsorted[s] = 0;
      S.pc_mode[s] = 0;
      if (S.qidx[s] >= 0) {
        if (!S.uniform[s]) S.allu = 0;
        const long long cp = S.seg_off[s] + (S.qp[s].max_checks - S.C[s] - 1);
        S.cutpos[s] = (int)max(min(cp, (long long)kIntMax - 1), -1ll);
      }
    }
    gsync<G>();
    TCCD_PHASE(1);
    TCCD_PHASE(2);
    const int n = S.n_cur;
    TCCD_ASSERT(n <= cap);
    if (n == 0) break;
    ++rounds;
    Box* const bx = pick(ar.box, cur);
    const Box* const bprev = pick(ar.box, prv);
    double* const wbc = pick(ar.wb, cur);
    const double* const wbp = pick(ar.wb, prv);
    const unsigned int* const rf = pick(ar.ref, cur);
    uint8_t* const sl = pick(slot_of, cur);
    uint8_t* const fl = pick(flags, cur);
    // ================= P1: materialize + classify
    // software pipeline: the reference of box i + 2*NT and the parent box of
    // box i + NT are in flight while box i is classified
    // (handed-over boxes are read from the tier's handover pool)
    const Box* const pool = io.in_pbox;
    // one query: boxes past its budget cut are never classified, and the query
    // ends this round (P3), so the round stops at the cut
    const int n1 = ONEQ ? (int)min((long long)n, S.seg_off[0] + max(S.qp[0].max_checks - S.C[0], 0ll))
                        : n;
    boxes += (unsigned long long)n1;
    // compact boxes (every resident query dyadic): this round's level arrays
    // hold lower corners; a box of the previous round's arrays (stored compact
    // if cprv) is completed with its query's widths when it is used
    const bool compact = S.allu != 0;
    const double* const cprev = reinterpret_cast<const double*>(bprev);
    double* const ccur = reinterpret_cast<double*>(bx);
    // load box r of the previous level or of the pool into o (a compact
    // parent only with its lower corner: completed when it is used)
    auto fetch = [&](unsigned int r, Box& o) {
      if (!(r & kRefRoot)) {
        if (cprv) {
          const double* q = cprev + 3 * (size_t)(r & kRefSrcMask);
          o.t0 = q[0]; o.u0 = q[1]; o.v0 = q[2];
        } else {
          o = bprev[r & kRefSrcMask];
        }
      } else if ((r & kRefExt) == kRefExt) {
        o = pool[r & kRefSrcMask];
      }
    };
    // a box of the current level (compact: completed with the level's widths)
    auto box_at = [&](int x, int s) -> Box {
      if (!compact) return bx[x];
      const double* q = ccur + 3 * (size_t)x;
      const double* w = S.w[s];
      return Box{q[0], q[0] + w[0], q[1], q[1] + w[1], q[2], q[2] + w[2]};
    };
    unsigned int r_cur = tid < n1 ? rf[tid] : kRefRoot;
    Box p_cur;
    // (global tier: the parent's flag byte travels with the parent box)
    const uint8_t* const flp = pick(flags, prv);
    uint8_t pf_cur = 0;
    fetch(r_cur, p_cur);
    if (!Cfg::SMEM && !(r_cur & kRefRoot)) pf_cur = flp[r_cur & kRefSrcMask];
    unsigned int r_nxt = tid + NT < n1 ? rf[tid + NT] : kRefRoot;
    // (global flags: prefetched one iteration ahead as well)
    uint8_t f_cur = 0;
    if constexpr (!Cfg::SMEM) f_cur = tid < n1 ? fl[tid] : 0;
    // (warp-uniform trip count: every lane reaches the chunk ballots)
    for (int i = tid; i - lane < n1; i += NT) {
      uint8_t f_pre = 0;
      if constexpr (!Cfg::SMEM) {
        f_pre = f_cur;
        f_cur = i + NT < n1 ? fl[i + NT] : 0;
      }
      Box p_nxt;
      uint8_t pf_nxt = 0;
      fetch(r_nxt, p_nxt);
      if (!Cfg::SMEM && !(r_nxt & kRefRoot)) pf_nxt = flp[r_nxt & kRefSrcMask];
      const unsigned int r_nn = i + 2 * NT < n1 ? rf[i + 2 * NT] : kRefRoot;
      const unsigned int r = r_cur;
      Box p = p_cur;
      const uint8_t pf = pf_cur;
      pf_cur = pf_nxt;
      r_cur = r_nxt;
      p_cur = p_nxt;
      r_nxt = r_nn;
      uint8_t f = 0;
      if (i < n1) {
      const int s = ONEQ ? 0 : sl[i];
      const QueryParams& qp = S.qp[s];
      if (cprv && !(r & kRefRoot)) {  // complete the parent (or the box itself)
        const double* wq = (r & kRefSelf) ? S.w[s] : S.wp[s];
        p.t1 = p.t0 + wq[0]; p.u1 = p.u0 + wq[1]; p.v1 = p.v0 + wq[2];
      }
      Box b;
      f = Cfg::SMEM ? fl[i] : f_pre;  // head bit (+ class, for roots and deferred boxes)
      double wb = 0.0;
      // every kind of box but the root starts from the loaded box p: handed
      // over (unclassified), deferred (itself, class carried) or a child
      // (p with one bound replaced by the parent's midpoint)
      b = p;
      if (r & kRefRoot) {
        if ((r & kRefExt) != kRefExt) {
          b = Box{0.0, qp.t_max, 0.0, 1.0, 0.0, 1.0};
          wb = S.root_wb[s];
        }
      } else if (r & kRefSelf) {
        if ((f & kClassified) && (f & 3) != kDisjoint) wb = wbp[r & kRefSrcMask];
      } else {
        // the parent's split: its dimension is in its flag byte (loaded with
        // the parent box in the global tier), the midpoint is recomputed
        // exactly
        const int src = (int)(r & kRefSrcMask);
        const int sdim = ((Cfg::SMEM ? flp[src] : pf) >> 3) & 3;
        const bool up = (r & kRefCb) != 0;
        if (sdim == 0) {
          const double mid = 0.5 * (p.t0 + p.t1);
          if (up) b.t0 = mid; else b.t1 = mid;
        } else if (sdim == 1) {
          const double mid = 0.5 * (p.u0 + p.u1);
          if (up) b.u0 = mid; else b.u1 = mid;
        } else {
          const double mid = 0.5 * (p.v0 + p.v1);
          if (up) b.v0 = mid; else b.v1 = mid;
        }
      }
#ifdef TCCD_DEBUG_ROOT
      if ((r & kRefRoot) && (r & kRefExt) != kRefExt) {
        if (f & kClassified) atomicAdd(&io.phase[13], 1ull);
        else if (!(i <= S.cutpos[s])) atomicAdd(&io.phase[14], 1ull);
        else atomicAdd(&io.phase[15], 1ull);
      }
#endif
      if (!(f & kClassified)) {
        if (i <= S.cutpos[s]) {
          const uint8_t head = f & kHead;
          const int cls = classify((const double*)S.P[s], qp.kind, b, qp.eps, qp.sep, wb, qp.tame != 0);
          ncls_ee += qp.kind;  // (kind is 0 or 1)
          ncls_vf += 1 - qp.kind;
          f = (uint8_t)cls;
          if (cls != kDisjoint) {
            int sdim; double mid; bool ph;
            const bool acc = split_decision(b, cls, wb, qp.kap, qp.delta, qp.kind, sdim, mid, ph);
            f = make_flag(cls, acc, sdim, ph);
          }
          f |= kClassified | head;
        }
      }
      if ((f & 3) != kDisjoint) {
        // only non-disjoint boxes are read again (parents, first / drop
        // records, merge keys): disjoint ones are never stored, which keeps
        // the level arrays' footprint in L2
        if (compact) {
          double* q = ccur + 3 * (size_t)i;
          q[0] = b.t0; q[1] = b.u0; q[2] = b.v0;
        } else {
          bx[i] = b;
        }
        // (classified here or carried, e.g. the root's: the same for every
        // refining box of a dyadic query's level)
        if (!(f & 4)) S.lvl_sdim[s] = (f >> 3) & 3;
        wbc[i] = wb;
        atomicMin(&S.j[s], i);
        // first accepted box: if it is not j itself it lies after j, and it is
        // the only candidate for the drop record (boxes are in t_lo order)
        if (f & 4) atomicMin(&S.acc[s], i);
      }
      fl[i] = f;
      }  // i < n
      // chunk masks (f = 0 past the end: disjoint, no head)
      {
        const bool refine = (f & 3) != kDisjoint && !(f & 4);
        const int sd = (f >> 3) & 3;
        const unsigned int mr = __ballot_sync(0xffffffffu, refine);
        const unsigned int mu = __ballot_sync(0xffffffffu, refine && sd != 0 && (f & 32));
        const unsigned int mt = __ballot_sync(0xffffffffu, refine && sd == 0);
        const unsigned int mh = __ballot_sync(0xffffffffu, (f & kHead) != 0);
        if (lane == 0) {
          const int c = (i - lane) >> 5;
          ch.m[kMR][c] = mr;
          ch.m[kMU][c] = mu;
          ch.m[kMT][c] = mt;
          ch.m[kMH][c] = mh;
        }
      }
    }
    gsync<G>();
    TCCD_PHASE(3);
    // ================= P3: per-query outcome (O(1) replay of the level's events)
    for (int s = tid; s < Q; s += NT) {
      if (S.qidx[s] < 0) continue;
      const int nn = S.seg_n[s];
      const long long C = S.C[s], mc = S.qp[s].max_checks;
      const long long cut = mc - C - 1;
      const long long ecls = nn < cut + 1 ? nn : cut + 1;
      const int j = S.j[s] == kIntMax ? kIntMax : S.j[s] - S.seg_off[s];  // (segment-relative)
      bool done = true;
#ifdef TCCD_DEBUG_ROOT
      if (j >= ecls && S.level[s] == 0 && C == 0 && !(S.root_flag[s] & kClassified)) {
        const Box rb = {0.0, S.qp[s].t_max, 0.0, 1.0, 0.0, 1.0};
        double w2;
        const int c2 = classify((const double*)S.P[s], S.qp[s].kind, rb, S.qp[s].eps, S.qp[s].sep, w2,
                                S.qp[s].tame != 0);
        if (c2 != kDisjoint) atomicAdd(&io.phase[12], 1ull);
        if (c2 != kDisjoint && nn != 1) atomicAdd(&io.phase[11], 1ull);
        if (c2 != kDisjoint) atomicAdd(&io.phase[10], (unsigned long long)(fl[S.seg_off[s]]));
      }
#endif
      if (j >= ecls) {
        if (cut < nn) {
          algo += mc - C;
          if (S.have_drop[s] || cut + 1 < nn) finish(s, true, mc);
          else free_result(s, mc);
        } else if (S.have_drop[s]) {
          algo += nn;
          const Rec& r = S.rec[s][1];
          write_result(a, S.qidx[s], kHit, r.b, r.codom, C + nn, 0, r.level);
        } else {
          algo += nn;
          free_result(s, C + nn);
        }
      } else {
        const int ij = S.seg_off[s] + j;
        const Box bj = box_at(ij, s);
        const double wbj = wbc[ij];
        Rec& fr = S.rec[s][0];
        fr.b = bj;
        fr.codom = wbj;
        fr.level = S.level[s];
        S.have_first[s] = 1;
        if (j == cut) {
          algo += mc - C;
          finish(s, true, mc);
        } else if (fl[ij] & 4) {
          algo += j + 1;
          // first colliding box of a fresh level accepted (_kernel.py:243-252)
          if (S.have_drop[s] && S.rec[s][1].b.t0 < bj.t0) {
            const Rec& r = S.rec[s][1];
            write_result(a, S.qidx[s], kHit, r.b, r.codom, C + j + 1, 0, r.level);
          } else {
            write_result(a, S.qidx[s], kHit, bj, wbj, C + j + 1, 0, S.level[s]);
          }
        } else {
          const long long eend = nn < cut ? nn : cut;
          const int ai = S.acc[s] == kIntMax ? kIntMax : S.acc[s] - S.seg_off[s];
          if (ai < eend) {
            const Box ba = box_at(S.seg_off[s] + ai, s);
            if (!S.have_drop[s] || ba.t0 < S.rec[s][1].b.t0) {
              Rec& dr = S.rec[s][1];
              dr.b = ba;
              dr.codom = wbc[S.seg_off[s] + ai];
              dr.level = S.level[s];
            }
            S.have_drop[s] = 1;
          }
          if (cut < nn) {
            algo += mc - C;
            finish(s, true, mc);
          } else {
            algo += nn;
            done = false;
            S.cont[s] = 1;
            S.C[s] = C + nn;
          }
        }
      }
      if (done) S.qidx[s] = -1;
    }
    // (P4 reads only P1's chunk masks, so it needs no barrier after P3; the
    // one-query tiers read P3's outcome below)
    if constexpr (ONEQ) gsync<G>();
    TCCD_PHASE(4);
    const int nxt = prv;
    // one query that ended this round: no next level to build
    const bool build_next = !(ONEQ && S.cont[0] == 0);
    if (!build_next && tid == 0) { S.n_next = 0; S.deferred_last = 0; }
    if (build_next) {
    // ================= P4: chunk scan -> flat prefixes (A, B, refining boxes P)
    // Threads own contiguous ranges of 32-box chunks (one or two chunks each
    // in the shared-memory tiers).  Every query's boxes are counted (also
    // finished ones): positions are segment-relative, so that only shifts the
    // flat numbering.  The run carries M / N come from a forward max-scan and
    // a reverse min-scan of the chunks' run heads.
    {
      const int nch = (n + 31) >> 5;
      const int cpt = (nch + NT - 1) / NT;
      const int c0 = tid * cpt < nch ? tid * cpt : nch;
      const int c1 = c0 + cpt < nch ? c0 + cpt : nch;
      unsigned int sA = 0, sB = 0;
      int sP = 0, lastHeadP = -1, firstHeadP = -1;
      for (int c = c0; c < c1; ++c) {
        const unsigned int R = ch.m[kMR][c], H = ch.m[kMH][c];
        if (H) {
          if (firstHeadP < 0) firstHeadP = sP + __popc(R & lowmask(__ffs(H) - 1));
          lastHeadP = sP + __popc(R & lowmask(31 - __clz(H)));
        }
        const int pr = __popc(R);
        sP += pr;
        sA += pr + __popc(ch.m[kMU][c]);
        sB += __popc(ch.m[kMT][c]);
      }
      unsigned long long pre, preP, tot, totP;
      group_excl_scan2<G>(((unsigned long long)sA << 32) | sB, (unsigned long long)sP, S.sw, pre,
                          preP, tot, totP);
      const int P0 = (int)preP;
      int carryM, carryN;
      group_scan_maxfwd_minrev<G>(lastHeadP >= 0 ? P0 + lastHeadP : -1,
                                  firstHeadP >= 0 ? P0 + firstHeadP : kIntMax, S.swi, carryM,
                                  carryN);
      if (carryN == kIntMax) carryN = (int)totP;
      if (tid == 0) {
        S.A_tot = (int)(tot >> 32);
        S.B_tot = (int)(tot & 0xffffffffu);
        S.P_tot = (int)totP;
        S.any_general = 0;
      }
      int Ar = (int)(pre >> 32), Br = (int)(pre & 0xffffffffu), Pr = P0, M = carryM;
      for (int c = c0; c < c1; ++c) {
        const unsigned int R = ch.m[kMR][c], H = ch.m[kMH][c];
        ch.c[kCA][c] = Ar;
        ch.c[kCB][c] = Br;
        ch.c[kCP][c] = Pr;
        ch.c[kCM][c] = M;
        if (H) M = Pr + __popc(R & lowmask(31 - __clz(H)));
        const int pr = __popc(R);
        Pr += pr;
        Ar += pr + __popc(ch.m[kMU][c]);
        Br += __popc(ch.m[kMT][c]);
      }
      int N = carryN;
      for (int c = c1 - 1; c >= c0; --c) {
        ch.c[kCN][c] = N;
        const unsigned int H = ch.m[kMH][c];
        if (H) N = ch.c[kCP][c] + __popc(ch.m[kMR][c] & lowmask(__ffs(H) - 1));
      }
    }
    gsync<G>();
    TCCD_PHASE(5);
    // ================= P5: next-level layout (slot order), eviction, deferral
    // Levels above the tier's per-query cap go to the next tier.  Otherwise
    // the first K slots (rotating order) keep their children and the rest
    // are deferred, K = the largest k with
    //   sum_{r<k} children_r + sum_{r>=k} boxes_r <= cap
    // (at least one query advances: if none fits, the first is evicted).
    // Segment bounds of the flat prefixes, O(1) each from the chunk masks.
    {
      const int A_tot = S.A_tot, B_tot = S.B_tot, P_tot = S.P_tot;
      auto prefix = [&](int x, int& pa, int& pb, int& pp) {
        if (x >= n) { pa = A_tot; pb = B_tot; pp = P_tot; return; }
        const int c = x >> 5;
        const unsigned int lm = lowmask(x & 31);
        const int pr = __popc(ch.m[kMR][c] & lm);
        pa = ch.c[kCA][c] + pr + __popc(ch.m[kMU][c] & lm);
        pb = ch.c[kCB][c] + __popc(ch.m[kMT][c] & lm);
        pp = ch.c[kCP][c] + pr;
      };
      for (int s = tid; s < Q; s += NT) {
        int t = 0;
        if (S.cont[s]) {
          int a0, b0, p0, a1, b1, p1;
          prefix(S.seg_off[s], a0, b0, p0);
          prefix(S.seg_off[s] + S.seg_n[s], a1, b1, p1);
          S.segA0[s] = a0; S.segB0[s] = b0; S.segP0[s] = p0;
          S.segA1[s] = a1; S.segB1[s] = b1; S.segP1[s] = p1;
          S.pc[s] = make_int4(0, p0, p1, a0);
          t = (a1 - a0) + (b1 - b0);
          if (!S.uniform[s]) S.any_general = 1;
          if (t > qcap) evict(s, t);
        }
        S.tot[s] = t;
      }
    }
    gsync<G>();
    TCCD_PHASE(6);
    if (tid < 32) {
      const int lane = tid;
      // layout order: all vertex-face queries, then all edge-edge queries
      // (rotating start), so the next level's warps see one kind only and
      // classify() does not diverge on the kind
      constexpr int kV = 2 * Q;
      constexpr int kPer = (kV + 31) / 32;
      auto vslot = [&](int rpos) -> int {
        if (rpos >= kV) return -1;
        const int s = (S.rot + (rpos % Q)) % Q;
        return S.qp[s].kind == (rpos >= Q ? 1 : 0) ? s : -1;
      };
      int vt[kPer], vn[kPer];
      int st, sn, it, in, Nn, K;
      for (;;) {
        st = 0; sn = 0;
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
          const int rpos = lane * kPer + m;
          const int s = vslot(rpos);
          const bool ok = s >= 0 && S.cont[s] == 1;
          vt[m] = ok ? S.tot[s] : 0;
          vn[m] = ok ? S.seg_n[s] : 0;
          st += vt[m];
          sn += vn[m];
        }
        it = st; in = sn;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int yt = __shfl_up_sync(0xffffffffu, it, o);
          const int yn = __shfl_up_sync(0xffffffffu, in, o);
          if (lane >= o) { it += yt; in += yn; }
        }
        Nn = __shfl_sync(0xffffffffu, in, 31);
        int pt = it - st, pn = in - sn;
        int bestk = 0;
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
          pt += vt[m];
          pn += vn[m];
          if (vn[m] > 0 && pt + (Nn - pn) <= cap) bestk = lane * kPer + m + 1;
        }
        K = bestk;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) K = max(K, __shfl_xor_sync(0xffffffffu, K, o));
        if (K > 0 || Nn == 0) break;
        const unsigned int has = __ballot_sync(0xffffffffu, sn > 0);
        if (lane == __ffs(has) - 1) {
#pragma unroll
          for (int m = 0; m < kPer; ++m) {
            const int rpos = lane * kPer + m;
            const int s = vslot(rpos);
            if (vn[m] > 0) { evict(s, S.tot[s]); break; }
          }
        }
        __syncwarp();
      }
      int cT = 0, cN = 0;
#pragma unroll
      for (int m = 0; m < kPer; ++m)
        if (lane * kPer + m < K) { cT += vt[m]; cN += vn[m]; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cT += __shfl_xor_sync(0xffffffffu, cT, o);
        cN += __shfl_xor_sync(0xffffffffu, cN, o);
      }
      int ut = it - st, un = in - sn;
      int deferred = 0;
#pragma unroll
      for (int m = 0; m < kPer; ++m) {
        const int rpos = lane * kPer + m;
        const int s = vslot(rpos);
        if (s >= 0 && S.cont[s] == 1) {
          if (rpos < K) {
            S.next_off[s] = ut;
            S.pc[s].x = ut;
            if (S.uniform[s]) S.pc_mode[s] = kPcKeep;
          } else {
            S.next_off[s] = cT + (un - cN);
            S.pc[s].x = cT + (un - cN);
            S.pc[s].y = S.seg_off[s];
            S.pc_mode[s] = kPcCarry;
            S.cont[s] = 2;
            ++deferred;
          }
        }
        ut += vt[m];
        un += vn[m];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) deferred += __shfl_xor_sync(0xffffffffu, deferred, o);
      if (lane == 0) {
        S.n_next = cT + (Nn - cN);
        S.rot = (S.rot + 1) % Q;
        S.deferred += deferred;
        S.deferred_last = deferred;
      }
    }
    gsync<G>();
    TCCD_PHASE(7);
    // ================= P4c: next level of uniform queries, closed form; deferred carry
    // For dyadic t_max every box of a level has the same widths, hence the
    // same split dimension.  u/v split: the children are already in stable
    // t_lo order (push order).  t split: within a run of equal t_lo, all
    // lower children (t_lo kept) then all upper children (t_lo + w/2, below
    // the next run's t_lo), so with P = refining boxes before the parent,
    // M / N = P at the run's head / at the next head (or the segment end):
    //   rank(lower) = M + P,  rank(upper) = N + P   (segment-relative).
    // New run heads: the children of the first refining box of a run.
    // Lane per box; P, M, N and A from the chunk masks in O(1).
    {
      unsigned int* const outr = pick(ar.ref, nxt);
      uint8_t* const sln = pick(slot_of, nxt);
      uint8_t* const fln = pick(flags, nxt);
      // (only deferred levels copy non-refining boxes: without deferrals this
      // round, the chunk mask settles those boxes without touching them)
      const bool any_deferred = S.deferred_last != 0;
      if (ONEQ && S.cont[0] == 1 && S.uniform[0]) {
        // one continuing query: warp per chunk, the chunk words (global) of
        // several chunks in flight together; slot bytes are not written (only
        // the general ordering path reads them)
        constexpr int CS = NT / 32;
        const int nch = (n + 31) >> 5;
        const int base = S.next_off[0], S0 = S.segP0[0], S1 = S.segP1[0], A0 = S.segA0[0];
        const unsigned int lm = lowmask(lane), bit = 1u << lane;
        // four chunks per pass: their 32 words are loaded together
        constexpr int UN = 4;
        for (int c0 = tid >> 5; c0 < nch; c0 += UN * CS) {
          unsigned int R[UN], H[UN], T[UN], U[UN];
          int cP[UN], cM[UN], cN[UN], cA[UN];
#pragma unroll
          for (int u = 0; u < UN; ++u) {
            const int c = c0 + u * CS;
            R[u] = 0; H[u] = 0; T[u] = 0; U[u] = 0; cP[u] = 0; cM[u] = 0; cN[u] = 0; cA[u] = 0;
            if (c < nch) {
              R[u] = ch.m[kMR][c]; H[u] = ch.m[kMH][c]; T[u] = ch.m[kMT][c]; U[u] = ch.m[kMU][c];
              cP[u] = ch.c[kCP][c]; cM[u] = ch.c[kCM][c]; cN[u] = ch.c[kCN][c]; cA[u] = ch.c[kCA][c];
            }
          }
#pragma unroll
          for (int u = 0; u < UN; ++u) {
            if (!(R[u] & bit)) continue;
            const int Pr = cP[u] + __popc(R[u] & lm);
            const unsigned int hle = H[u] & (lm | bit), hgt = H[u] & ~(lm | bit);
            const int M = hle ? cP[u] + __popc(R[u] & lowmask(31 - __clz(hle))) : cM[u];
            int N = hgt ? cP[u] + __popc(R[u] & lowmask(__ffs(hgt) - 1)) : cN[u];
            if (N > S1) N = S1;
            const bool tsplit = (T[u] & bit) != 0;
            const uint8_t hd = Pr == M ? kHead : 0;
            const int i = (c0 + u * CS) * 32 + lane;
            int rl, ru = -1;
            if (tsplit) {
              rl = (M - S0) + (Pr - S0);
              ru = (N - S0) + (Pr - S0);
            } else {
              rl = cA[u] + __popc(R[u] & lm) + __popc(U[u] & lm) - A0;
              if (U[u] & bit) ru = rl + 1;
            }
            TCCD_ASSERT(base + rl < cap && base + ru < cap);
            outr[base + rl] = (unsigned)i;
            fln[base + rl] = hd;
            if (ru >= 0) {
              outr[base + ru] = (unsigned)i | kRefCb;
              fln[base + ru] = tsplit ? hd : 0;
            }
          }
        }
      } else if constexpr (!ONEQ) {
        // lane per box; the slot's view is one 16-byte word (pc) and a mode
        for (int i = tid; i < n; i += NT) {
          const int c = i >> 5, l = i & 31;
          const unsigned int lm = lowmask(l), bit = 1u << l;
          const unsigned int R = ch.m[kMR][c];
          if (!any_deferred && !(R & bit)) continue;
          const int s = sl[i];
          const int md = S.pc_mode[s];
          if (md == 0) continue;
          const int4 pv = S.pc[s];
          if (md == kPcCarry) {
            const int pos = pv.x + (i - pv.y);
            TCCD_ASSERT(pos < cap);
            outr[pos] = (unsigned)i | kRefSelf;
            sln[pos] = (uint8_t)s;
            fln[pos] = fl[i];
            continue;
          }
          if (!(R & bit)) continue;
          const unsigned int H = ch.m[kMH][c], T = ch.m[kMT][c], U = ch.m[kMU][c];
          const int cP = ch.c[kCP][c], cM = ch.c[kCM][c], cN = ch.c[kCN][c], cA = ch.c[kCA][c];
          const int Pr = cP + __popc(R & lm);
          const unsigned int hle = H & (lm | bit), hgt = H & ~(lm | bit);
          const int M = hle ? cP + __popc(R & lowmask(31 - __clz(hle))) : cM;
          int N = hgt ? cP + __popc(R & lowmask(__ffs(hgt) - 1)) : cN;
          if (N > pv.z) N = pv.z;  // the last run ends at the segment end
          const int S0 = pv.y;
          const bool tsplit = (T & bit) != 0;
          const uint8_t hd = Pr == M ? kHead : 0;
          int rl, ru = -1;
          if (tsplit) {
            rl = (M - S0) + (Pr - S0);
            ru = (N - S0) + (Pr - S0);
          } else {
            rl = cA + __popc(R & lm) + __popc(U & lm) - pv.w;
            if (U & bit) ru = rl + 1;
          }
          const uint8_t hu = tsplit ? hd : 0;
          if (md == kPcKeep) {
            const int base = pv.x;
            TCCD_ASSERT(base + rl < cap && base + ru < cap);
            outr[base + rl] = (unsigned)i;
            sln[base + rl] = (uint8_t)s;
            fln[base + rl] = hd;
            if (ru >= 0) {
              outr[base + ru] = (unsigned)i | kRefCb;
              sln[base + ru] = (uint8_t)s;
              fln[base + ru] = hu;
            }
          } else {
            // materialize the handed-over level in the next tier's pool
            const long long base = S.hoff[s];
            const Box pb = box_at(i, s);
            double mid;
            const int sd = split_dim(pb, S.qp[s].kap, mid);
            Box c0, c1;
            children(pb, sd, mid, c0, c1);
            TCCD_ASSERT(base + rl < io.pool_cap && base + ru < io.pool_cap);
            io.out_pbox[base + rl] = c0;
            io.out_pflag[base + rl] = hd;
            if (ru >= 0) {
              io.out_pbox[base + ru] = c1;
              io.out_pflag[base + ru] = hu;
            }
          }
        }
      } else
      for (int i = tid; i < n; i += NT) {
        const int c = i >> 5, l = i & 31;
        const unsigned int lm = lowmask(l), bit = 1u << l;
        // (one query: the chunk words are global; issue them together)
        unsigned int R = ch.m[kMR][c], H, T, U;
        int cP, cM, cN, cA;
        if constexpr (ONEQ) {
          H = ch.m[kMH][c]; T = ch.m[kMT][c]; U = ch.m[kMU][c];
          cP = ch.c[kCP][c]; cM = ch.c[kCM][c]; cN = ch.c[kCN][c]; cA = ch.c[kCA][c];
        }
        if (!any_deferred && !(R & bit)) continue;
        const int s = ONEQ ? 0 : sl[i];
        const int cs = S.cont[s];
        if (cs == 0) continue;
        if (cs == 2) {
          const int pos = S.next_off[s] + (i - S.seg_off[s]);
          TCCD_ASSERT(pos < cap);
          outr[pos] = (unsigned)i | kRefSelf;
          sln[pos] = (uint8_t)s;
          fln[pos] = fl[i];
          continue;
        }
        // refining boxes only; their split dimension and clipped upper child
        // are in the chunk masks (T: t split, U: u / v split with an upper child)
        if (!(R & bit) || !S.uniform[s]) continue;
        const bool hand = cs == 3 && S.hoff[s] >= 0;
        if (cs != 1 && !hand) continue;
        if constexpr (!ONEQ) {
          H = ch.m[kMH][c]; T = ch.m[kMT][c]; U = ch.m[kMU][c];
          cP = ch.c[kCP][c]; cM = ch.c[kCM][c]; cN = ch.c[kCN][c]; cA = ch.c[kCA][c];
        }
        const int Pr = cP + __popc(R & lm);
        const unsigned int hle = H & (lm | bit), hgt = H & ~(lm | bit);
        const int M = hle ? cP + __popc(R & lowmask(31 - __clz(hle))) : cM;
        int N = hgt ? cP + __popc(R & lowmask(__ffs(hgt) - 1)) : cN;
        if (N > S.segP1[s]) N = S.segP1[s];  // the last run ends at the segment end
        const int S0 = S.segP0[s];
        const bool tsplit = (T & bit) != 0;
        const uint8_t hd = Pr == M ? kHead : 0;
        int rl, ru = -1;
        if (tsplit) {
          rl = (M - S0) + (Pr - S0);
          ru = (N - S0) + (Pr - S0);
        } else {
          rl = cA + __popc(R & lm) + __popc(U & lm) - S.segA0[s];
          if (U & bit) ru = rl + 1;
        }
        const uint8_t hu = tsplit ? hd : 0;
        if (!hand) {
          const int base = S.next_off[s];
          TCCD_ASSERT(base + rl < cap && base + ru < cap);
          outr[base + rl] = (unsigned)i;
          sln[base + rl] = (uint8_t)s;
          fln[base + rl] = hd;
          if (ru >= 0) {
            outr[base + ru] = (unsigned)i | kRefCb;
            sln[base + ru] = (uint8_t)s;
            fln[base + ru] = hu;
          }
        } else {
          // materialize the handed-over level in the next tier's pool
          const long long base = S.hoff[s];
          const Box pb = box_at(i, s);
          double mid;
          const int sd = split_dim(pb, S.qp[s].kap, mid);
          Box c0, c1;
          children(pb, sd, mid, c0, c1);
          TCCD_ASSERT(base + rl < io.pool_cap && base + ru < io.pool_cap);
          io.out_pbox[base + rl] = c0;
          io.out_pflag[base + rl] = hd;
          if (ru >= 0) {
            io.out_pbox[base + ru] = c1;
            io.out_pflag[base + ru] = hu;
          }
        }
      }
    }
    gsync<G>();
    TCCD_PHASE(8);
    if (S.any_general) {
    // ================= P5b: A / B entries (key, push, ref)
    // Entries are written for every refining box of the list (whatever its
    // query's state) so that no stale entry sits inside the flat A / B ranges.
    for (int i = tid; i < n; i += NT) {
      const uint8_t f = fl[i];
      if ((f & 3) == kDisjoint || (f & 4)) continue;
      const int sdim = (f >> 3) & 3;
      const Box b = box_at(i, ONEQ ? 0 : sl[i]);
      const int c = i >> 5;
      const unsigned int lm = lowmask(i & 31);
      const unsigned int oa = (unsigned)(ch.c[kCA][c] + __popc(ch.m[kMR][c] & lm) +
                                         __popc(ch.m[kMU][c] & lm));
      const unsigned int ob = (unsigned)(ch.c[kCB][c] + __popc(ch.m[kMT][c] & lm));
      const unsigned int push = oa + ob;
      const unsigned long long k0 = tkey(b.t0);
      TCCD_ASSERT(oa + 1 < 2 * cap && ob < cap);
      ar.akey[oa] = k0;
      ar.apush[oa] = push;
      ar.aref[oa] = (unsigned)i;
      if (sdim != 0) {
        if (f & 32) {
          ar.akey[oa + 1] = k0;
          ar.apush[oa + 1] = push + 1;
          ar.aref[oa + 1] = (unsigned)i | kRefCb;
        }
      } else {
        ar.bkey[ob] = tkey(0.5 * (b.t0 + b.t1));
        ar.bpush[ob] = push + 1;
        ar.bref[ob] = (unsigned)i | kRefCb;
      }
    }
    gsync<G>();
    // B runs sorted?  (always, for dyadic t_max)
    {
      const int B_tot = S.B_tot;
      for (int b = tid + 1; b < B_tot; b += NT) {
        const int s = sl[ar.bref[b] & kRefSrcMask];
        if (!(S.cont[s] == 1 || (S.cont[s] == 3 && S.hoff[s] >= 0)) || S.uniform[s] ||
            b <= S.segB0[s])
          continue;
        if (ar.bkey[b - 1] > ar.bkey[b]) S.unsorted[s] = 1;
      }
    }
    gsync<G>();
    // ================= P6: merge by rank into the next level's reference list
    {
      const int A_tot = S.A_tot, B_tot = S.B_tot;
      unsigned int* out = pick(ar.ref, nxt);
      uint8_t* sln = pick(slot_of, nxt);
      uint8_t* fln = pick(flags, nxt);
      for (int e = tid; e < A_tot + B_tot; e += NT) {
        const bool isA = e < A_tot;
        const int x = isA ? e : e - A_tot;
        const unsigned int r = isA ? ar.aref[x] : ar.bref[x];
        const int s = sl[r & kRefSrcMask];
        const bool hand = S.cont[s] == 3 && S.hoff[s] >= 0;
        if (!(S.cont[s] == 1 || hand) || S.uniform[s]) continue;
        const unsigned long long kk = isA ? ar.akey[x] : ar.bkey[x];
        const unsigned int pp = isA ? ar.apush[x] : ar.bpush[x];
        int rank;
        if (!S.unsorted[s]) {
          if (isA) {
            int l = S.segB0[s], h = S.segB1[s];  // B elements < (kk, pp)
            while (l < h) {
              const int m = (l + h) >> 1;
              if (kp_less(ar.bkey[m], ar.bpush[m], kk, pp)) l = m + 1;
              else h = m;
            }
            rank = (x - S.segA0[s]) + (l - S.segB0[s]);
          } else {
            int l = S.segA0[s], h = S.segA1[s];  // A elements < (kk, pp)
            while (l < h) {
              const int m = (l + h) >> 1;
              if (kp_less(ar.akey[m], ar.apush[m], kk, pp)) l = m + 1;
              else h = m;
            }
            rank = (x - S.segB0[s]) + (l - S.segA0[s]);
          }
        } else {
          // exact rank count over the query's children (general t_max)
          rank = 0;
          for (int m = S.segA0[s]; m < S.segA1[s]; ++m)
            rank += kp_less(ar.akey[m], ar.apush[m], kk, pp) ? 1 : 0;
          for (int m = S.segB0[s]; m < S.segB1[s]; ++m)
            rank += kp_less(ar.bkey[m], ar.bpush[m], kk, pp) ? 1 : 0;
        }
        if (!hand) {
          const int pos = S.next_off[s] + rank;
          TCCD_ASSERT(pos < cap);
          out[pos] = r;
          sln[pos] = (uint8_t)s;
          fln[pos] = 0;
        } else {
          const Box pb = box_at(r & kRefSrcMask, s);
          double mid;
          const int sd = split_dim(pb, S.qp[s].kap, mid);
          Box c0, c1;
          children(pb, sd, mid, c0, c1);
          TCCD_ASSERT(S.hoff[s] + rank < io.pool_cap);
          io.out_pbox[S.hoff[s] + rank] = (r & kRefCb) ? c1 : c0;
          io.out_pflag[S.hoff[s] + rank] = 0;
        }
      }
    }
    gsync<G>();
    }  // any_general
    }  // build_next
    // ================= P7: commit
    for (int s = tid; s < Q; s += NT) {
      if (S.cont[s] == 1) {
        S.seg_n[s] = S.tot[s];
        S.level[s] += 1;
        S.seg_off[s] = S.next_off[s];
        if (S.uniform[s]) {  // the next level's boxes: this level's split dimension halved
          double* w = S.w[s];
          S.wp[s][0] = w[0]; S.wp[s][1] = w[1]; S.wp[s][2] = w[2];
          w[S.lvl_sdim[s]] = 0.5 * w[S.lvl_sdim[s]];
        }
      } else if (S.cont[s] == 2) {
        S.C[s] -= S.seg_n[s];  // the level re-runs next round
        algo -= S.seg_n[s];
        S.seg_off[s] = S.next_off[s];
      }
    }
    gsync<G>();
    TCCD_PHASE(9);
    if (tid == 0) S.n_cur = S.n_next;
    cur = nxt;
    cprv = compact;
    gsync<G>();
    TCCD_PHASE(10);
  }
  if (tid == 0) {
    atomicAdd(io.rounds, (unsigned long long)rounds);
    atomicAdd(io.deferred, S.deferred);
    atomicAdd(io.boxes, boxes);
#ifdef TCCD_PHASE_PROF
    for (int k = 0; k < 11; ++k) atomicAdd(&io.phase[k], ph_acc[k]);
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    atomicAdd(&io.phase[11], t_end - t_start);  // group lifetime (ns)
    atomicAdd(&io.phase[12], 1ull);
    atomicMax(&io.phase[13], t_end);
    atomicMin(&io.phase[14], t_start);
#endif
  }
  if (evicted) atomicAdd(io.evicted, evicted);
  if (algo) atomicAdd(io.algo, (unsigned long long)algo);  // (two's complement: a signed sum)
  {  // (all lanes reach here: the round loop exits group-wide)
    const unsigned int wv = __reduce_add_sync(0xffffffffu, ncls_vf);
    const unsigned int we = __reduce_add_sync(0xffffffffu, ncls_ee);
    if (lane == 0 && wv) atomicAdd(&io.cls[0], (unsigned long long)wv);
    if (lane == 0 && we) atomicAdd(&io.cls[1], (unsigned long long)we);
  }
}

}  // namespace tccd
