// Pool engine: one persistent CTA keeps up to kPQ queries resident and
// advances all of them one BFS level per round.
//
// The current levels of all resident queries form one flat box list
// (segment per query, each segment in the reference's visiting order:
// stable by t_lo, _kernel.py:174-175).  A round:
//   P1 classify every box (lane per box, queries mixed) -> class flags;
//      block-wide atomicMin per query = first non-disjoint box j
//   P2 atomicMin per query = first accepted box after j before the budget
//      cut (the only box that can become the "drop" record)
//   P3 one thread per query replays the reference's events from (j, drop,
//      cut) in O(1): normal return, budget return, queue exhaustion or
//      continue (_kernel.py:176-312)
//   P4 block scan of child counts over the flat list (threads own
//      contiguous chunks); children land in two flat subsequences -- A
//      (t_lo = parent t_lo: lower children and u/v upper children) and B
//      (t-split upper children) -- each already sorted by (t_lo, push)
//   P5 per query: next-level extent, eviction of queries whose level
//      outgrew the pool (restarted by the block-per-query engine)
//   P6 every child computes its rank in its query's next level by a binary
//      search of the other subsequence (merge by rank); a query whose B run
//      is not sorted (non-dyadic t_max) uses an exact O(n) rank count
//   P7 commit; admission refills free slots from the global work counter.
// Box lists live in a per-CTA global arena (L2-resident working set); the
// per-box class flags and slot ids live in shared memory.
#pragma once

namespace tccd {

constexpr int kPT = 256;     // threads per pool CTA
constexpr int kPQ = 128;     // query slots per pool CTA
constexpr int kPCap = 8192;  // boxes per level buffer per CTA
constexpr int kPQCap = 4096; // largest per-query level kept in the pool
constexpr int kPAdmit = kPCap / 2;  // admit new queries only below this fill
constexpr uint8_t kPNone = 0xFF;
constexpr uint8_t kClassified = 64;  // flag bit: box already classified (deferred level)
constexpr int kIntMax = 0x7fffffff;

struct PoolRec {  // first / drop record of a slot (global)
  Box b;
  double codom;
  int level;
  int pad;
};

struct PoolArena {
  Box* lvl[2];            // [kPCap] level buffers (ping-pong)
  Box* ab;                // [2*kPCap] children: A from the front, B from the back
  unsigned long long* key;  // [2*kPCap]
  unsigned int* push;     // [2*kPCap] flat push index
  uint8_t* cslot;         // [2*kPCap] owning slot of each child
  double* wb[2];          // [kPCap] hull width per box (ping-pong with lvl)
  PoolRec* rec;           // [kPQ][2]
};

__host__ __device__ inline size_t pool_arena_bytes() {
  return 2 * align256((size_t)kPCap * sizeof(Box)) + align256((size_t)2 * kPCap * sizeof(Box)) +
         align256((size_t)2 * kPCap * 8) + align256((size_t)2 * kPCap * 4) +
         align256((size_t)2 * kPCap) + 2 * align256((size_t)kPCap * 8) +
         align256((size_t)kPQ * 2 * sizeof(PoolRec));
}

__device__ inline PoolArena pool_arena_at(unsigned char* base) {
  PoolArena r;
  size_t o = 0;
  r.lvl[0] = (Box*)(base + o); o += align256((size_t)kPCap * sizeof(Box));
  r.lvl[1] = (Box*)(base + o); o += align256((size_t)kPCap * sizeof(Box));
  r.ab = (Box*)(base + o); o += align256((size_t)2 * kPCap * sizeof(Box));
  r.key = (unsigned long long*)(base + o); o += align256((size_t)2 * kPCap * 8);
  r.push = (unsigned int*)(base + o); o += align256((size_t)2 * kPCap * 4);
  r.cslot = (uint8_t*)(base + o); o += align256((size_t)2 * kPCap);
  r.wb[0] = (double*)(base + o); o += align256((size_t)kPCap * 8);
  r.wb[1] = (double*)(base + o); o += align256((size_t)kPCap * 8);
  r.rec = (PoolRec*)(base + o);
  return r;
}

struct PoolShared {
  double P[kPQ][24];
  QueryParams qp[kPQ];
  long long C[kPQ];      // checks before the current level
  long long qidx[kPQ];   // -1: free slot
  double f_t0[kPQ], d_t0[kPQ];
  int level[kPQ];
  int seg_off[kPQ], seg_n[kPQ];
  int j[kPQ], acc[kPQ];
  int segA0[kPQ], segB0[kPQ], segA1[kPQ], segB1[kPQ];
  int next_off[kPQ];
  int tot[kPQ];          // children of the current level (continuing slots)
  uint8_t have_first[kPQ], have_drop[kPQ];
  uint8_t cont[kPQ];     // 1: level completed, children kept; 2: deferred
  uint8_t unsorted[kPQ];
  uint8_t slot_of[2][kPCap];
  uint8_t flag[2][kPCap];  // class flags; kClassified set once a box was checked
  unsigned long long sw[kPT / 32];
  int n_cur, n_next, admit_k, exhausted, A_tot, B_tot, rot;
  unsigned long long deferred;
  long long admit_base;
  unsigned int free_mask[kPQ / 32];
};

__device__ __forceinline__ void pool_write_rec(const Args& a, const PoolArena& ar, long long q,
                                               int which, long long checks, int early) {
  const PoolRec& r = ar.rec[which];
  write_result(a, q, kHit, r.b, r.codom, checks, early, r.level);
}

// report min(drop, first) (_kernel.py:192-199, 208-213)
__device__ __forceinline__ void pool_finish(const Args& a, const PoolArena& ar, PoolShared& S,
                                            int s, bool early, long long checks) {
  const bool use_drop = S.have_drop[s] && (!S.have_first[s] || S.d_t0[s] < S.f_t0[s]);
  const PoolRec& r = ar.rec[2 * s + (use_drop ? 1 : 0)];
  write_result(a, S.qidx[s], kHit, r.b, r.codom, checks, early, r.level);
}

__device__ __forceinline__ void pool_free(const Args& a, PoolShared& S, int s, long long checks) {
  const Box z = {0, 0, 0, 0, 0, 0};
  write_result(a, S.qidx[s], kFree, z, 0.0, checks, 0, 0);
}

__global__ void __launch_bounds__(kPT, 2) pool_kernel(Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PoolShared& S = *reinterpret_cast<PoolShared*>(smem_raw);
  const PoolArena ar = pool_arena_at(a.pool_arenas + (size_t)blockIdx.x * a.pool_arena_bytes);
  const int tid = threadIdx.x;
  if (tid < kPQ) S.qidx[tid] = -1;
  if (tid == 0) { S.n_cur = 0; S.exhausted = 0; S.rot = 0; S.deferred = 0; }
  __syncthreads();
  int cur = 0;
  long long rounds = 0;
  for (;;) {
    // ================= P0: admission
    if (tid < 32) {
      unsigned int cnt = 0;
      for (int w = 0; w < kPQ / 32; ++w) {
        const unsigned int m = __ballot_sync(0xffffffffu, S.qidx[w * 32 + tid] < 0);
        if (tid == 0) S.free_mask[w] = m;
        cnt += __popc(m);
      }
      if (tid == 0) {
        int k = (int)cnt;
        int room = kPAdmit - S.n_cur;  // headroom for the resident levels to grow
        if (room < 0) room = 0;
        if (k > room) k = room;
        long long base = 0;
        if (S.exhausted) k = 0;
        if (k > 0) {
          base = (long long)atomicAdd(&a.ctr->light_next, (unsigned long long)k);
          if (base >= a.n) { k = 0; S.exhausted = 1; }
          else if (base + k >= a.n) { k = (int)(a.n - base); S.exhausted = 1; }
        }
        S.admit_k = k;
        S.admit_base = base;
      }
    }
    __syncthreads();
    const int k_adm = S.admit_k;
    if (tid < kPQ) {
      const int s = tid;
      if (S.qidx[s] < 0 && k_adm > 0) {
        const int w = s >> 5, lane = s & 31;
        int r = __popc(S.free_mask[w] & ((1u << lane) - 1u));
        for (int ww = 0; ww < w; ++ww) r += __popc(S.free_mask[ww]);
        if (r < k_adm) {
          const long long q = S.admit_base + r;
          const int pos = S.n_cur + r;
          double* P = S.P[s];
          const double* src = a.points + 24 * q;
#pragma unroll
          for (int i = 0; i < 24; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(src + i);
            P[i] = v.x;
            P[i + 1] = v.y;
          }
          const uint8_t st = prologue(a, q, (const double*)P, S.qp[s]);
          if (st != kHit) {
            const Box z = {0, 0, 0, 0, 0, 0};
            write_result(a, q, st, z, 0.0, 0, 0, 0);
            S.slot_of[cur][pos] = kPNone;
          } else {
            S.qidx[s] = q;
            S.C[s] = 0;
            S.level[s] = 0;
            S.have_first[s] = 0;
            S.have_drop[s] = 0;
            S.seg_off[s] = pos;
            S.seg_n[s] = 1;
            ar.lvl[cur][pos] = Box{0.0, S.qp[s].t_max, 0.0, 1.0, 0.0, 1.0};
            S.slot_of[cur][pos] = (uint8_t)s;
            S.flag[cur][pos] = 0;
          }
        }
      }
      S.j[s] = kIntMax;
      S.acc[s] = kIntMax;
      S.cont[s] = 0;
      S.unsorted[s] = 0;
    }
    __syncthreads();
    if (tid == 0) S.n_cur += k_adm;
    __syncthreads();
    const int n = S.n_cur;
    if (n == 0) break;
    ++rounds;
    Box* lv = ar.lvl[cur];
    // ================= P1: classify (boxes of deferred levels keep their class)
    uint8_t* flg = S.flag[cur];
    double* wbc = ar.wb[cur];
    for (int i = tid; i < n; i += kPT) {
      const int s = S.slot_of[cur][i];
      if (s == kPNone) continue;
      const int k = i - S.seg_off[s];
      uint8_t f = flg[i];
      if (!(f & kClassified)) {
        const long long cut = S.qp[s].max_checks - S.C[s] - 1;
        if (k > cut) continue;  // past the budget: never checked
        const Box b = lv[i];
        const QueryParams& qp = S.qp[s];
        double wb;
        const int cls = classify((const double*)S.P[s], qp.kind, b, qp.eps, qp.sep, wb);
        f = (uint8_t)cls;
        if (cls != kDisjoint) {
          int sdim; double mid; bool ph;
          const bool acc = split_decision(b, cls, wb, qp.kap, qp.delta, qp.kind, sdim, mid, ph);
          f = make_flag(cls, acc, sdim, ph);
          wbc[i] = wb;
        }
        flg[i] = f | kClassified;
      }
      if ((f & 3) != kDisjoint) atomicMin(&S.j[s], k);
    }
    __syncthreads();
    // ================= P2: first accepted box after j, before the cut
    for (int i = tid; i < n; i += kPT) {
      const int s = S.slot_of[cur][i];
      if (s == kPNone) continue;
      const int k = i - S.seg_off[s];
      if (k <= S.j[s]) continue;
      const long long cut = S.qp[s].max_checks - S.C[s] - 1;
      const long long eend = S.seg_n[s] < cut ? S.seg_n[s] : cut;
      if (k >= eend) continue;
      const uint8_t f = flg[i];
      if ((f & 3) != kDisjoint && (f & 4)) atomicMin(&S.acc[s], k);
    }
    __syncthreads();
    // ================= P3: per-query outcome (O(1) replay of the level's events)
    if (tid < kPQ && S.qidx[tid] >= 0) {
      const int s = tid;
      const int nn = S.seg_n[s];
      const long long C = S.C[s], mc = S.qp[s].max_checks;
      const long long cut = mc - C - 1;
      const long long ecls = nn < cut + 1 ? nn : cut + 1;
      const int j = S.j[s];
      bool done = true;
      if (j >= ecls) {
        if (cut < nn) {
          if (S.have_drop[s] || cut + 1 < nn) pool_finish(a, ar, S, s, true, mc);
          else pool_free(a, S, s, mc);
        } else if (S.have_drop[s]) {
          const PoolRec& r = ar.rec[2 * s + 1];
          write_result(a, S.qidx[s], kHit, r.b, r.codom, C + nn, 0, r.level);
        } else {
          pool_free(a, S, s, C + nn);
        }
      } else {
        const int ij = S.seg_off[s] + j;
        const Box bj = lv[ij];
        const double wbj = wbc[ij];
        PoolRec& fr = ar.rec[2 * s];
        fr.b = bj;
        fr.codom = wbj;
        fr.level = S.level[s];
        S.have_first[s] = 1;
        S.f_t0[s] = bj.t0;
        if (j == cut) {
          pool_finish(a, ar, S, s, true, mc);
        } else if (flg[ij] & 4) {
          // first colliding box of a fresh level accepted (_kernel.py:243-252)
          if (S.have_drop[s] && S.d_t0[s] < bj.t0) {
            const PoolRec& r = ar.rec[2 * s + 1];
            write_result(a, S.qidx[s], kHit, r.b, r.codom, C + j + 1, 0, r.level);
          } else {
            write_result(a, S.qidx[s], kHit, bj, wbj, C + j + 1, 0, S.level[s]);
          }
        } else {
          const long long eend = nn < cut ? nn : cut;
          const int ai = S.acc[s];
          if (ai < eend) {
            const Box ba = lv[S.seg_off[s] + ai];
            if (!S.have_drop[s] || ba.t0 < S.d_t0[s]) {
              PoolRec& dr = ar.rec[2 * s + 1];
              dr.b = ba;
              dr.codom = wbc[S.seg_off[s] + ai];
              dr.level = S.level[s];
              S.d_t0[s] = ba.t0;
            }
            S.have_drop[s] = 1;
          }
          if (cut < nn) {
            pool_finish(a, ar, S, s, true, mc);
          } else {
            done = false;
            S.cont[s] = 1;
            S.C[s] = C + nn;
          }
        }
      }
      if (done) S.qidx[s] = -1;
    }
    __syncthreads();
    // ================= P4: children of continuing queries, flat A / B subsequences
    const int nxt = cur ^ 1;
    {
      const int c = (n + kPT - 1) / kPT;
      const int lo = tid * c;
      const int hi = lo + c < n ? lo + c : n;
      unsigned int sA = 0, sB = 0;
      for (int i = lo; i < hi; ++i) {
        const int s = S.slot_of[cur][i];
        if (s == kPNone || !S.cont[s]) continue;
        if (i - S.seg_off[s] < S.j[s]) continue;
        const uint8_t f = flg[i];
        if ((f & 3) == kDisjoint || (f & 4)) continue;
        const int sdim = (f >> 3) & 3;
        sA += 1 + ((sdim != 0 && (f & 32)) ? 1 : 0);
        sB += sdim == 0 ? 1 : 0;
      }
      unsigned long long tot;
      const unsigned long long pre =
          block_excl_scan<kPT>(((unsigned long long)sA << 32) | sB, S.sw, tot);
      unsigned int Ar = (unsigned int)(pre >> 32), Br = (unsigned int)(pre & 0xffffffffu);
      const int A_tot = (int)(tot >> 32), B_tot = (int)(tot & 0xffffffffu);
      if (tid == 0) { S.A_tot = A_tot; S.B_tot = B_tot; }
      for (int i = lo; i < hi; ++i) {
        const int s = S.slot_of[cur][i];
        if (s == kPNone) continue;
        const int k = i - S.seg_off[s];
        if (k == 0) { S.segA0[s] = (int)Ar; S.segB0[s] = (int)Br; }
        if (S.cont[s] && k >= S.j[s]) {
          const uint8_t f = flg[i];
          if ((f & 3) != kDisjoint && !(f & 4)) {
            const int sdim = (f >> 3) & 3;
            const Box b = lv[i];
            const double blo = sdim == 0 ? b.t0 : (sdim == 1 ? b.u0 : b.v0);
            const double bhi = sdim == 0 ? b.t1 : (sdim == 1 ? b.u1 : b.v1);
            const double mid = 0.5 * (blo + bhi);
            Box c0, c1;
            children(b, sdim, mid, c0, c1);
            const unsigned int push = Ar + Br;
            ar.ab[Ar] = c0;
            ar.key[Ar] = tkey(c0.t0);
            ar.push[Ar] = push;
            ar.cslot[Ar] = (uint8_t)s;
            ++Ar;
            if (sdim != 0) {
              if (f & 32) {
                ar.ab[Ar] = c1;
                ar.key[Ar] = tkey(c1.t0);
                ar.push[Ar] = push + 1;
                ar.cslot[Ar] = (uint8_t)s;
                ++Ar;
              }
            } else {
              const int ib = 2 * kPCap - 1 - (int)Br;
              ar.ab[ib] = c1;
              ar.key[ib] = tkey(c1.t0);
              ar.push[ib] = push + 1;
              ar.cslot[ib] = (uint8_t)s;
              ++Br;
            }
          }
        }
        if (k == S.seg_n[s] - 1) { S.segA1[s] = (int)Ar; S.segB1[s] = (int)Br; }
      }
    }
    __syncthreads();
    // ================= P5: next-level layout (slot order), eviction, deferral
    // A query whose level outgrew kPQCap goes to the block-per-query
    // engine (restart).  Otherwise the first K slots (rotating order) keep
    // their children, the rest are deferred: their current level is copied
    // forward and re-run next round.  Re-running a level is exact: its
    // first/drop record updates are idempotent and the check count is
    // rolled back.  K = the largest k with
    //   sum_{r<k} children_r + sum_{r>=k} boxes_r <= kPCap.
    if (tid < kPQ) {
      const int s = tid;
      int t = 0;
      if (S.cont[s]) {
        t = (S.segA1[s] - S.segA0[s]) + (S.segB1[s] - S.segB0[s]);
        if (t > kPQCap) {
          const unsigned long long h = atomicAdd(&a.ctr->heavy_count, 1ull);
          a.heavy_queue[h] = S.qidx[s];
          S.qidx[s] = -1;
          S.cont[s] = 0;
        }
      }
      S.tot[s] = t;
    }
    __syncthreads();
    if (tid < 32) {
      const int lane = tid;
      constexpr int kPer = kPQ / 32;
      int vt[kPer], vn[kPer];
      int st, sn, it, in, Nn, K;
      for (;;) {
        st = 0; sn = 0;
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
          const int s = (S.rot + lane * kPer + m) % kPQ;
          vt[m] = S.cont[s] ? S.tot[s] : 0;
          vn[m] = S.cont[s] ? S.seg_n[s] : 0;
          st += vt[m];
          sn += vn[m];
        }
        it = st; in = sn;  // inclusive warp scans of the per-lane sums
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
          if (vn[m] > 0 && pt + (Nn - pn) <= kPCap) bestk = lane * kPer + m + 1;
        }
        K = bestk;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) K = max(K, __shfl_xor_sync(0xffffffffu, K, o));
        if (K > 0 || Nn == 0) break;
        // no query can advance: evict the first continuing one (progress guarantee)
        const unsigned int has = __ballot_sync(0xffffffffu, sn > 0);
        const int l0 = __ffs(has) - 1;
        if (lane == l0) {
#pragma unroll
          for (int m = 0; m < kPer; ++m) {
            const int s = (S.rot + lane * kPer + m) % kPQ;
            if (vn[m] > 0) {
              const unsigned long long h = atomicAdd(&a.ctr->heavy_count, 1ull);
              a.heavy_queue[h] = S.qidx[s];
              S.qidx[s] = -1;
              S.cont[s] = 0;
              break;
            }
          }
        }
        __syncwarp();
      }
      // kept positions r < K take their children, the rest carry their level
      int cT = 0, cN = 0;
#pragma unroll
      for (int m = 0; m < kPer; ++m) {
        if (lane * kPer + m < K) { cT += vt[m]; cN += vn[m]; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cT += __shfl_xor_sync(0xffffffffu, cT, o);
        cN += __shfl_xor_sync(0xffffffffu, cN, o);
      }
      const int TK = cT, NK = cN;
      int ut = it - st, un = in - sn;
      int deferred = 0;
#pragma unroll
      for (int m = 0; m < kPer; ++m) {
        const int r = lane * kPer + m;
        const int s = (S.rot + r) % kPQ;
        if (S.cont[s]) {
          if (r < K) {
            S.next_off[s] = ut;
          } else {
            S.next_off[s] = TK + (un - NK);
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
        S.n_next = TK + (Nn - NK);
        S.rot = (S.rot + 1) % kPQ;
        S.deferred += deferred;
      }
    }
    __syncthreads();
    // B runs sorted?  (always true for dyadic t_max)
    {
      const int B_tot = S.B_tot;
      for (int b = tid + 1; b < B_tot; b += kPT) {
        const int ib = 2 * kPCap - 1 - b;
        const int s = ar.cslot[ib];
        if (S.cont[s] != 1 || b <= S.segB0[s]) continue;
        if (ar.key[ib + 1] > ar.key[ib]) S.unsorted[s] = 1;
      }
    }
    __syncthreads();
    // ================= P6: merge by rank into the next level
    {
      const int A_tot = S.A_tot, B_tot = S.B_tot;
      Box* out = ar.lvl[nxt];
      for (int e = tid; e < A_tot + B_tot; e += kPT) {
        const bool isA = e < A_tot;
        const int idx = isA ? e : 2 * kPCap - 1 - (e - A_tot);
        const int s = ar.cslot[idx];
        if (S.cont[s] != 1) continue;
        const unsigned long long kk = ar.key[idx];
        const unsigned int pp = ar.push[idx];
        int rank;
        if (!S.unsorted[s]) {
          if (isA) {
            int l = S.segB0[s], h = S.segB1[s];  // B elements < (kk, pp)
            while (l < h) {
              const int m = (l + h) >> 1;
              const int im = 2 * kPCap - 1 - m;
              if (kp_less(ar.key[im], ar.push[im], kk, pp)) l = m + 1;
              else h = m;
            }
            rank = (e - S.segA0[s]) + (l - S.segB0[s]);
          } else {
            int l = S.segA0[s], h = S.segA1[s];  // A elements < (kk, pp)
            while (l < h) {
              const int m = (l + h) >> 1;
              if (kp_less(ar.key[m], ar.push[m], kk, pp)) l = m + 1;
              else h = m;
            }
            rank = ((e - A_tot) - S.segB0[s]) + (l - S.segA0[s]);
          }
        } else {
          // exact rank count over the query's children (general t_max)
          rank = 0;
          for (int m = S.segA0[s]; m < S.segA1[s]; ++m)
            rank += kp_less(ar.key[m], ar.push[m], kk, pp) ? 1 : 0;
          for (int m = S.segB0[s]; m < S.segB1[s]; ++m) {
            const int im = 2 * kPCap - 1 - m;
            rank += kp_less(ar.key[im], ar.push[im], kk, pp) ? 1 : 0;
          }
        }
        const int pos = S.next_off[s] + rank;
        out[pos] = ar.ab[idx];
        S.slot_of[nxt][pos] = (uint8_t)s;
        S.flag[nxt][pos] = 0;
      }
      // deferred queries: carry the current level forward unchanged
      for (int i = tid; i < n; i += kPT) {
        const int s = S.slot_of[cur][i];
        if (s == kPNone || S.cont[s] != 2) continue;
        const int pos = S.next_off[s] + (i - S.seg_off[s]);
        out[pos] = lv[i];
        S.slot_of[nxt][pos] = (uint8_t)s;
        const uint8_t f = flg[i];
        S.flag[nxt][pos] = f;
        if ((f & 3) != kDisjoint) ar.wb[nxt][pos] = wbc[i];
      }
    }
    __syncthreads();
    // ================= P7: commit
    if (tid < kPQ && S.cont[tid]) {
      const int s = tid;
      if (S.cont[s] == 1) {
        S.seg_n[s] = S.tot[s];
        S.level[s] += 1;
      } else {
        S.C[s] -= S.seg_n[s];  // the level re-runs next round
      }
      S.seg_off[s] = S.next_off[s];
    }
    __syncthreads();
    if (tid == 0) S.n_cur = S.n_next;
    cur = nxt;
    __syncthreads();
  }
  if (tid == 0) {
    atomicAdd(&a.ctr->rounds, (unsigned long long)rounds);
    atomicAdd(&a.ctr->deferred, S.deferred);
  }
}

}  // namespace tccd
