// IRF baseline on the GPU: the reference's interval
// root finder ccdkit.baselines.irf_solve (pkg/src/ccdkit/baselines.py:123-206)
// for a batch of queries, bit-identical to it.
//
// The method is a best-first search: boxes wait in a min-heap keyed by
// (t_lo, level, push sequence) (:144, :202), every interval operation is
// widened one representable step outward (IntervalScalar, :37-106), and the
// first accepted box (F's enclosure contains 0 on every axis and every
// domain side < delta) or the first box popped once the budget is spent is
// the answer.  The pop order decides toi, witness and checks, so each query
// keeps a real binary heap: one thread per query (queries fetched
// dynamically), its heap an 8-ary heap in a global arena (see Heap).  A heap
// can hold at most checks + 1 boxes;
// queries whose heap outgrows the first pass's capacity are re-run from the
// root by a second pass with max_checks + 2 entries per slot (exact: the
// search is deterministic).
#include <cuda_runtime.h>

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
  unsigned long long next[2];  // next query of pass 1 / next overflow entry of pass 2
  unsigned long long overflow; // queries handed to pass 2
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
__device__ bool irf_query(const Args& a, long long q, Heap& H) {
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

// pass 0: every query (index list = identity); pass 1: the overflow list.
// Per thread: cap keys (16 B) then cap boxes (48 B), contiguous.
__global__ void __launch_bounds__(128) irf_kernel(Args a, Ctr* ctr, unsigned char* arena,
                                                  long long cap, const long long* list,
                                                  long long* overflow, int pass) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  Heap H;
  unsigned char* mine = arena + tid * cap * 64;
  H.key = (Key*)mine;
  H.box = (double2*)(mine + cap * 16);
  H.cap = cap;
  H.n = 0;
  const unsigned long long total = pass == 0 ? (unsigned long long)a.n : ctr->overflow;
  for (;;) {
    const unsigned long long i = atomicAdd(&ctr->next[pass], 1ull);
    if (i >= total) break;
    const long long q = pass == 0 ? (long long)i : list[i];
    if (!irf_query(a, q, H)) {
      if (pass == 0) overflow[atomicAdd(&ctr->overflow, 1ull)] = q;
      else a.status[q] = 0xFF;  // unreachable: a heap never exceeds checks + 1 <= cap - 1
    }
  }
}

}  // namespace tccd_irf

using namespace tccd_irf;

namespace {

constexpr long long kCap1 = 2048;  // heap entries per thread in pass 1
constexpr int kThreads = 128;

size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

struct IrfLayout {
  size_t ctr, overflow, arena1, arena2, total;
  long long threads1, slots2, cap2;
};

int resident_blocks() {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, irf_kernel, kThreads, 0) != cudaSuccess ||
      nb < 1)
    nb = 2;
  return nb;
}

// slots2 <= 0: as many second-pass threads as a quarter of the device
// memory holds (one per SM at least, 4096 at most)
IrfLayout irf_layout(long long n, long long mcmax, int slots2, int sms) {
  IrfLayout L;
  L.threads1 = (long long)sms * resident_blocks() * kThreads;
  L.cap2 = (mcmax > 0 ? mcmax : 0) + 2;
  long long s2 = slots2;
  if (s2 <= 0) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) tot = (size_t)16 << 30;
    s2 = (long long)(tot / 4 / ((size_t)L.cap2 * 64));
    if (s2 > 4096) s2 = 4096;
    if (s2 < sms) s2 = sms;
  }
  L.slots2 = (s2 + 31) / 32 * 32;
  size_t o = 0;
  L.ctr = o; o += a256(sizeof(Ctr));
  L.overflow = o; o += a256((size_t)(n > 0 ? n : 1) * 8);
  L.arena1 = o; o += a256((size_t)L.threads1 * kCap1 * 64);
  L.arena2 = o; o += a256((size_t)L.slots2 * L.cap2 * 64);
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
  if (cudaMemsetAsync(ctr, 0, sizeof(Ctr), st) != cudaSuccess) return TCCD_E_CUDA;
  irf_kernel<<<(unsigned)(L.threads1 / kThreads), kThreads, 0, st>>>(
      a, ctr, ws + L.arena1, kCap1, nullptr, ovf, 0);
  if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  // pass 2 (a no-op when nothing overflowed): max_checks + 2 entries per slot
  irf_kernel<<<(unsigned)(L.slots2 / 32), 32, 0, st>>>(a, ctr, ws + L.arena2, L.cap2, ovf, ovf,
                                                       1);
  if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  return TCCD_OK;
}

}  // extern "C"
