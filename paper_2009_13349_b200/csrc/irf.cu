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
// dynamically), its heap in a global arena laid out warp-interleaved (entry
// k of the 32 lanes of a warp is one contiguous 2 KB run, so the hot top of
// the heaps is read coalesced).  A heap can hold at most checks + 1 boxes;
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

// a heap of one lane: entry k at base + (k * 32) * 8 doubles (warp-interleaved)
struct Heap {
  double* base;  // this lane's entry 0
  long long cap, n;
  __device__ __forceinline__ double* at(long long k) const { return base + k * 256; }
  __device__ __forceinline__ bool less(long long i, double tl, long long lv, long long sq) const {
    const double* e = at(i);
    const double ti = e[0];
    if (ti != tl) return ti < tl;
    const long long li = __double_as_longlong(e[6]);
    if (li != lv) return li < lv;
    return __double_as_longlong(e[7]) < sq;
  }
  __device__ __forceinline__ void put(long long i, const double b[6], long long lv, long long sq) {
    double* e = at(i);
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = b[k];
    e[6] = __longlong_as_double(lv);
    e[7] = __longlong_as_double(sq);
  }
  __device__ __forceinline__ void move(long long dst, long long src) {
    double* d = at(dst);
    const double* s = at(src);
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k] = s[k];
  }
  __device__ void push(const double b[6], long long lv, long long sq) {
    long long i = n++;
    while (i > 0) {
      const long long p = (i - 1) >> 1;
      if (!less_key(b[0], lv, sq, p)) break;
      move(i, p);
      i = p;
    }
    put(i, b, lv, sq);
  }
  // (tl, lv, sq) < entry p ?
  __device__ __forceinline__ bool less_key(double tl, long long lv, long long sq, long long p) const {
    const double* e = at(p);
    const double tp = e[0];
    if (tl != tp) return tl < tp;
    const long long lp = __double_as_longlong(e[6]);
    if (lv != lp) return lv < lp;
    return sq < __double_as_longlong(e[7]);
  }
  __device__ void pop(double b[6], long long& lv) {
    const double* top = at(0);
#pragma unroll
    for (int k = 0; k < 6; ++k) b[k] = top[k];
    lv = __double_as_longlong(top[6]);
    --n;
    if (n == 0) return;
    double last[8];
    const double* le = at(n);
#pragma unroll
    for (int k = 0; k < 8; ++k) last[k] = le[k];
    const long long llv = __double_as_longlong(last[6]), lsq = __double_as_longlong(last[7]);
    long long i = 0;
    for (;;) {
      long long c = 2 * i + 1;
      if (c >= n) break;
      if (c + 1 < n) {
        const double* e1 = at(c + 1);
        if (less(c, e1[0], __double_as_longlong(e1[6]), __double_as_longlong(e1[7])) == false) ++c;
      }
      if (!less(c, last[0], llv, lsq)) break;
      move(i, c);
      i = c;
    }
    double* d = at(i);
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k] = last[k];
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
    H.push(root, 0, 0);
    long long seq = 0;
    while (H.n > 0) {
      double b[6];
      long long lv;
      H.pop(b, lv);
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
      if (!all) continue;
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
      const double m = 0.5 * (b[2 * dim] + b[2 * dim + 1]);
      double k0[6], k1[6];
      for (int k = 0; k < 6; ++k) { k0[k] = b[k]; k1[k] = b[k]; }
      k0[2 * dim + 1] = m;
      k1[2 * dim] = m;
      const bool keep0 = !(kind == 0 && k0[2] + k0[4] > 1.0);  // :197-199
      const bool keep1 = !(kind == 0 && k1[2] + k1[4] > 1.0);
      if (H.n + (keep0 ? 1 : 0) + (keep1 ? 1 : 0) > H.cap) return false;
      if (keep0) H.push(k0, lv + 1, ++seq);
      if (keep1) H.push(k1, lv + 1, ++seq);
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

// pass 0: every query (index list = identity); pass 1: the overflow list
__global__ void __launch_bounds__(128) irf_kernel(Args a, Ctr* ctr, double* arena, long long cap,
                                                  const long long* list, long long* overflow,
                                                  int pass) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  Heap H;
  H.base = arena + ((tid >> 5) * cap * 32 + lane) * 8;
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

constexpr long long kCap1 = 256;   // heap entries per thread in pass 1
constexpr int kThreads = 128;

size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

struct IrfLayout {
  size_t ctr, overflow, arena1, arena2, total;
  long long threads1, slots2, cap2;
};

IrfLayout irf_layout(long long n, long long mcmax, int slots2, int sms) {
  IrfLayout L;
  L.threads1 = (long long)sms * 8 * kThreads;  // 8 blocks of 128 per SM
  L.slots2 = ((long long)(slots2 > 0 ? slots2 : sms) + 31) / 32 * 32;
  L.cap2 = (mcmax > 0 ? mcmax : 0) + 2;
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
      a, ctr, (double*)(ws + L.arena1), kCap1, nullptr, ovf, 0);
  if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  // pass 2 (a no-op when nothing overflowed): max_checks + 2 entries per slot
  irf_kernel<<<(unsigned)(L.slots2 / 32), 32, 0, st>>>(a, ctr, (double*)(ws + L.arena2), L.cap2,
                                                       ovf, ovf, 1);
  if (cudaGetLastError() != cudaSuccess) return TCCD_E_CUDA;
  return TCCD_OK;
}

}  // extern "C"
