// Device-side numerics of the inclusion-based CCD root finder.
//
// Every function here reproduces the reference's binary64 operation order
// exactly (the filter constants were derived for it: pkg/src/ccdkit/core.py:
// 19-23, inclusion.py:8-15).  The translation unit is compiled with
// --fmad=false so no multiply/add pair is contracted into a DFMA; common
// subexpressions are shared only where the shared value is bit-identical to
// what the reference recomputes (same operands, same single operation).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tccd {

// Bounds checks of a diagnostic build (-DTCCD_CHECKS): a violated index
// traps the kernel (the launch fails with an error) instead of corrupting
// memory.  Compiled out otherwise.
#ifdef TCCD_CHECKS
#define TCCD_ASSERT(c) \
  do {                 \
    if (!(c)) __trap(); \
  } while (0)
#else
#define TCCD_ASSERT(c) \
  do {                 \
  } while (0)
#endif
constexpr int kDisjoint = 0;    // _kernel.py:36
constexpr int kIntersects = 1;  // _kernel.py:37
constexpr int kContained = 2;   // _kernel.py:38

// per-query status (include/tccd.h)
constexpr uint8_t kFree = 0, kHit = 1, kErrSeparation = 2, kErrNonfinite = 3, kErrParam = 4;

// inclusion.py:35-38
constexpr double kCoefVF = 6.661338147750939e-15;
constexpr double kCoefEE = 6.217248937900877e-15;
constexpr double kCoefVFd = 7.549516567451064e-15;
constexpr double kCoefEEd = 7.105427357601002e-15;

struct alignas(16) Box {
  double t0, t1, u0, u1, v0, v1;
};

// Per-query constants every box check needs.  Points are point-major:
// P[3*k + ax] is point k at t0 (k = 0..3), P[12 + 3*k + ax] at t1.
struct QueryParams {
  double eps[3];
  double kap[3];
  double sep, delta, t_max;
  long long max_checks;
  int kind;
  int tame;  // all |coordinates| < 1e300: every corner value is finite
};

// F on one axis at the 4 (u, v) corners for one time value; the lerped
// point coordinates a..d are (1 - t) * s + t * e (core.py:221-222).
// VF: p - (((1 - u) - v) * v1 + u * v2 + v * v3)        (core.py:236)
// EE: ((1 - u) * p1 + u * p2) - ((1 - v) * p3 + v * p4)  (core.py:254)
struct CornerWeights {
  double u0, u1, v0, v1;
  double omu0, omu1, omv0, omv1;  // 1 - u, 1 - v
  double w00, w01, w10, w11;      // (1 - u) - v   (VF only)
};

__device__ __forceinline__ CornerWeights corner_weights(const Box& b) {
  CornerWeights w;
  w.u0 = b.u0; w.u1 = b.u1; w.v0 = b.v0; w.v1 = b.v1;
  w.omu0 = 1.0 - b.u0; w.omu1 = 1.0 - b.u1;
  w.omv0 = 1.0 - b.v0; w.omv1 = 1.0 - b.v1;
  w.w00 = w.omu0 - b.v0; w.w01 = w.omu0 - b.v1;
  w.w10 = w.omu1 - b.v0; w.w11 = w.omu1 - b.v1;
  return w;
}

// compare-exchange: one comparison gives both the min and the max (exact for
// non-NaN operands; +-0 order never changes a classification or a width)
__device__ __forceinline__ void cmpx(double a, double b, double& lo, double& hi) {
  const bool p = a < b;
  lo = p ? a : b;
  hi = p ? b : a;
}

template <int KIND>
__device__ __forceinline__ void corners4(double a, double b, double c, double d,
                                         const CornerWeights& w, double& f00, double& f01,
                                         double& f10, double& f11) {
  if (KIND == 0) {
    const double cu0 = w.u0 * c, cu1 = w.u1 * c, dv0 = w.v0 * d, dv1 = w.v1 * d;
    f00 = a - ((w.w00 * b + cu0) + dv0);
    f01 = a - ((w.w01 * b + cu0) + dv1);
    f10 = a - ((w.w10 * b + cu1) + dv0);
    f11 = a - ((w.w11 * b + cu1) + dv1);
  } else {
    const double l0 = w.omu0 * a + w.u0 * b, l1 = w.omu1 * a + w.u1 * b;
    const double r0 = w.omv0 * c + w.v0 * d, r1 = w.omv1 * c + w.v1 * d;
    f00 = l0 - r0; f01 = l0 - r1; f10 = l1 - r0; f11 = l1 - r1;
  }
}

// _kernel._hull_axis (_kernel.py:44-67) for one axis.  TAME (all corner
// values finite): compare-exchange tournament, 10 comparisons for min and max
// of 8 values.  Otherwise fmin/fmax from +-inf, which ignore NaN exactly like
// the reference's `val < mn` / `val > mx` updates.
template <int KIND, bool TAME, typename PtrT>
__device__ __forceinline__ void hull_axis(PtrT P, int ax, double t0, double omt0, double t1,
                                          double omt1, const CornerWeights& w, double& mn,
                                          double& mx) {
  const double s0 = P[ax], s1 = P[3 + ax], s2 = P[6 + ax], s3 = P[9 + ax];
  const double e0 = P[12 + ax], e1 = P[15 + ax], e2 = P[18 + ax], e3 = P[21 + ax];
  double f[8];
  corners4<KIND>(omt0 * s0 + t0 * e0, omt0 * s1 + t0 * e1, omt0 * s2 + t0 * e2,
                 omt0 * s3 + t0 * e3, w, f[0], f[1], f[2], f[3]);
  corners4<KIND>(omt1 * s0 + t1 * e0, omt1 * s1 + t1 * e1, omt1 * s2 + t1 * e2,
                 omt1 * s3 + t1 * e3, w, f[4], f[5], f[6], f[7]);
  if (TAME) {
    double l0, h0, l1, h1, l2, h2, l3, h3;
    cmpx(f[0], f[1], l0, h0);
    cmpx(f[2], f[3], l1, h1);
    cmpx(f[4], f[5], l2, h2);
    cmpx(f[6], f[7], l3, h3);
    const double la = l0 < l1 ? l0 : l1, lb = l2 < l3 ? l2 : l3;
    const double ha = h0 > h1 ? h0 : h1, hb = h2 > h3 ? h2 : h3;
    mn = la < lb ? la : lb;
    mx = ha > hb ? ha : hb;
  } else {
    mn = __longlong_as_double(0x7ff0000000000000LL);              // +inf
    mx = __longlong_as_double((long long)0xfff0000000000000ULL);  // -inf
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      mn = fmin(mn, f[k]);
      mx = fmax(mx, f[k]);
    }
  }
}

// _kernel._classify (_kernel.py:71-94): axes x, y, z with an early return
// at the first separated axis; hull enlarged by sep before comparing; wb is
// the raw (unenlarged) max width, 0 when disjoint.
template <int KIND, bool TAME, typename PtrT>
__device__ __forceinline__ int classify_k(PtrT P, const Box& b, const double* eps, double sep,
                                          double& wb) {
  const CornerWeights w = corner_weights(b);
  const double omt0 = 1.0 - b.t0, omt1 = 1.0 - b.t1;
  bool contained = true;
  double width = 0.0;
#ifdef TCCD_UNROLL_AXES
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int ax = 0; ax < 3; ++ax) {
    double mn, mx;
    hull_axis<KIND, TAME>(P, ax, b.t0, omt0, b.t1, omt1, w, mn, mx);
    const double e = eps[ax];
    const double lo = mn - sep, hi = mx + sep;
    if (lo > e || hi < -e) {
      wb = 0.0;
      return kDisjoint;
    }
    if (!(lo >= -e && hi <= e)) contained = false;
    const double d = mx - mn;
    if (d > width) width = d;
  }
  wb = width;
  return contained ? kContained : kIntersects;
}

// The same classification with all three axes evaluated (tame coordinates):
// the reference returns at the first separated axis, but the class and wb it
// returns do not depend on which axis that was (DISJOINT, wb = 0), and for a
// non-disjoint box it has evaluated all three.  A warp pays for the three
// axes as soon as one lane's box is not separated on the first, so the
// branch-free form costs the warp no flops and lets the three hulls
// interleave.  EpsT indexes like an array (pointer or strided accessor).
template <int KIND, typename PtrT, typename EpsT>
__device__ __forceinline__ int classify_full(PtrT P, const Box& b, EpsT eps, double sep,
                                             double& wb) {
  const CornerWeights w = corner_weights(b);
  const double omt0 = 1.0 - b.t0, omt1 = 1.0 - b.t1;
  bool disjoint = false, contained = true;
  double width = 0.0;
#ifdef TCCD_FULL_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int ax = 0; ax < 3; ++ax) {
    double mn, mx;
    hull_axis<KIND, true>(P, ax, b.t0, omt0, b.t1, omt1, w, mn, mx);
    const double e = eps[ax];
    const double lo = mn - sep, hi = mx + sep;
    disjoint |= lo > e || hi < -e;
    contained &= lo >= -e && hi <= e;
    const double d = mx - mn;
    width = d > width ? d : width;
  }
  wb = disjoint ? 0.0 : width;
  return disjoint ? kDisjoint : (contained ? kContained : kIntersects);
}

// classify_full of two boxes at once (the two children of a refined box):
// two independent evaluations a thread interleaves axis by axis (the lane
// tier classifies children when their parent is refined).  Each box sees
// exactly classify_full's operations.
// (SEP0: the whole call has separation 0 -- the hull is compared as is: x -
// 0 and x + 0 change no comparison.)
template <int KIND, bool SEP0, typename PtrT, typename EpsT>
__device__ __forceinline__ void classify_pair(PtrT P, const Box& a, const Box& b, EpsT eps,
                                              double sep, int& cls_a, double& wb_a, int& cls_b,
                                              double& wb_b) {
#ifdef TCCD_PAIR_HOIST
  const CornerWeights wa = corner_weights(a), wb = corner_weights(b);
  const double a_omt0 = 1.0 - a.t0, a_omt1 = 1.0 - a.t1;
  const double b_omt0 = 1.0 - b.t0, b_omt1 = 1.0 - b.t1;
#endif
  bool dis_a = false, con_a = true, dis_b = false, con_b = true;
  double wid_a = 0.0, wid_b = 0.0;
#ifdef TCCD_FULL_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int ax = 0; ax < 3; ++ax) {
    double mna, mxa, mnb, mxb;
#ifndef TCCD_PAIR_HOIST
    // the corner weights are recomputed per axis (10 DADD per box) instead
    // of held in 2 x 14 double registers across the axis loop: the boxes
    // are made opaque to the compiler's loop-invariant hoisting
    Box a2 = a, b2 = b;
    asm volatile("" : "+d"(a2.t0), "+d"(a2.t1), "+d"(a2.u0), "+d"(a2.u1), "+d"(a2.v0), "+d"(a2.v1));
    asm volatile("" : "+d"(b2.t0), "+d"(b2.t1), "+d"(b2.u0), "+d"(b2.u1), "+d"(b2.v0), "+d"(b2.v1));
    {
      const CornerWeights wa = corner_weights(a2);
      hull_axis<KIND, true>(P, ax, a2.t0, 1.0 - a2.t0, a2.t1, 1.0 - a2.t1, wa, mna, mxa);
    }
    {
      const CornerWeights wb = corner_weights(b2);
      hull_axis<KIND, true>(P, ax, b2.t0, 1.0 - b2.t0, b2.t1, 1.0 - b2.t1, wb, mnb, mxb);
    }
#else
    hull_axis<KIND, true>(P, ax, a.t0, a_omt0, a.t1, a_omt1, wa, mna, mxa);
    hull_axis<KIND, true>(P, ax, b.t0, b_omt0, b.t1, b_omt1, wb, mnb, mxb);
#endif
    const double e = eps[ax];
    const double loa = SEP0 ? mna : mna - sep, hia = SEP0 ? mxa : mxa + sep;
    const double lob = SEP0 ? mnb : mnb - sep, hib = SEP0 ? mxb : mxb + sep;
    dis_a |= loa > e || hia < -e;
    dis_b |= lob > e || hib < -e;
    con_a &= loa >= -e && hia <= e;
    con_b &= lob >= -e && hib <= e;
    const double da = mxa - mna, db = mxb - mnb;
    wid_a = da > wid_a ? da : wid_a;
    wid_b = db > wid_b ? db : wid_b;
  }
  wb_a = dis_a ? 0.0 : wid_a;
  wb_b = dis_b ? 0.0 : wid_b;
  cls_a = dis_a ? kDisjoint : (con_a ? kContained : kIntersects);
  cls_b = dis_b ? kDisjoint : (con_b ? kContained : kIntersects);
}

template <typename PtrT>
__device__ __forceinline__ int classify(PtrT P, int kind, const Box& b, const double* eps,
                                        double sep, double& wb, bool tame = false) {
  if (tame) return kind == 0 ? classify_k<0, true>(P, b, eps, sep, wb)
                             : classify_k<1, true>(P, b, eps, sep, wb);
  return kind == 0 ? classify_k<0, false>(P, b, eps, sep, wb)
                   : classify_k<1, false>(P, b, eps, sep, wb);
}

// all |coordinates| < 1e300 (and finite): lerps and corner values stay
// below 8e300, so no comparison in the hull ever sees a NaN
template <typename PtrT>
__device__ __forceinline__ int tame_coords(PtrT P) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 24; ++i) ok &= fabs(P[i]) < 1e300;
  return ok ? 1 : 0;
}

// F at the 8 corners of the domain [0, t_max] x [0,1]^2, corner index
// 4 t + 2 u + v: the values _kernel._kappas differences (_kernel.py:98-132)
// and, bit for bit, the 8 corner values _hull_axis takes of the root box
// (the same operations: a lerp with t in {0, t_max}, then (1 - u) - v with
// u, v in {0, 1}).
template <typename PtrT>
__device__ __forceinline__ void root_corners(PtrT P, int kind, double t_max, double F[8][3]) {
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double t = it ? t_max : 0.0;
    const double omt = 1.0 - t;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double a = omt * P[ax] + t * P[12 + ax];
      const double b = omt * P[3 + ax] + t * P[15 + ax];
      const double c = omt * P[6 + ax] + t * P[18 + ax];
      const double d = omt * P[9 + ax] + t * P[21 + ax];
#pragma unroll
      for (int iu = 0; iu < 2; ++iu)
#pragma unroll
        for (int iv = 0; iv < 2; ++iv) {
          const double u = iu ? 1.0 : 0.0, v = iv ? 1.0 : 0.0;
          double val;
          if (kind == 0) val = a - ((1.0 - u - v) * b + u * c + v * d);
          else val = ((1.0 - u) * a + u * b) - ((1.0 - v) * c + v * d);
          F[4 * it + 2 * iu + iv][ax] = val;
        }
    }
  }
}

// kappas from the domain's corner values (strides t=4, u=2, v=1)
__device__ __forceinline__ void kappas_from(const double F[8][3], double out[3]) {
  const int strides[3] = {4, 2, 1};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double best = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i & strides[k]) continue;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const double d = fabs(F[i + strides[k]][ax] - F[i][ax]);
        if (d > best) best = d;
      }
    }
    out[k] = 3.0 * best;
  }
}

// _kernel._classify of the root box from its corner values: the same
// comparisons as classify_k (the hull ignores NaN like the reference's
// `val < mn` / `val > mx` updates)
__device__ __forceinline__ int classify_root(const double F[8][3], const double* eps, double sep,
                                             double& wb) {
  bool contained = true;
  double width = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    double mn = __longlong_as_double(0x7ff0000000000000LL);
    double mx = __longlong_as_double((long long)0xfff0000000000000ULL);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      mn = fmin(mn, F[k][ax]);
      mx = fmax(mx, F[k][ax]);
    }
    const double e = eps[ax];
    const double lo = mn - sep, hi = mx + sep;
    if (lo > e || hi < -e) {
      wb = 0.0;
      return kDisjoint;
    }
    if (!(lo >= -e && hi <= e)) contained = false;
    const double d = mx - mn;
    if (d > width) width = d;
  }
  wb = width;
  return contained ? kContained : kIntersects;
}

// _kernel._kappas (_kernel.py:98-132): 3 * max |F(corner + stride) - F(corner)|
// over the domain [0, t_max] x [0,1]^2, strides t=4, u=2, v=1.
template <typename PtrT>
__device__ __forceinline__ void kappas(PtrT P, int kind, double t_max, double out[3]) {
  double F[8][3];
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double t = it ? t_max : 0.0;
    const double omt = 1.0 - t;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double a = omt * P[ax] + t * P[12 + ax];
      const double b = omt * P[3 + ax] + t * P[15 + ax];
      const double c = omt * P[6 + ax] + t * P[18 + ax];
      const double d = omt * P[9 + ax] + t * P[21 + ax];
#pragma unroll
      for (int iu = 0; iu < 2; ++iu)
#pragma unroll
        for (int iv = 0; iv < 2; ++iv) {
          const double u = iu ? 1.0 : 0.0, v = iv ? 1.0 : 0.0;
          double val;
          if (kind == 0) val = a - ((1.0 - u - v) * b + u * c + v * d);
          else val = ((1.0 - u) * a + u * b) - ((1.0 - v) * c + v * d);
          F[4 * it + 2 * iu + iv][ax] = val;
        }
    }
  }
  const int strides[3] = {4, 2, 1};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double best = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i & strides[k]) continue;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const double d = fabs(F[i + strides[k]][ax] - F[i][ax]);
        if (d > best) best = d;
      }
    }
    out[k] = 3.0 * best;
  }
}

// compute_gamma + compute_filters (inclusion.py:85-122).  Returns kHit on
// success, else the per-query error status.
template <typename PtrT>
__device__ __forceinline__ uint8_t filters(PtrT P, int kind, double sep, double eps[3]) {
  double g[3] = {0.0, 0.0, 0.0};
  bool finite = true;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double x = P[3 * i + ax];
      finite &= isfinite(x);
      g[ax] = fmax(g[ax], fabs(x));
    }
  if (!finite) return kErrNonfinite;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) g[ax] = g[ax] > 1.0 ? g[ax] : 1.0;
  double c;
  if (sep > 0.0) {
    if (!(sep < g[0] && sep < g[1] && sep < g[2])) return kErrSeparation;
    c = kind == 0 ? kCoefVFd : kCoefEEd;
  } else {
    c = kind == 0 ? kCoefVF : kCoefEE;
  }
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) eps[ax] = c * (g[ax] * g[ax] * g[ax]);
  return kHit;
}

__device__ __forceinline__ bool params_valid(int kind, double delta, long long mc, double sep,
                                             double t_max) {
  return (kind == 0 || kind == 1) && delta > 0.0 && isfinite(delta) && mc >= 1 && sep >= 0.0 &&
         isfinite(sep) && t_max > 0.0 && t_max <= 1.0;
}

// Split decision for a non-disjoint box (_kernel.py:215-241): returns the
// final accept flag; on refine, sdim/mid/push_hi describe the children
// (_kernel.py:259-310: VF clips only the upper child of a u or v split).
__device__ __forceinline__ bool split_decision(const Box& b, int cls, double wb,
                                               const double* kap, double delta, int kind,
                                               int& sdim, double& mid, bool& push_hi) {
  bool accept = wb < delta || cls == kContained;
  sdim = 0;
  mid = 0.0;
  push_hi = true;
  if (!accept) {
    const double ct = (b.t1 - b.t0) * kap[0];
    const double cu = (b.u1 - b.u0) * kap[1];
    const double cv = (b.v1 - b.v0) * kap[2];
    double best = ct;
    if (cu > best) { sdim = 1; best = cu; }
    if (cv > best) { sdim = 2; best = cv; }
    const double lo = sdim == 0 ? b.t0 : (sdim == 1 ? b.u0 : b.v0);
    const double hi = sdim == 0 ? b.t1 : (sdim == 1 ? b.u1 : b.v1);
    mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) accept = true;  // float resolution (_kernel.py:230-241)
    if (kind == 0) {
      if (sdim == 1) push_hi = mid + b.v0 <= 1.0;
      else if (sdim == 2) push_hi = b.u0 + mid <= 1.0;
    }
  }
  return accept;
}

__device__ __forceinline__ void children(const Box& b, int sdim, double mid, Box& lo, Box& hi) {
  lo = b;
  hi = b;
  if (sdim == 0) { lo.t1 = mid; hi.t0 = mid; }
  else if (sdim == 1) { lo.u1 = mid; hi.u0 = mid; }
  else { lo.v1 = mid; hi.v0 = mid; }
}

// Ordering key of a box inside a level: t_lo >= 0 is never -0 (domain
// bounds are built from 0, t_max and midpoints), so its IEEE bit pattern
// orders like the value.
__device__ __forceinline__ unsigned long long tkey(double t) {
  return (unsigned long long)__double_as_longlong(t);
}

}  // namespace tccd
