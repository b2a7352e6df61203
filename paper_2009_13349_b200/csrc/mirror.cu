// The reference's spec-level inclusion functions as batched device kernels,
// evaluated with the solver's own device numerics (tccd_device.cuh):
//
//   tccd_box_hulls <- ccdkit.inclusion.box_inclusion (pkg/src/ccdkit/
//                     inclusion.py:131-156): per query, the min / max of each
//                     axis of F over the 8 corners of a box
//   tccd_kappas    <- ccdkit.inclusion.kappas (inclusion.py:195-217) /
//                     ccdkit._kernel._kappas (_kernel.py:98-132)
//
// They exist so that a ccdkit caller finds these entry points (and so that
// the reference's own inclusion tests can be re-run against the device
// arithmetic); the solver does not call them.
#include <cuda_runtime.h>

#include <cstdint>

#include "tccd.h"
#include "tccd_device.cuh"

namespace tccd_mirror {
using namespace tccd;

// numpy's min / max: NaN as soon as one operand is NaN
__device__ __forceinline__ double nmin(double a, double b) { return (a != a || b != b) ? a + b : (a < b ? a : b); }
__device__ __forceinline__ double nmax(double a, double b) { return (a != a || b != b) ? a + b : (a > b ? a : b); }

template <int KIND>
__device__ void hulls(const double* P, const Box& b, double* lo, double* hi) {
  const CornerWeights w = corner_weights(b);
  const double omt0 = 1.0 - b.t0, omt1 = 1.0 - b.t1;
  for (int ax = 0; ax < 3; ++ax) {
    const double s0 = P[ax], s1 = P[3 + ax], s2 = P[6 + ax], s3 = P[9 + ax];
    const double e0 = P[12 + ax], e1 = P[15 + ax], e2 = P[18 + ax], e3 = P[21 + ax];
    double f[8];
    corners4<KIND>(omt0 * s0 + b.t0 * e0, omt0 * s1 + b.t0 * e1, omt0 * s2 + b.t0 * e2,
                   omt0 * s3 + b.t0 * e3, w, f[0], f[1], f[2], f[3]);
    corners4<KIND>(omt1 * s0 + b.t1 * e0, omt1 * s1 + b.t1 * e1, omt1 * s2 + b.t1 * e2,
                   omt1 * s3 + b.t1 * e3, w, f[4], f[5], f[6], f[7]);
    double mn = f[0], mx = f[0];
    for (int k = 1; k < 8; ++k) {
      mn = nmin(mn, f[k]);
      mx = nmax(mx, f[k]);
    }
    lo[ax] = mn;
    hi[ax] = mx;
  }
}

__global__ void hulls_kernel(const double* points, const uint8_t* kind, int kind_all,
                             const double* boxes, long long n, double* lo, double* hi) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* bx = boxes + 6 * i;
  const Box b = {bx[0], bx[1], bx[2], bx[3], bx[4], bx[5]};
  const int k = kind ? kind[i] : kind_all;
  if (k == 0) hulls<0>(points + 24 * i, b, lo + 3 * i, hi + 3 * i);
  else hulls<1>(points + 24 * i, b, lo + 3 * i, hi + 3 * i);
}

__global__ void kappas_kernel(const double* points, const uint8_t* kind, int kind_all,
                              const double* t_max, double t_max_all, long long n, double* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  kappas(points + 24 * i, kind ? kind[i] : kind_all, t_max ? t_max[i] : t_max_all, out + 3 * i);
}

}  // namespace tccd_mirror

extern "C" {

int tccd_box_hulls(const double* points, const uint8_t* kind, int kind_all, const double* boxes,
                   int64_t n, double* lo, double* hi, void* stream) {
  if (n < 0) return TCCD_E_N;
  if (n == 0) return TCCD_OK;
  if (!points || !boxes || !lo || !hi) return TCCD_E_NULL;
  if (!kind && kind_all != 0 && kind_all != 1) return TCCD_E_KIND;
  tccd_mirror::hulls_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      points, kind, kind_all, boxes, (long long)n, lo, hi);
  return cudaGetLastError() == cudaSuccess ? TCCD_OK : TCCD_E_CUDA;
}

int tccd_kappas(const double* points, const uint8_t* kind, int kind_all, const double* t_max,
                double t_max_all, int64_t n, double* out, void* stream) {
  if (n < 0) return TCCD_E_N;
  if (n == 0) return TCCD_OK;
  if (!points || !out) return TCCD_E_NULL;
  if (!kind && kind_all != 0 && kind_all != 1) return TCCD_E_KIND;
  tccd_mirror::kappas_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      points, kind, kind_all, t_max, t_max_all, (long long)n, out);
  return cudaGetLastError() == cudaSuccess ? TCCD_OK : TCCD_E_CUDA;
}

}  // extern "C"
