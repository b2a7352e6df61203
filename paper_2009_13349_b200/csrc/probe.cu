// FP64 peak probes for the roofline denominator (MEASURED_PEAKS.json has no
// FP64 entry).  Not part of the solver: bench.py loads libtccd_probe.so to
// measure, on the box it runs on, the DFMA rate (FMA-counted peak, 2 flops
// per DFMA) and the DADD rate (the ceiling for an FMA-free kernel).
#include <cuda_runtime.h>

namespace {

constexpr int kChains = 8;

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dadd_loop(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __dadd_rn(x[c], a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s + b;
}

double run(bool fma_mode, int iters, int reps) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 512, blocks = sms * 4;
  double* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps + 1; ++r) {
    cudaEventRecord(e0);
    if (fma_mode) dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    else dadd_loop<<<blocks, threads>>>(out, iters, 1e-7, 0.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;  // first run is warm-up
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  const double ops = (double)blocks * threads * iters * kChains * (fma_mode ? 2.0 : 1.0);
  return ops / (best * 1e-3) / 1e12;
}

}  // namespace

extern "C" {
// TFLOP/s of DFMA (2 flops each) and of DADD (1 flop each), device 0 / current.
double tccd_probe_dfma_tflops(int iters, int reps) { return run(true, iters, reps); }
double tccd_probe_dadd_tflops(int iters, int reps) { return run(false, iters, reps); }
}
