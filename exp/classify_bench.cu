// Experiment: standalone throughput of tccd::classify (no engine bookkeeping).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2009_13349_b200/csrc/tccd_device.cuh"
using namespace tccd;

__global__ void bench(const double* pts, int nq, int iters, int mixed, unsigned long long* out, int tame) {
  __shared__ double P[64][24];
  for (int i = threadIdx.x; i < 64 * 24; i += blockDim.x) P[i / 24][i % 24] = pts[(i / 24) % nq * 24 + i % 24];
  __syncthreads();
  const double eps[3] = {6.7e-15, 6.7e-15, 6.7e-15};
  unsigned long long acc = 0;
  const int q = (threadIdx.x + blockIdx.x) & 63;
  const int kind = mixed ? (threadIdx.x & 1) : ((blockIdx.x / 4) & 1);
  for (int it = 0; it < iters; ++it) {
    const double a = ((threadIdx.x * 37 + it * 11) & 1023) / 1024.0, w = 1.0 / 64;
    Box b{a * 0.9, a * 0.9 + w, a * 0.5, a * 0.5 + w, a * 0.25, a * 0.25 + w};
    double wb;
    const int c = classify((const double*)P[q], kind, b, eps, 0.0, wb, tame != 0);
    acc += c + (wb > 0.5);
  }
  if (acc == 123456789ull) out[0] = acc;
}

int main() {
  const int nq = 64;
  double h[nq * 24];
  for (int i = 0; i < nq * 24; ++i) h[i] = ((i * 7919) % 1000) / 1000.0 - (i % 24 >= 12 ? 0.3 : 0.0);
  double* d; unsigned long long* o;
  cudaMalloc(&d, sizeof h); cudaMalloc(&o, 8);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int tame = 0; tame < 2; ++tame) for (int mixed = 0; mixed < 1; ++mixed)
    for (int wps : {20, 32}) {
      const int tpb = 128, blocks = sms * wps / 4, iters = 2000;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      bench<<<blocks, tpb>>>(d, nq, 10, mixed, o, tame);
      cudaEventRecord(e0);
      bench<<<blocks, tpb>>>(d, nq, iters, mixed, o, tame);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double boxes = (double)blocks * tpb * iters;
      printf("tame=%d warps/SM=%d mixed=%d tpb=%d blocks=%d: %.3e boxes/s (%.2f ms)\n", tame, wps, mixed, tpb, blocks, boxes / (ms * 1e-3), ms);
    }
  return 0;
}
