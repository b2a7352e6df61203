__global__ void k1(const double* a, double* o) {
  double x = a[threadIdx.x], y = a[threadIdx.x + 32], r;
  asm("min.f64 %0, %1, %2;" : "=d"(r) : "d"(x), "d"(y));
  double s;
  asm("max.f64 %0, %1, %2;" : "=d"(s) : "d"(x), "d"(y));
  o[threadIdx.x] = r + s;
}
__global__ void k2(const double* a, double* o) {
  double x = a[threadIdx.x], y = a[threadIdx.x + 32];
  o[threadIdx.x] = fmin(x, y) + fmax(x, y);
}
__global__ void k3(const double* a, double* o) {
  double x = a[threadIdx.x], y = a[threadIdx.x + 32];
  o[threadIdx.x] = (x < y ? x : y) + (x > y ? x : y);
}
