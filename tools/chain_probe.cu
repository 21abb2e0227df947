// Cycles per element of the sequential squared-norm chain on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const double* g, double* out, long long* cyc, int mode, int n) {
  __shared__ double buf[32 * 66];  // 32 leaves x 64 doubles, padded
  for (int i = threadIdx.x; i < 32 * 66; i += blockDim.x) buf[i] = g[i] ;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const double* p = buf + threadIdx.x * 66;
  double acc = 0.0; unsigned long long bits = 0;
  long long t0 = clock64();
  for (int rep = 0; rep < n / 64; ++rep) {
    if (mode == 0) {
#pragma unroll 16
      for (int e = 0; e < 64; ++e) { double x = p[e]; acc = __dadd_rn(acc, __dmul_rn(x, x)); }
    } else if (mode == 1) {
#pragma unroll 16
      for (int e = 0; e < 64; ++e) { double x = p[e]; bits |= __double_as_longlong(x); acc = __dadd_rn(acc, __dmul_rn(x, x)); }
    } else {
#pragma unroll 16
      for (int e = 0; e < 64; ++e) { double x = p[e]; acc = __dadd_rn(acc, x); }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc + (double)bits;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double *g, *o; long long* c; cudaMallocManaged(&g, 8 * 32 * 66); cudaMallocManaged(&o, 8 * 32); cudaMallocManaged(&c, 8);
  for (int i = 0; i < 32 * 66; ++i) g[i] = 1.0 + 1e-3 * i;
  const int n = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    chain<<<1, 64>>>(g, o, c, mode, n); cudaDeviceSynchronize();
    chain<<<1, 64>>>(g, o, c, mode, n); cudaDeviceSynchronize();
    printf("mode %d: %.2f cycles/element\n", mode, (double)*c / n);
  }
  return 0;
}
