// Cycles per element of the K1 chain-warp inner loop (data in smem, no barriers).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain2(double* out, long long* cyc, int chunks, int mode) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x;
  for (int i = lane; i < 32 * 528 / 8; i += 32) ((double*)sm)[i] = 1.0 + i * 1e-7;
  __syncwarp();
  const unsigned char* pp = sm + lane * 528;
  double acc = 0.0, acc2 = 0.0;
  long long t0 = clock64();
  for (int c = 0; c < chunks; ++c) {
    for (int v = 0; v < 32; v += 8) {
      uint4 w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) w[u] = *reinterpret_cast<const uint4*>(pp + 16 * (v + u));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double* q2 = reinterpret_cast<const double*>(&w[u]);
        if (mode == 0) { acc = __dadd_rn(acc, q2[0]); acc = __dadd_rn(acc, q2[1]); }
        else { acc = __dadd_rn(acc, q2[0]); acc2 = __dadd_rn(acc2, q2[1]); }
      }
    }
  }
  long long t1 = clock64();
  out[lane] = acc + acc2;
  if (lane == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMallocManaged(&o, 8 * 32); cudaMallocManaged(&c, 8);
  for (int mode = 0; mode < 2; ++mode) {
    chain2<<<1, 32, 32 * 528>>>(o, c, 64, mode); cudaDeviceSynchronize();
    chain2<<<1, 32, 32 * 528>>>(o, c, 64, mode); cudaDeviceSynchronize();
    printf("mode %d: %.2f cycles/element (%s)\n", mode, (double)*c / (64 * 64), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
