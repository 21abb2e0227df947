// Dependent-load latency probe (pointer chase) for L1 / L2 / HBM footprints,
// plus atomic round trips, from one thread.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__global__ void chase(const unsigned *next, int hops, unsigned long long *out, unsigned *sink) {
  unsigned p = 0;
  for (int i = 0; i < 64; ++i) p = next[p];  // warm
  const long long c0 = clock64();
  const unsigned long long t0 = gt();
  for (int i = 0; i < hops; ++i) p = __ldcg(next + p);
  const long long c1 = clock64();
  out[0] = gt() - t0;
  out[1] = c1 - c0;
  *sink = p;
}
__global__ void chase_l1(const unsigned *next, int hops, unsigned long long *out, unsigned *sink) {
  unsigned p = 0;
  for (int i = 0; i < 2048; ++i) p = next[p];
  const long long c0 = clock64();
  for (int i = 0; i < hops; ++i) p = next[p];
  out[1] = clock64() - c0;
  *sink = p;
}
__global__ void atom_rt(unsigned *ctr, int n, unsigned long long *out) {
  unsigned v = 0;
  const long long c0 = clock64();
  for (int i = 0; i < n; ++i) v = atomicAdd(ctr + (v & 0), 1u);
  out[1] = clock64() - c0;
  out[2] = v;
}

int main() {
  unsigned long long *out, h[3];
  unsigned *sink;
  cudaMalloc(&out, 64);
  cudaMalloc(&sink, 4);
  for (size_t bytes : {size_t(16) << 10, size_t(1) << 20, size_t(16) << 20, size_t(64) << 20, size_t(1) << 30}) {
    size_t n = bytes / 128;  // one element per 128B line
    std::vector<unsigned> perm(n);
    for (size_t i = 0; i < n; ++i) perm[i] = (unsigned)i;
    std::shuffle(perm.begin() + 1, perm.end(), std::mt19937(1));
    std::vector<unsigned> next(n * 32);
    for (size_t i = 0; i < n; ++i) next[perm[i] * 32] = perm[(i + 1) % n] * 32;
    unsigned *d;
    cudaMalloc(&d, n * 32 * 4);
    cudaMemcpy(d, next.data(), n * 32 * 4, cudaMemcpyHostToDevice);
    for (int sm_rep = 0; sm_rep < 2; ++sm_rep) {
      chase<<<1, 1>>>(d, 2000, out, sink);
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    }
    printf("ldcg chase %8zu KB: %7.1f ns/hop  %7.1f cycles/hop\n", bytes >> 10, h[0] / 2000.0, h[1] / 2000.0);
    if (bytes <= (size_t(16) << 10)) {
      chase_l1<<<1, 1>>>(d, 2000, out, sink);
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("L1 chase   %8zu KB: %7.1f cycles/hop\n", bytes >> 10, h[1] / 2000.0);
    }
    cudaFree(d);
  }
  unsigned *ctr;
  cudaMalloc(&ctr, 4096);
  cudaMemset(ctr, 0, 4096);
  for (int rep = 0; rep < 2; ++rep) atom_rt<<<1, 1>>>(ctr, 1000, out);
  cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
  printf("atomicAdd round trip: %.1f cycles\n", h[1] / 1000.0);
  return 0;
}
