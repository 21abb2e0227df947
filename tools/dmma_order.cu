// Does DMMA (mma.sync f64) accumulate exactly like a sequential FMA chain
// over k?  Compares m8n8k4 / m16n8k16 chains against host std::fma chains.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <cuda_runtime.h>

constexpr int K = 64;

__global__ void k_m8n8k4(const double* A, const double* B, double* C) {
  // A: 8 x K row-major, B: K x 8 row-major, C: 8 x 8
  int lane = threadIdx.x;
  double c0 = 0, c1 = 0;
  for (int k0 = 0; k0 < K; k0 += 4) {
    double a = A[(lane >> 2) * K + k0 + (lane & 3)];
    double b = B[(k0 + (lane & 3)) * 8 + (lane >> 2)];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  }
  C[(lane >> 2) * 8 + (lane & 3) * 2] = c0;
  C[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = c1;
}

__global__ void k_m16n8k16(const double* A, const double* B, double* C) {
  // A: 16 x K, B: K x 8, C: 16 x 8
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double c[4] = {0, 0, 0, 0};
  for (int k0 = 0; k0 < K; k0 += 16) {
    double a[8], b[4];
    // A frag (m16k16 row): a_i: row = g + 8*(i&1), col = t + 4*(i>>1)
    for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i & 1)) * K + k0 + t + 4 * (i >> 1)];
    // B frag (k16n8 col): b_i: row = t + 4*i, col = g
    for (int i = 0; i < 4; ++i) b[i] = B[(k0 + t + 4 * i) * 8 + g];
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  // C frag: c_i: row = g + 8*(i>>1), col = 2t + (i&1)
  for (int i = 0; i < 4; ++i) C[(g + 8 * (i >> 1)) * 8 + 2 * t + (i & 1)] = c[i];
}

int main() {
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  double *A, *B, *C;
  cudaMallocManaged(&A, 16 * K * 8); cudaMallocManaged(&B, K * 8 * 8); cudaMallocManaged(&C, 16 * 8 * 8);
  int trials = 200, bad8 = 0, bad16 = 0, badfused8 = 0;
  for (int tr = 0; tr < trials; ++tr) {
    for (int i = 0; i < 16 * K; ++i) A[i] = nd(rng) * std::exp(nd(rng) * 3);
    for (int i = 0; i < K * 8; ++i) B[i] = nd(rng) * std::exp(nd(rng) * 3);
    k_m8n8k4<<<1, 32>>>(A, B, C); cudaDeviceSynchronize();
    for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) {
      double acc = 0; for (int k = 0; k < K; ++k) acc = std::fma(A[r * K + k], B[k * 8 + c], acc);
      if (acc != C[r * 8 + c]) ++bad8;
      // alternative: each group of 4 summed with one rounding then added (approximate with long double)
      long double acc2 = 0; double accd = 0;
      for (int k0 = 0; k0 < K; k0 += 4) { long double s = accd; for (int k = k0; k < k0 + 4; ++k) s += (long double)A[r*K+k] * B[k*8+c]; accd = (double)s; }
      (void)acc2; if (accd != C[r * 8 + c]) ++badfused8;
    }
    k_m16n8k16<<<1, 32>>>(A, B, C); cudaDeviceSynchronize();
    for (int r = 0; r < 16; ++r) for (int c = 0; c < 8; ++c) {
      double acc = 0; for (int k = 0; k < K; ++k) acc = std::fma(A[r * K + k], B[k * 8 + c], acc);
      if (acc != C[r * 8 + c]) ++bad16;
    }
  }
  printf("{\"m8n8k4_mismatch_vs_fma_chain\": %d, \"m8n8k4_mismatch_vs_fused4\": %d, \"m16n8k16_mismatch_vs_fma_chain\": %d, \"elements\": %d}\n",
         bad8, badfused8, bad16, trials * 64);
  return 0;
}
