// FP64 peak microbenchmarks for B200 (sm_100a): DMMA (mma.sync f64) throughput,
// DFMA throughput and DADD dependent-chain latency.  Output is one JSON line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int ACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[ACC][4];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_tp(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  const double m = 0.999999, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], m, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_tp(float* out, int iters) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  const float m = 0.999999f, c = 1e-9f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], m, c);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dadd_chain(double* out, int iters, long long* cyc) {
  double acc = threadIdx.x, e = 1e-7 * (threadIdx.x + 1);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, e);
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(double) * 1 << 22));
  CK(cudaMalloc(&cyc, sizeof(long long)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto launch) -> float {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
  };
  const int iters = 4096;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  for (int warps : {4, 8, 16}) {
    int blocks = sms * 2, threads = warps * 32;
    float ms = timeit([&] { dmma_m8n8k4<8><<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * warps);
    printf(", \"dmma_m8n8k4_w%d_tflops\": %.3f", warps, flops / ms / 1e9);
    ms = timeit([&] { dmma_m16n8k16<4><<<blocks, threads>>>(out, iters / 4); });
    flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (blocks * warps);
    printf(", \"dmma_m16n8k16_w%d_tflops\": %.3f", warps, flops / ms / 1e9);
  }
  {
    int blocks = sms * 4, threads = 512;
    float ms = timeit([&] { dfma_tp<<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf(", \"dfma_tflops\": %.3f", flops / ms / 1e9);
    ms = timeit([&] { ffma_tp<<<blocks, threads>>>((float *)out, iters); });
    flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf(", \"ffma_tflops\": %.3f", flops / ms / 1e9);
  }
  {
    dadd_chain<<<1, 32>>>(out, 1024, cyc); CK(cudaDeviceSynchronize());
    long long c; CK(cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost));
    printf(", \"dadd_latency_cycles\": %.2f", c / (1024.0 * 16));
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
