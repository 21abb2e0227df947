// What limits the leaf GEMM?  Synthetic loops with the K3 inner structure:
//  mode 0: fragments from smem + DMMA, no barrier
//  mode 1: + __syncthreads every 32-k step
//  mode 2: + cp.async refill of a 32 KB stage from L2 every step (3-stage ring)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ int swz(int row, int col) {
  const int chunk = col >> 1;
  return (((chunk & ~7) | ((chunk & 7) ^ ((row & 3) << 1))) << 1) | (col & 1);
}
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
template <int MODE>
__global__ void __launch_bounds__(256) probe(const double *g, double *out, int steps, long long span) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / 4, wn = warp % 4, gg = lane >> 2, t = lane & 3;
  for (int i = tid; i < 3 * 4096; i += 256) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double acc[2][2][4] = {};
  const double *src = g + (blockIdx.x % 64) * 4096;
  for (int step = 0; step < steps; ++step) {
    const int stage = step % 3;
    if (MODE == 2) {
      asm volatile("cp.async.wait_group 1;\n");
      __syncthreads();
      double *dst = sm + ((step + 2) % 3) * 4096;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = tid + q * 256;
        cp16(dst + 2 * e, g + (((long long)blockIdx.x * 7919 + (long long)step * 37) % (span / 4096)) * 4096 + 2 * e);
      }
      asm volatile("cp.async.commit_group;\n");
    } else if (MODE == 1) {
      __syncthreads();
    }
    const double *As = sm + stage * 4096, *Bs = As + 2048;
#pragma unroll
    for (int kk = 0; kk < 32; kk += 16) {
      double af[2][2][4], bf[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            const int r = wm * 32 + mt * 16 + 8 * h + gg;
            af[mt][h][s4] = As[r * 32 + swz(r, kk + 4 * s4 + t)];
          }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
          const int r = kk + 4 * s4 + t;
          bf[nt][s4] = Bs[r * 64 + swz(r, wn * 16 + nt * 8 + gg)];
        }
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
              dmma884(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1], af[mt][h][s4], bf[nt][s4]);
    }
  }
  double s = 0;
  for (int a = 0; a < 2; ++a) for (int b = 0; b < 2; ++b) for (int c = 0; c < 4; ++c) s += acc[a][b][c];
  out[blockIdx.x * 256 + tid] = s;
}
int main() {
  double *g, *o;
  cudaMalloc(&g, 8ull << 25);
  cudaMalloc(&o, 8 << 20);
  cudaMemset(g, 0, 8ull << 25);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int steps = 2000;
  long long span = 0;
  auto run = [&](auto kern, const char *name, int per_sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 4096 * 8);
    kern<<<sms * per_sm, 256, 3 * 4096 * 8>>>(g, o, steps, span);
    cudaEventRecord(e0);
    kern<<<sms * per_sm, 256, 3 * 4096 * 8>>>(g, o, steps, span);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * 64 * 32 * steps * (double)sms * per_sm;
    printf("%s ctas/sm=%d: %.2f TFLOP/s (%s)\n", name, per_sm, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (long long sp : {1ll << 18, 1ll << 22, 1ll << 24}) {  // doubles: 2 MB, 32 MB, 128 MB
    span = sp - 8192;
    printf("span %lld MB\n", sp * 8 >> 20);
    run(probe<2>, "+cp.async      ", 2);
  }
  return 0;
}
