// Grid-barrier latency probe: cooperative kernel, many CTAs, K barriers in a
// row; reports ns per barrier for several barrier implementations.
#include <cooperative_groups.h>
#include <cuda/atomic>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

template <int V>
__device__ void bar_sync(unsigned *bar, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (V == 0) {  // current library implementation
      cuda::atomic_ref<unsigned, cuda::thread_scope_device> cnt(bar[0]), gen(bar[1]);
      const unsigned g = gen.load(cuda::memory_order_acquire);
      __threadfence();
      if (cnt.fetch_add(1u, cuda::memory_order_acq_rel) == n - 1) {
        cnt.store(0u, cuda::memory_order_relaxed);
        gen.fetch_add(1u, cuda::memory_order_release);
      } else {
        while (gen.load(cuda::memory_order_acquire) == g) __nanosleep(32);
      }
      __threadfence();
    } else if (V == 1) {  // relaxed polling, one fence each side
      volatile unsigned *vgen = bar + 1;
      const unsigned g = *vgen;
      __threadfence();
      if (atomicAdd(bar, 1u) == n - 1) {
        bar[0] = 0;
        __threadfence();
        atomicAdd(bar + 1, 1u);
      } else {
        while (*vgen == g) {}
      }
      __threadfence();
    } else if (V == 2) {  // generation counter only: arrival = add, wait for multiple of n
      unsigned old;
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
      const unsigned target = (old / n + 1) * n;
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      } while ((int)(cur - target) < 0);
    } else if (V == 3) {  // same, relaxed poll then one acquire fence
      unsigned old;
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
      const unsigned target = (old / n + 1) * n;
      unsigned cur;
      do {
        asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      } while ((int)(cur - target) < 0);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
  __syncthreads();
}

template <int V>
__global__ void probe(unsigned *bar, unsigned long long *out, int K) {
  if (V == 4) {
    cg::grid_group g = cg::this_grid();
    g.sync();
    const unsigned long long t0 = gt();
    for (int k = 0; k < K; ++k) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = gt() - t0;
    return;
  }
  bar_sync<V>(bar, gridDim.x);
  const unsigned long long t0 = gt();
  for (int k = 0; k < K; ++k) bar_sync<V>(bar, gridDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = gt() - t0;
}

template <int V>
void run(int blocks, const char *name) {
  unsigned *bar;
  unsigned long long *out, h;
  cudaMalloc(&bar, 64);
  cudaMemset(bar, 0, 64);
  cudaMalloc(&out, 8);
  int K = 200;
  void *args[] = {&bar, &out, &K};
  for (int rep = 0; rep < 2; ++rep)
    cudaLaunchCooperativeKernel((void *)probe<V>, blocks, 256, args, 0, 0);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%-36s blocks=%4d  %8.1f ns/barrier  (%s)\n", name, blocks, (double)h / K, cudaGetErrorString(e));
  cudaFree(bar);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int b : {sms, 2 * sms}) {
    run<0>(b, "acq/acq_rel + threadfence + nanosleep");
    run<1>(b, "volatile poll + threadfence");
    run<2>(b, "gen counter, acquire poll");
    run<3>(b, "gen counter, relaxed poll + fence");
    run<4>(b, "cooperative_groups grid.sync");
  }
  // launch overhead: empty cooperative vs normal launch
  return 0;
}
