// HBM read ceiling on one B200 for a streaming read of a large array (the K1
// dense build's access pattern): (a) LDG.128 grid-stride with a sum, (b) 1-D
// bulk copies (cp.async.bulk, SASS UBLKCP) into a shared-memory ring of
// CHUNK-byte stages per CTA, one elected thread issuing, a warp consuming.
// usage: read_probe [GiB=32]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void ldg_sum(const double2 *__restrict__ p, size_t n2, double *out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2;
       i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) *out = s;
}

__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(64) bulk_sum(const char *__restrict__ p, size_t bytes, double *out, int rows = 0) {
  // rows != 0: K1's dense-build pattern on an N = 65536 f64 matrix (512 KB per
  // row): chunk c = (group, r) reads the 16 KB of row r of a 32-leaf group;
  // rows == 1: a CTA streams whole groups (64 rows, 512 KB apart);
  // rows == 2: the same with four adjacent CTAs sharing a block row's pages
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const size_t nchunks = bytes / CHUNK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) {
    if (lane == 0) {
      int it = 0;
      for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) {
          const unsigned par = ((it / STAGES) - 1) & 1;
          asm volatile("{\n .reg .pred q;\n W_%=: mbarrier.try_wait.parity.shared.b64 q, [%0], %1;\n @!q bra W_%=;\n}"
                       ::"r"(sa(&empty[s])), "r"(par));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(CHUNK));
        size_t off = c * CHUNK;
        if (rows) {
          // the CTA's it-th chunk: group blockIdx.x + (it / 64) * gridDim.x, row it % 64
          const size_t g = blockIdx.x + (size_t)(it / 64) * gridDim.x, r = it % 64;
          off = ((g / 32) * 64 + r) * (size_t)(65536 * 8) + (g % 32) * (size_t)16384;
          if (off + CHUNK > bytes) off = 0;
        }
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(smem + s * CHUNK)), "l"(p + off), "r"(CHUNK), "r"(sa(&full[s])) : "memory");
      }
    }
  } else {
    double acc = 0;
    int it = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
      const int s = it % STAGES;
      const unsigned par = (it / STAGES) & 1;
      asm volatile("{\n .reg .pred q;\n W_%=: mbarrier.try_wait.parity.shared.b64 q, [%0], %1;\n @!q bra W_%=;\n}"
                   ::"r"(sa(&full[s])), "r"(par));
      const double2 *q = reinterpret_cast<const double2 *>(smem + s * CHUNK);
      for (int i = lane; i < CHUNK / 16; i += 32) acc += q[i].x + q[i].y;
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(sa(&empty[s])));
    }
    if (acc == 12345.678) *out = acc;
  }
}

template <int STAGES, int CHUNK>
static void run_bulk(const char *p, size_t bytes, double *out, int ctas_per_sm, int sms, int rows = 0) {
  auto k = bulk_sum<STAGES, CHUNK>;
  const int sm = STAGES * CHUNK;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<<<sms * ctas_per_sm, 64, sm>>>(p, bytes, out, rows);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("bulk%s stages=%d chunk=%d ctas/sm=%d: %.3f ms %.0f GB/s\n", rows ? " (K1 row pattern)" : "", STAGES, CHUNK, ctas_per_sm, best,
         bytes / (best * 1e-3) / 1e9);
}

int main(int argc, char **argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 32.0;
  const size_t bytes = (size_t)(gib * (1ull << 30)) / 65536 * 65536;
  char *p; double *out;
  CK(cudaMalloc(&p, bytes));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(p, 1, bytes));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int cps : {4, 8, 16}) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      ldg_sum<<<sms * cps, 256>>>((const double2 *)p, bytes / 16, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("ldg ctas/sm=%d: %.3f ms %.0f GB/s\n", cps, best, bytes / (best * 1e-3) / 1e9);
  }
  run_bulk<4, 16384>(p, bytes, out, 2, sms);
  run_bulk<4, 16384>(p, bytes, out, 3, sms);
  run_bulk<6, 16384>(p, bytes, out, 2, sms);
  run_bulk<3, 32768>(p, bytes, out, 2, sms);
  run_bulk<8, 8192>(p, bytes, out, 3, sms);
  run_bulk<4, 32768>(p, bytes, out, 1, sms);
  run_bulk<3, 16384>(p, bytes, out, 4, sms);
  run_bulk<3, 16384>(p, bytes, out, 4, sms, 1);
  run_bulk<4, 16384>(p, bytes, out, 3, sms, 1);
  run_bulk<6, 16384>(p, bytes, out, 2, sms, 1);
  return 0;
}
